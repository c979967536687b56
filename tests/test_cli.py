"""GPU CLI (cli.py) and Matrix Market I/O: the reference's commands, JSON/CSV
schema, error wording and exit codes (reference cli.py, matrix_io.py:111-252)."""

import io
import json

import numpy as np
import pytest

import paper_2204_06666_b200 as E
from paper_2204_06666_b200 import cli
from paper_2204_06666_b200 import workloads as W


def _write_mtx(tmp_path, name="a.mtx", symmetric=False):
    n, r, c, v = W.permute_symmetric(*W.stencil27(8, 8, 8), seed=3)
    m = E.CooMatrix(n, n, r, c, v)
    path = tmp_path / name
    E.write_matrix_market(m, str(path))
    return m, path


def test_matrix_market_round_trip_and_symmetric_expansion(tmp_path):
    m, path = _write_mtx(tmp_path)
    m2 = E.parse_matrix_market(str(path))
    assert (m2.n_rows, m2.nnz) == (m.n_rows, m.nnz)
    order = np.lexsort((m.cols, m.rows))
    assert np.array_equal(m2.rows, m.rows[order]) and np.array_equal(m2.cols, m.cols[order])
    assert np.array_equal(m2.values, m.values[order])  # %.17g round-trips doubles
    text = (b"%%MatrixMarket matrix coordinate real symmetric\n% c\n3 3 3\n1 1 2.0\n"
            b"3 1 -1.5\n3 1 0.5\n")
    s = E.parse_matrix_market(text)
    assert s.rows.tolist() == [0, 0, 2] and s.cols.tolist() == [0, 2, 0]
    assert s.values.tolist() == [2.0, -1.0, -1.0]  # mirrored, duplicates summed
    p = E.parse_matrix_market(b"%%MatrixMarket matrix coordinate pattern general\n2 2 1\n2 1\n")
    assert p.values.tolist() == [1.0]


@pytest.mark.parametrize("text,exc,msg", [
    (b"", E.MatrixMarketError, "line 1: empty input"),
    (b"%%MatrixMarket matrix array real general\n1 1\n1\n", E.UnsupportedFormatError, "array"),
    (b"%%MatrixMarket matrix coordinate complex general\n", E.UnsupportedFormatError, "complex"),
    (b"%%MatrixMarket matrix coordinate real hermitian\n", E.UnsupportedFormatError, "symmetry"),
    (b"%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1.0\n", E.MatrixMarketError,
     "line 3: index out of declared bounds"),
    (b"%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n", E.MatrixMarketError,
     "expected 2 entries, found 1"),
    (b"%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 1.0\n2 2 1.0\n",
     E.MatrixMarketError, "line 4: extra entry"),
    (b"%%MatrixMarket matrix coordinate real general\n2 2 1\n1 x 1.0\n", E.MatrixMarketError,
     "line 3: malformed entry"),
    (b"%%MatrixMarket matrix coordinate real general\n2 2\n", E.MatrixMarketError,
     "line 2: size line must be"),
])
def test_matrix_market_errors_name_the_line(text, exc, msg):
    with pytest.raises(exc, match=msg):
        E.parse_matrix_market(text)


def test_convert_and_stats_commands(tmp_path, capsys):
    m, path = _write_mtx(tmp_path)
    flags = ["--P", "8", "--shm-bytes", "8192"]
    assert cli.main(["convert", str(path), "-o", str(tmp_path / "a.ehyb"), *flags]) == 0
    rec = json.loads(capsys.readouterr().out)
    assert rec["dimension"] == m.n_rows and rec["nnz"] == m.nnz and rec["n_parts"] == 8
    e = E.read_ehyb_container(str(tmp_path / "a.ehyb"))
    assert e.nnz_ell == rec["nnz_ell"] and e.nnz_er == rec["nnz_er"]
    assert cli.main(["stats", str(path), *flags]) == 0
    st = json.loads(capsys.readouterr().out)
    assert st["nnz_ell"] + st["nnz_er"] == m.nnz and len(st["width_histograms"]) == 8
    assert "quoted_double_precision_savings" in st["footprint"]


def test_usage_errors_exit_2(tmp_path, capsys):
    assert cli.main(["stats", str(tmp_path / "missing.mtx")]) == 2
    bad = tmp_path / "bad.mtx"
    bad.write_bytes(b"%%MatrixMarket matrix coordinate real general\n2 3 1\n1 1 1.0\n")
    assert cli.main(["convert", str(bad)]) == 2
    assert "matrix must be square" in capsys.readouterr().err


def test_bench_csv_schema_round_trip():
    rep = cli.BenchReport(
        matrix="a.mtx", dimension=10, nnz=20, n_parts=2, vec_cache_size=32, inner_fraction=0.5,
        nnz_ell=12, nnz_er=8, footprint_total_bytes=100, savings_vs_32bit_cols=0.1,
        traffic_model_bytes=200, workers=1, scheduling="static", reps=3, warmup=1,
        partition_s=0.1, reorder_assemble_s=0.2, prep_to_spmv_ratio=3.0,
        kernels=[cli.KernelTiming("ehyb", 1e-5, 4.0), cli.KernelTiming("csr-oracle", 2e-5, 2.0)])
    buf = io.StringIO()
    cli.write_bench_csv(rep, buf)
    rows = cli.read_bench_csv(io.StringIO(buf.getvalue()))
    assert [r["kernel"] for r in rows] == ["ehyb", "csr-oracle"]
    assert rows[0]["schema_version"] == 1 and rows[0]["nnz"] == 20 and rows[1]["gflops"] == 2.0
    assert list(rows[0]) == cli.BENCH_CSV_COLUMNS
    with pytest.raises(ValueError, match="unsupported bench CSV schema"):
        cli.read_bench_csv(io.StringIO(buf.getvalue().replace("\n1,", "\n2,")))


@pytest.mark.gpu
def test_verify_and_bench_on_gpu(tmp_path, capsys):
    m, path = _write_mtx(tmp_path)
    flags = ["--P", "8", "--shm-bytes", "8192"]
    assert cli.main(["verify", str(path), "--vectors", "3", *flags]) == 0
    rec = json.loads(capsys.readouterr().out)
    assert rec["status"] == "pass" and rec["max_rel_error"] <= 1e-12
    assert cli.main(["verify", str(path), "--tau", "4", *flags]) == 0
    assert json.loads(capsys.readouterr().out)["max_rel_error"] <= 1e-5
    assert cli.main(["convert", str(path), "-o", str(tmp_path / "a.ehyb"), *flags]) == 0
    capsys.readouterr()
    assert cli.main(["verify", str(tmp_path / "a.ehyb")]) == 0
    assert json.loads(capsys.readouterr().out)["status"] == "pass"
    assert cli.main(["bench", str(path), "--reps", "5", "--warmup", "2", *flags]) == 0
    rep = json.loads(capsys.readouterr().out)
    assert [k["kernel"] for k in rep["kernels"]] == ["ehyb", "csr-oracle"]
    assert rep["gpu"]["csr_cusparse"]["gflops"] > 0
    assert rep["gpu"]["effective_gbs"] > 0
    out = tmp_path / "b.csv"
    assert cli.main(["bench", str(path), "--reps", "3", "--out", "csv", "--output", str(out),
                     *flags]) == 0
    assert len(cli.read_bench_csv(str(out))) == 2
