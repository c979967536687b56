"""Synthetic workloads for the BASELINE.json configs, parity tests and bench.

Pure numpy (plus scipy's cKDTree for the random geometric graph); no native
code, so the golden-fixture script can feed the very same matrices to the
reference package. Every generator returns ``(n, rows, cols, values)`` with
int64 coordinates and float64 values and no duplicate coordinates.

Config map (BASELINE.json ``configs``, construction per SURVEY.md §8d):

* ``cfg1`` 2D 5-point Laplacian 512x512, natural order, fp64.
* ``cfg2`` 27-point stencil on 128^3 (diag 26, off -1), symmetric random
  permutation ``P A P^T`` with ``default_rng(1).permutation(n)``, fp64.
* ``cfg3`` 3D random geometric graph, 5M points, mean degree 14, fp32 / fp64.
* ``cfg4`` cfg2 generator at 96^3 plus 32 symmetric heavy-tailed coupling
  rows (Pareto(1.2) lengths 1e3 .. 3e5), fp64.
* ``cfg5`` 27-point stencil on 256^3, natural order, fp64 (multi-GPU CG).
"""

from __future__ import annotations

import numpy as np

LCG_A = 6364136223846793005
LCG_C = 1442695040888963407
LCG_MIX = 0x9E3779B97F4A7C15


def deterministic_vector(length: int, seed: int) -> np.ndarray:
    """The reference's platform-independent x generator (cli.py:89-108).

    64-bit LCG s_{k+1} = a s_k + c mod 2^64 started from seed ^ MIX; entry k is
    the top 53 bits of s_{k+1} mapped onto [-1, 1). Computed here by block
    doubling: with (A_m, C_m) the m-step affine map, state_{i+m} = A_m state_i
    + C_m, so each pass doubles the number of known states.
    """
    if length < 0:
        raise ValueError("length must be non-negative")
    if length == 0:
        return np.zeros(0, dtype=np.float64)
    mask = (1 << 64) - 1
    s1 = (LCG_A * ((seed ^ LCG_MIX) & mask) + LCG_C) & mask
    states = np.empty(length, dtype=np.uint64)
    states[0] = np.uint64(s1)
    known = 1
    step_a, step_c = LCG_A, LCG_C  # map for `known` steps
    with np.errstate(over="ignore"):
        while known < length:
            take = min(known, length - known)
            states[known : known + take] = (
                states[:take] * np.uint64(step_a) + np.uint64(step_c)
            )
            # compose the map with itself: x -> a(a x + c) + c
            step_a, step_c = (step_a * step_a) & mask, (step_a * step_c + step_c) & mask
            known += take
    return 2.0 * ((states >> np.uint64(11)).astype(np.float64) * 2.0**-53) - 1.0


def laplacian_2d(nx: int, ny: int):
    """5-point stencil, diag 4 / off -1, vertex id ix*ny + iy."""
    n = nx * ny
    ix, iy = np.meshgrid(np.arange(nx), np.arange(ny), indexing="ij")
    vid = (ix * ny + iy).ravel()
    rows, cols, vals = [vid], [vid], [np.full(n, 4.0)]
    for dx, dy in ((1, 0), (-1, 0), (0, 1), (0, -1)):
        jx, jy = ix + dx, iy + dy
        ok = ((jx >= 0) & (jx < nx) & (jy >= 0) & (jy < ny)).ravel()
        rows.append(vid[ok])
        cols.append((jx * ny + jy).ravel()[ok])
        vals.append(np.full(int(ok.sum()), -1.0))
    return n, np.concatenate(rows), np.concatenate(cols), np.concatenate(vals)


def stencil27(nx: int, ny: int, nz: int, diag: float = 26.0, off: float = -1.0):
    """27-point hexahedral stencil, vertex id (ix*ny + iy)*nz + iz.

    Entries are emitted row-major (row ascending, column ascending), which is
    also the order the reference's assembly sorts into.
    """
    n = nx * ny * nz
    idx = np.arange(n, dtype=np.int64)
    iz = idx % nz
    iy = (idx // nz) % ny
    ix = idx // (ny * nz)
    rows_l, cols_l, vals_l = [], [], []
    for dx in (-1, 0, 1):
        for dy in (-1, 0, 1):
            for dz in (-1, 0, 1):
                ok = (
                    (ix + dx >= 0) & (ix + dx < nx)
                    & (iy + dy >= 0) & (iy + dy < ny)
                    & (iz + dz >= 0) & (iz + dz < nz)
                )
                r = idx[ok]
                rows_l.append(r)
                cols_l.append(r + (dx * ny + dy) * nz + dz)
                v = diag if (dx, dy, dz) == (0, 0, 0) else off
                vals_l.append(np.full(r.size, v))
    rows = np.concatenate(rows_l)
    cols = np.concatenate(cols_l)
    vals = np.concatenate(vals_l)
    if n > 4_000_000:
        # entry order does not change any EHYB structure (assembly sorts each
        # row by column); skip the 400M-key sort at multi-GPU sizes
        return n, rows, cols, vals
    order = np.argsort(rows * np.int64(n) + cols, kind="stable")
    return n, rows[order], cols[order], vals[order]


def permute_symmetric(n: int, rows, cols, vals, seed: int):
    """P A P^T with perm = default_rng(seed).permutation(n): old vertex i
    becomes new vertex perm[i]."""
    perm = np.random.default_rng(seed).permutation(n).astype(np.int64)
    return n, perm[rows], perm[cols], vals


def rgg3d(n: int, mean_degree: float = 14.0, seed: int = 7):
    """3D random geometric graph: uniform points in [0,1)^3 from
    default_rng(seed), edge when the distance is below
    r = (3 * mean_degree / (4 pi n))^(1/3); off-diagonal -1, diagonal
    degree + 1 (strictly diagonally dominant, SPD)."""
    from scipy.spatial import cKDTree

    pts = np.random.default_rng(seed).random((n, 3))
    r = (3.0 * mean_degree / (4.0 * np.pi * n)) ** (1.0 / 3.0)
    pairs = cKDTree(pts).query_pairs(r, output_type="ndarray").astype(np.int64)
    i, j = pairs[:, 0], pairs[:, 1]
    deg = np.bincount(i, minlength=n) + np.bincount(j, minlength=n)
    diag = np.arange(n, dtype=np.int64)
    rows = np.concatenate([i, j, diag])
    cols = np.concatenate([j, i, diag])
    vals = np.concatenate([np.full(2 * i.size, -1.0), deg.astype(np.float64) + 1.0])
    order = np.argsort(rows * np.int64(n) + cols, kind="stable")
    return n, rows[order], cols[order], vals[order]


def heavy_tail(k: int = 96, n_hubs: int = 32, seed: int = 4,
               min_len: int = 1000, max_len: int = 300_000):
    """Permuted 27-point k^3 stencil plus `n_hubs` symmetric dense coupling
    rows/columns with Pareto(1.2) lengths in [min_len, max_len]. Coupling
    values are -1e-3 and each diagonal grows by 1e-3 per coupling, so the
    matrix stays strictly diagonally dominant (SPD)."""
    n, r, c, v = permute_symmetric(*stencil27(k, k, k), seed=1)
    rng = np.random.default_rng(seed)
    hubs = rng.choice(n, size=n_hubs, replace=False).astype(np.int64)
    lengths = np.clip((min_len * (1.0 + rng.pareto(1.2, size=n_hubs))).astype(np.int64),
                      min_len, min(max_len, n - 1))
    hr, hc = [], []
    for h, length in zip(hubs, lengths):
        t = rng.choice(n, size=int(length), replace=False).astype(np.int64)
        t = t[t != h]
        hr += [np.full(t.size, h), t]
        hc += [t, np.full(t.size, h)]
    hr = np.concatenate(hr)
    hc = np.concatenate(hc)
    key_new = np.unique(hr * np.int64(n) + hc)
    key_old = r * np.int64(n) + c
    key_new = key_new[~np.isin(key_new, key_old)]
    nr, nc = key_new // n, key_new % n
    extra = np.bincount(nr, minlength=n).astype(np.float64) * 1e-3
    v = v.copy()
    d = r == c
    v[d] += extra[r[d]]
    rows = np.concatenate([r, nr])
    cols = np.concatenate([c, nc])
    vals = np.concatenate([v, np.full(nr.size, -1e-3)])
    order = np.argsort(rows * np.int64(n) + cols, kind="stable")
    return n, rows[order], cols[order], vals[order]


# --------------------------------------------------------------------------
# named configs
# --------------------------------------------------------------------------

#: config name -> (description, tau, builder)
CONFIGS = {
    "cfg1": ("2D 5-point Laplacian 512x512 (natural order)", 8,
             lambda: laplacian_2d(512, 512)),
    "cfg2": ("3D 27-point stencil 128^3, random symmetric permutation (seed 1)", 8,
             lambda: permute_symmetric(*stencil27(128, 128, 128), seed=1)),
    "cfg3f32": ("3D random geometric graph 5M rows, mean degree 14 (seed 7)", 4,
                lambda: rgg3d(5_000_000)),
    "cfg3f64": ("3D random geometric graph 5M rows, mean degree 14 (seed 7)", 8,
                lambda: rgg3d(5_000_000)),
    "cfg4": ("27-point 96^3 permuted + 32 heavy-tailed coupling rows (seed 4)", 8,
             lambda: heavy_tail()),
    "cfg5": ("3D 27-point stencil 256^3 (natural order)", 8,
             lambda: stencil27(256, 256, 256)),
    # scaled-down variants used by parity tests
    "cfg2s": ("3D 27-point stencil 32^3, random symmetric permutation (seed 1)", 8,
              lambda: permute_symmetric(*stencil27(32, 32, 32), seed=1)),
    "cfg3s": ("3D random geometric graph 200k rows (seed 7)", 4,
              lambda: rgg3d(200_000)),
    "cfg4s": ("27-point 24^3 permuted + 8 heavy-tailed coupling rows", 8,
              lambda: heavy_tail(k=24, n_hubs=8, min_len=100, max_len=5000)),
    # cfg5's structure (natural-order 27-point stencil, K=4 persistent CTAs,
    # 592 partitions on 148 SMs) at 1/8 scale, under a profile whose
    # shared-memory budget forces K=4: pins the K-wave path to the reference
    "cfg5k4": ("3D 27-point stencil 128^3 (natural order), K=4 profile (148, 32, 28416)", 8,
               lambda: stencil27(128, 128, 128)),
}

#: configs quoted on a profile other than the B200 default (148, 32, 231424)
CONFIG_PROFILES = {
    "cfg5k4": (148, 32, 28416),
}


def build_config(name: str):
    """Return (n, rows, cols, values, tau) for a named config."""
    _, tau, fn = CONFIGS[name]
    n, r, c, v = fn()
    return n, r, c, v, tau


# --------------------------------------------------------------------------
# the reference test corpus, regenerated (same numpy call sequence as the
# reference's tests/helpers.py:75-81 and 128-157, so the matrices are equal)
# --------------------------------------------------------------------------

def random_coo(n: int, density: float, seed: int):
    rng = np.random.default_rng(seed)
    nnz = max(1, int(round(density * n * n)))
    flat = rng.choice(n * n, size=min(nnz, n * n), replace=False)
    vals = rng.uniform(-1.0, 1.0, size=flat.size)
    return n, (flat // n).astype(np.int64), (flat % n).astype(np.int64), vals


def tridiagonal(n: int, diag: float = 2.0, off: float = -1.0):
    rows, cols, vals = [], [], []
    for i in range(n):
        for j in (i - 1, i, i + 1):
            if 0 <= j < n:
                rows.append(i)
                cols.append(j)
                vals.append(diag if i == j else off)
    return n, np.asarray(rows, np.int64), np.asarray(cols, np.int64), np.asarray(vals, float)


def laplacian_3d7(nx: int, ny: int, nz: int):
    """7-point stencil, diag 6 / off -1."""
    n = nx * ny * nz
    ix, iy, iz = np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij")
    vid = ((ix * ny + iy) * nz + iz).ravel()
    rows, cols, vals = [vid], [vid], [np.full(n, 6.0)]
    for dx, dy, dz in ((1, 0, 0), (-1, 0, 0), (0, 1, 0), (0, -1, 0), (0, 0, 1), (0, 0, -1)):
        jx, jy, jz = ix + dx, iy + dy, iz + dz
        ok = ((jx >= 0) & (jx < nx) & (jy >= 0) & (jy < ny) & (jz >= 0) & (jz < nz)).ravel()
        rows.append(vid[ok])
        cols.append(((jx * ny + jy) * nz + jz).ravel()[ok])
        vals.append(np.full(int(ok.sum()), -1.0))
    return n, np.concatenate(rows), np.concatenate(cols), np.concatenate(vals)


def balanced_random_assignment(n_vertices: int, n_parts: int, seed: int) -> np.ndarray:
    """Seeded balanced random assignment (reference partition.py:207-221):
    permutation split into n_parts nearly equal chunks."""
    perm = np.random.default_rng(seed).permutation(n_vertices)
    assignment = np.empty(n_vertices, dtype=np.int64)
    for pid, chunk in enumerate(np.array_split(perm, n_parts)):
        assignment[chunk] = pid
    return assignment


def corpus_specs():
    """The reference acceptance corpus (500 random cases + stencil families).

    Yields dicts: name, n, rows, cols, vals, tau, profile (procs, warp, shm),
    assignment (None -> built-in partitioner, else an external partition
    over `n_parts_hint` parts), seed.
    """
    rng = np.random.default_rng(20240611)
    for i in range(500):
        n = int(rng.integers(8, 513))
        density = float(np.exp(rng.uniform(np.log(0.001), np.log(0.1))))
        tau = 4 if i % 5 == 4 else 8
        procs = int(rng.choice([1, 2, 4]))
        warp = int(rng.choice([4, 8, 32]))
        slots = warp * int(rng.integers(1, 9))
        shm = slots * tau
        mseed = int(rng.integers(0, 2**31))
        _, r, c, v = random_coo(n, density, seed=mseed)
        # compute_params inline (format.py:83-107) to size the external partition
        k = 1
        while True:
            n_parts = k * procs
            vec = -(-(-(-n // n_parts)) // warp) * warp
            if vec * tau <= shm and vec <= 1 << 16:
                break
            k += 1
        if i % 2 == 0:
            assignment = None
        else:
            assignment = balanced_random_assignment(n, n_parts, int(rng.integers(0, 2**31)))
        yield dict(name=f"random[{i}] n={n}", n=n, rows=r, cols=c, vals=v, tau=tau,
                   profile=(procs, warp, shm), assignment=assignment,
                   n_parts_hint=n_parts, seed=i)
    sp = (4, 32, 48 * 1024)
    for n in (64, 512, 4096, 32768):
        _, r, c, v = tridiagonal(n)
        yield dict(name=f"chain n={n}", n=n, rows=r, cols=c, vals=v, tau=8, profile=sp,
                   assignment=None, n_parts_hint=None, seed=0)
    for k in (8, 16, 64, 181):
        nn, r, c, v = laplacian_2d(k, k)
        yield dict(name=f"grid2d {k}x{k}", n=nn, rows=r, cols=c, vals=v, tau=8, profile=sp,
                   assignment=None, n_parts_hint=None, seed=0)
    for k in (4, 8, 16, 32):
        nn, r, c, v = laplacian_3d7(k, k, k)
        yield dict(name=f"grid3d {k}^3", n=nn, rows=r, cols=c, vals=v, tau=8, profile=sp,
                   assignment=None, n_parts_hint=None, seed=0)
