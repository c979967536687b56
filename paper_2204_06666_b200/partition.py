"""Graph construction and balanced partitioning (reference partition.py).

`build_graph`, `partition_graph` and `rebalance_partition` run natively
(csrc/prep.cpp) and return arrays byte-identical to the reference's; the
dataclasses and error wording are the reference's.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib as L
from .matrix_io import CooMatrix


@dataclass(eq=False)
class AdjacencyGraph:
    """Undirected graph, CSR-like, neighbour lists sorted (partition.py:22-39)."""

    n_vertices: int
    adj_ptr: np.ndarray
    adj: np.ndarray

    def neighbors(self, v: int) -> np.ndarray:
        return self.adj[self.adj_ptr[v]: self.adj_ptr[v + 1]]

    @property
    def degrees(self) -> np.ndarray:
        return np.diff(self.adj_ptr)

    @property
    def n_edges(self) -> int:
        return int(self.adj.size) // 2


@dataclass(eq=False)
class PartitionMap:
    """Vertex -> partition assignment plus part sizes (partition.py:42-67)."""

    n_parts: int
    assignment: np.ndarray
    part_sizes: np.ndarray

    @classmethod
    def from_assignment(cls, assignment, n_parts: int | None = None) -> "PartitionMap":
        assignment = np.asarray(assignment, dtype=np.int64)
        if assignment.ndim != 1:
            raise ValueError("assignment must be one-dimensional")
        if assignment.size and assignment.min() < 0:
            raise ValueError("negative partition id")
        inferred = int(assignment.max()) + 1 if assignment.size else 0
        if n_parts is None:
            n_parts = max(inferred, 1)
        elif inferred > n_parts:
            raise ValueError(f"partition id {inferred - 1} >= n_parts {n_parts}")
        sizes = np.bincount(assignment, minlength=n_parts).astype(np.int64)
        return cls(n_parts=n_parts, assignment=assignment, part_sizes=sizes)

    @property
    def n_vertices(self) -> int:
        return int(self.assignment.size)


@dataclass(frozen=True)
class CutMetrics:
    inner_entries: int
    extra_entries: int
    inner_fraction: float


def build_graph(m: CooMatrix) -> AdjacencyGraph:
    """Symmetrised off-diagonal adjacency (partition.py:77-98), native."""
    if not m.is_square:
        raise ValueError("matrix must be square")
    n = m.n_rows
    rows = L.c_array(m.rows, np.int64)
    cols = L.c_array(m.cols, np.int64)
    adj_ptr = np.zeros(n + 1, dtype=np.int64)
    out = L.i32p()
    n_adj = C.c_int64()
    L.call("ehyb_build_graph", n, rows.size, L.ptr(rows, L.i64p), L.ptr(cols, L.i64p),
           L.ptr(adj_ptr, L.i64p), C.byref(out), C.byref(n_adj))
    return AdjacencyGraph(n_vertices=n, adj_ptr=adj_ptr,
                          adj=L.adopt(out, n_adj.value, np.int32))


def partition_graph(g: AdjacencyGraph, n_parts: int, capacity: int, seed: int = 0) -> PartitionMap:
    """BFS region growing + one refinement pass (partition.py:101-204), native
    and bit-exact, including the CPython MT19937 seed draws."""
    n = g.n_vertices
    if n_parts < 1:
        raise ValueError("n_parts must be >= 1")
    if capacity < 1 or n_parts * capacity < n:
        raise ValueError(
            f"infeasible: {n_parts} parts of capacity {capacity} cannot hold {n} vertices")
    adj_ptr = L.c_array(g.adj_ptr, np.int64)
    adj = L.c_array(g.adj, np.int32)
    assignment = np.empty(n, dtype=np.int64)
    sizes = np.empty(n_parts, dtype=np.int64)
    L.call("ehyb_partition_graph", n, L.ptr(adj_ptr, L.i64p), L.ptr(adj, L.i32p), n_parts,
           capacity, int(seed), L.ptr(assignment, L.i64p), L.ptr(sizes, L.i64p))
    return PartitionMap(n_parts=n_parts, assignment=assignment, part_sizes=sizes)


def random_partition(n_vertices: int, n_parts: int, capacity: int | None = None,
                     seed: int = 0) -> PartitionMap:
    """Seeded balanced random partition (partition.py:207-221); test utility."""
    if n_parts < 1:
        raise ValueError("n_parts must be >= 1")
    max_size = -(-n_vertices // n_parts)
    if capacity is not None and max_size > capacity:
        raise ValueError(f"balanced parts of size {max_size} exceed capacity {capacity}")
    perm = np.random.default_rng(seed).permutation(n_vertices)
    assignment = np.empty(n_vertices, dtype=np.int64)
    for pid, chunk in enumerate(np.array_split(perm, n_parts)):
        assignment[chunk] = pid
    return PartitionMap.from_assignment(assignment, n_parts=n_parts)


def rebalance_partition(g: AdjacencyGraph, parts: PartitionMap, capacity: int) -> PartitionMap:
    """Evict highest-cut boundary vertices from overfull parts
    (partition.py:224-262), native."""
    n_parts = parts.n_parts
    if n_parts * capacity < g.n_vertices:
        raise ValueError("infeasible capacity")
    adj_ptr = L.c_array(g.adj_ptr, np.int64)
    adj = L.c_array(g.adj, np.int32)
    a_in = L.c_array(parts.assignment, np.int64)
    assignment = np.empty(g.n_vertices, dtype=np.int64)
    sizes = np.empty(n_parts, dtype=np.int64)
    L.call("ehyb_rebalance_partition", g.n_vertices, L.ptr(adj_ptr, L.i64p), L.ptr(adj, L.i32p),
           n_parts, capacity, L.ptr(a_in, L.i64p), L.ptr(assignment, L.i64p),
           L.ptr(sizes, L.i64p))
    return PartitionMap(n_parts=n_parts, assignment=assignment, part_sizes=sizes)


def save_partition_file(parts: PartitionMap, sink) -> None:
    """METIS-style interchange: one 0-based id per vertex per line
    (partition.py:280-290); feeds build_ehyb(partition=...)."""
    import os

    text = "\n".join(str(int(p)) for p in parts.assignment) + "\n"
    if isinstance(sink, (str, os.PathLike)):
        with open(sink, "w") as fh:
            fh.write(text)
    else:
        try:
            sink.write(text)
        except TypeError:
            sink.write(text.encode("ascii"))


def load_partition_file(source, n_vertices: int, n_parts: int | None = None) -> PartitionMap:
    """Inverse of save_partition_file with the reference's checks
    (partition.py:293-317)."""
    import os

    if isinstance(source, (str, os.PathLike)):
        with open(source) as fh:
            text = fh.read()
    else:
        text = source.read()
        if isinstance(text, bytes):
            text = text.decode("ascii")
    tokens = text.split()
    if len(tokens) != n_vertices:
        raise ValueError(f"partition file has {len(tokens)} entries, expected {n_vertices}")
    try:
        assignment = np.asarray([int(t) for t in tokens], dtype=np.int64)
    except ValueError:
        raise ValueError("partition file must contain one integer per line") from None
    return PartitionMap.from_assignment(assignment, n_parts=n_parts)


def cut_metrics(m: CooMatrix, parts: PartitionMap) -> CutMetrics:
    """Inner (same-partition) vs extra entries (partition.py:265-277)."""
    if not m.is_square or parts.n_vertices != m.n_rows:
        raise ValueError("dimension mismatch between matrix and partition")
    if m.nnz == 0:
        return CutMetrics(0, 0, 1.0)
    a = parts.assignment
    inner = int(np.count_nonzero(a[m.rows] == a[m.cols]))
    return CutMetrics(inner, m.nnz - inner, inner / m.nnz)
