"""Row-sharded EHYB SpMV and CG over several B200s of one node
(SURVEY.md §8e).

The reordered row space is partition-major, so rank g owns a contiguous
block of partitions [p0, p1): a contiguous slice of x, y and of the ELL slab
(format.py:176-177, 362). The ELL phase needs only owned x (inner entries
reference their own partition's window). Owned ER rows reference remote
columns; the halo plan lists them per peer once, and every SpMV exchanges
exactly those values with one NCCL all-to-all that overlaps the ELL launch:

    pack (gather kernel) -> all_to_all_single (async)  ||  local launch
                         -> wait -> halo launch

The local launch runs ELL and every ER row whose columns are all owned; the
halo launch only the ER rows that read a halo column (and long rows).

`x_ext = [owned x (local_rows) | halo (n_halo)]`; the derived ER columns of
the shard are remapped into that space at upload (ehyb_dev_create_shard).
One process per GPU; `torch.distributed` supplies the communicator (NCCL on
GPUs, gloo for the CPU tests of the host logic).
"""

from __future__ import annotations

import ctypes as C
import os
import sys
import time
import weakref
from dataclasses import dataclass

import numpy as np

from . import _lib as L
from .format import EhybMatrix, host_view


def part_range(n_parts: int, world: int, rank: int):
    """Balanced contiguous partition block of `rank`."""
    base, extra = divmod(n_parts, world)
    p0 = rank * base + min(rank, extra)
    return p0, p0 + base + (1 if rank < extra else 0)


def er_pad_column(e: EhybMatrix) -> int:
    """The column the reference's ER padding slots hold (global column 0,
    format.py:379-380; moved by renumber_partitions), or -1 without ER
    padding. Rows with padding multiply x at this column once (0*x[col])."""
    warp = e.params.warp_size
    w = np.asarray(e.er_row_widths, np.int64)
    if w.size == 0:
        return -1
    sw = np.asarray(e.width_er, np.int64)[np.arange(w.size) // warp]
    j = np.flatnonzero(w < sw)
    if j.size == 0:
        return -1
    j = int(j[0])
    return int(e.col_er[int(e.position_er[j // warp]) + j % warp + warp * int(w[j])])


def halo_columns(e: EhybMatrix, p0: int, p1: int) -> np.ndarray:
    """Sorted distinct global (new-order) columns outside [p0*vec, p1*vec)
    referenced by the real entries of the ER rows that [p0, p1) owns, plus
    the ER padding column when an owned row has padding slots and another
    rank owns that column (the reference's 0*x[0] products, SURVEY.md 8a
    gotcha 4: reproduced after the exchange, so shard y is byte-identical
    for every x, NaN/inf included)."""
    vec = e.params.vec_cache_size
    warp = e.params.warp_size
    lo, hi = p0 * vec, p1 * vec
    y_idx = np.asarray(e.plan.y_idx_er, np.int64)
    slots = np.flatnonzero((y_idx >= lo) & (y_idx < hi))
    if slots.size == 0:
        return np.zeros(0, np.int64)
    w = np.asarray(e.er_row_widths, np.int64)[slots]
    owner = np.repeat(slots, w)
    start = np.cumsum(w) - w
    k = np.arange(owner.size, dtype=np.int64) - np.repeat(start, w)
    pos = np.asarray(e.position_er, np.int64)[owner // warp] + owner % warp + k * warp
    cols = np.asarray(e.col_er, np.int64)[pos]
    cols = cols[(cols < lo) | (cols >= hi)]
    pad = er_pad_column(e)
    if pad >= 0 and not (lo <= pad < hi):
        if np.any(w < np.asarray(e.width_er, np.int64)[slots // warp]):
            cols = np.append(cols, pad)
    return np.unique(cols)


def partition_quotient(e: EhybMatrix) -> np.ndarray:
    """Dense n_parts x n_parts weights: ER entries of a row owned by partition
    p that read a column of partition q (the traffic a p/q split would move)."""
    vec, warp = e.params.vec_cache_size, e.params.warp_size
    n_parts = e.n_parts
    w = np.asarray(e.er_row_widths, np.int64)
    slots = np.repeat(np.arange(w.size, dtype=np.int64), w)
    k = np.arange(slots.size, dtype=np.int64) - np.repeat(np.cumsum(w) - w, w)
    pos = np.asarray(e.position_er, np.int64)[slots // warp] + slots % warp + k * warp
    src = np.asarray(e.plan.y_idx_er, np.int64)[slots] // vec
    dst = np.asarray(e.col_er, np.int64)[pos] // vec
    q = np.zeros((n_parts, n_parts), np.int64)
    np.add.at(q, (src, dst), 1)
    return q


def group_partitions(e: EhybMatrix, world: int) -> np.ndarray:
    """Partition order whose contiguous `part_range` blocks are compact in the
    partition quotient graph: greedy graph growing — each
    group starts from the unassigned partition with the least weight to other
    unassigned ones and repeatedly takes the unassigned partition it is most
    connected to (ties: lowest id). BFS partition ids are not spatially
    ordered, so contiguous id blocks would make most ER rows halo rows."""
    n_parts = e.n_parts
    if world <= 1 or n_parts <= world:
        return np.arange(n_parts, dtype=np.int64)
    q = partition_quotient(e)
    wsym = q + q.T
    np.fill_diagonal(wsym, 0)
    free = np.ones(n_parts, bool)
    order = []
    for g in range(world):
        p0, p1 = part_range(n_parts, world, g)
        size = p1 - p0
        deg = np.where(free, (wsym * free[None, :]).sum(1), np.iinfo(np.int64).max)
        seed = int(np.argmin(deg))
        conn = np.zeros(n_parts, np.int64)
        for _ in range(size):
            free[seed] = False
            order.append(seed)
            conn += wsym[seed]
            if not free.any():
                break
            cand = np.where(free, conn, -1)
            seed = int(np.argmax(cand))
    return np.asarray(order, np.int64)


def renumber_partitions(e: EhybMatrix, order: np.ndarray) -> EhybMatrix:
    """The same matrix with partitions renumbered (new partition i = old
    partition order[i]): row r of old partition p becomes row
    new(p)*vec + r%vec. Every row keeps its entries, k order and slicing, so
    products are bitwise those of `e` under the block permutation; a derived
    device-side layout for sharding, not a parity object."""
    from .format import ReorderPlan

    vec, warp = e.params.vec_cache_size, e.params.warp_size
    n_parts = e.n_parts
    order = np.asarray(order, np.int64)
    if sorted(order.tolist()) != list(range(n_parts)):
        raise ValueError("order must be a permutation of the partitions")
    new_of_old = np.empty(n_parts, np.int64)
    new_of_old[order] = np.arange(n_parts)

    def rowmap(r):
        r = np.asarray(r, np.int64)
        return new_of_old[r // vec] * vec + r % vec

    padded = e.padded_dimension
    reorder = rowmap(e.plan.reorder_table)
    inverse = np.empty_like(e.plan.inverse_table)
    inverse[rowmap(np.arange(padded))] = e.plan.inverse_table
    spp = vec // warp  # slices per partition
    pos = np.asarray(e.position_ell, np.int64)
    width = np.asarray(e.width_ell).reshape(n_parts, spp)[order].ravel()
    seg_lo, seg_hi = pos[order * spp], pos[(order + 1) * spp]
    take = np.concatenate([np.arange(a, b) for a, b in zip(seg_lo, seg_hi)]) if pos[-1] else         np.zeros(0, np.int64)
    position = np.zeros(width.size + 1, np.int64)
    np.cumsum(np.asarray(width, np.int64) * warp, out=position[1:])
    position = position.astype(np.int32)
    plan = ReorderPlan(reorder_table=reorder, inverse_table=inverse,
                       arrange_table=e.plan.arrange_table, y_idx_er=rowmap(e.plan.y_idx_er),
                       n_er_rows=e.plan.n_er_rows, dimension=e.dimension, padded_dimension=padded)
    return EhybMatrix(
        params=e.params, plan=plan, dimension=e.dimension, padded_dimension=padded,
        val_ell=e.val_ell[take], col_ell=e.col_ell[take], position_ell=position,
        width_ell=np.asarray(width, np.int32), part_boundary=e.part_boundary,
        ell_row_widths=np.asarray(e.ell_row_widths).reshape(n_parts, vec)[order].ravel(),
        val_er=e.val_er, col_er=rowmap(e.col_er).astype(np.uint32), position_er=e.position_er,
        width_er=e.width_er, er_row_widths=e.er_row_widths)


@dataclass(eq=False)  # identity hash: plans key the device index-tensor cache
class HaloPlan:
    rank: int
    world: int
    p0: int
    p1: int
    vec: int
    local_rows: int
    halo_cols: np.ndarray      # global columns of the halo slots (ascending)
    recv_splits: list          # halo values received from each peer
    send_splits: list          # values sent to each peer
    send_idx: np.ndarray       # local row offsets gathered into the send buffer

    @property
    def n_halo(self) -> int:
        return int(self.halo_cols.size)


def _comm_device(group):
    import torch.distributed as dist

    backend = dist.get_backend(group)
    if backend == "nccl":
        import torch

        return f"cuda:{torch.cuda.current_device()}"
    return "cpu"


def plan_for(e: EhybMatrix, rank: int, world: int) -> HaloPlan:
    """Halo plan of `rank`, computed locally: every rank holds the assembled
    matrix, so what peer q must send to rank g is g's halo restricted to q's
    rows, in g's (ascending) halo order."""
    vec = e.params.vec_cache_size
    ranges = [part_range(e.n_parts, world, q) for q in range(world)]
    starts = np.array([r[0] * vec for r in ranges], np.int64)
    p0, p1 = ranges[rank]
    halo = halo_columns(e, p0, p1)
    owner = np.searchsorted(starts, halo, side="right") - 1
    recv_splits = np.bincount(owner, minlength=world).astype(np.int64)
    send_parts, send_splits = [], []
    for q in range(world):
        if q == rank:
            send_splits.append(0)
            continue
        hq = halo_columns(e, *ranges[q])
        mine = hq[(hq >= p0 * vec) & (hq < p1 * vec)]
        send_parts.append(mine - p0 * vec)
        send_splits.append(int(mine.size))
    send_idx = np.concatenate(send_parts) if send_parts else np.zeros(0, np.int64)
    return HaloPlan(rank=rank, world=world, p0=p0, p1=p1, vec=vec, local_rows=(p1 - p0) * vec,
                    halo_cols=halo, recv_splits=recv_splits.tolist(), send_splits=send_splits,
                    send_idx=send_idx.astype(np.int64))


def build_halo_plan(e: EhybMatrix, group=None) -> HaloPlan:
    """This rank's halo plan; one all-to-all of counts cross-checks that every
    peer agrees on what it sends (plans are computed locally)."""
    import torch
    import torch.distributed as dist

    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    plan = plan_for(e, rank, world)
    dev = _comm_device(group)
    rs = torch.tensor(plan.recv_splits, dtype=torch.int64, device=dev)
    ss = torch.empty_like(rs)
    dist.all_to_all_single(ss, rs, group=group)
    if ss.cpu().tolist() != plan.send_splits:
        raise RuntimeError("halo plans disagree between ranks")
    return plan


def halo_exchange(x_ext, plan: HaloPlan, group=None, send_buf=None, async_op=False):
    """Fill x_ext[local_rows:] with the halo values owned by the peers.
    CPU tensors (gloo) gather with indexing; CUDA tensors use the gather
    kernel. Returns the collective's work handle when async_op."""
    import torch
    import torch.distributed as dist

    n_send = int(sum(plan.send_splits))
    if x_ext.is_cuda:
        if send_buf is None:
            send_buf = torch.empty(n_send, dtype=x_ext.dtype, device=x_ext.device)
        idx = _idx_tensor(plan, x_ext.device)
        tau = 4 if x_ext.dtype == torch.float32 else 8
        L.call("ehyb_dev_gather", C.c_void_p(x_ext.data_ptr()), C.c_void_p(idx.data_ptr()),
               n_send, C.c_void_p(send_buf.data_ptr()), tau,
               C.c_void_p(torch.cuda.current_stream(x_ext.device).cuda_stream))
    else:
        send_buf = x_ext[torch.from_numpy(plan.send_idx)]
    recv = x_ext[plan.local_rows: plan.local_rows + plan.n_halo]
    if x_ext.is_cuda and dist.get_backend(group) != "nccl":
        # gloo has no CUDA all-to-all: stage through host memory (test path)
        recv_h = torch.empty(recv.numel(), dtype=recv.dtype)
        dist.all_to_all_single(recv_h, send_buf.cpu(), plan.recv_splits, plan.send_splits,
                               group=group)
        recv.copy_(recv_h)
        return _Done() if async_op else None
    return dist.all_to_all_single(recv, send_buf, plan.recv_splits, plan.send_splits,
                                  group=group, async_op=async_op)


class _Done:
    def wait(self):
        return True


_idx_cache: "weakref.WeakKeyDictionary" = weakref.WeakKeyDictionary()


def _idx_tensor(plan: HaloPlan, device):
    import torch

    t = _idx_cache.get(plan)
    if t is None or t.device != device:
        t = torch.from_numpy(plan.send_idx).to(device)
        _idx_cache[plan] = t
    return t


class DistributedEhyb:
    """This rank's shard of a globally assembled EhybMatrix on its GPU."""

    def __init__(self, e: EhybMatrix, group=None, device: int | None = None,
                 plan: HaloPlan | None = None, exchange: str = "nccl"):
        """exchange "nccl": pack + NCCL all-to-all overlapped with the local
        launch, then the halo launch. exchange "p2p": the halo is pulled from
        the peers' x buffers over peer memory (CUDA IPC / NVLink) inside ONE
        fused launch per SpMV — no NCCL, no pack kernel, no second launch;
        x lives in a handle-owned, peer-mapped buffer (`ext_buffer()`)."""
        import torch

        if exchange not in ("nccl", "p2p"):
            raise ValueError("exchange must be 'nccl' or 'p2p'")
        self.exchange = exchange
        self.group = group
        self.device = torch.cuda.current_device() if device is None else int(device)
        self.plan = build_halo_plan(e, group) if plan is None else plan
        self.plan_n_parts = e.n_parts
        self.tau = e.params.tau
        self.dtype = torch.float32 if self.tau == 4 else torch.float64
        self.nnz_local = int(e.ell_row_widths[self.plan.p0 * self.plan.vec:
                                              self.plan.p1 * self.plan.vec].sum())
        y_idx = np.asarray(e.plan.y_idx_er, np.int64)
        lo, hi = self.plan.p0 * self.plan.vec, self.plan.p1 * self.plan.vec
        self.nnz_local += int(np.asarray(e.er_row_widths)[(y_idx >= lo) & (y_idx < hi)].sum())
        hv, keep = host_view(e)
        halo = np.ascontiguousarray(self.plan.halo_cols, np.int64)
        sp = L.ShardPlan(p0=self.plan.p0, p1=self.plan.p1, n_halo=halo.size,
                         halo_cols=L.ptr(halo, L.i64p))
        h = L.vp()
        L.call("ehyb_dev_create_shard", C.byref(hv), C.byref(sp), self.device, C.byref(h))
        del keep
        self._h = h
        self._finalizer = weakref.finalize(self, L.lib().ehyb_dev_destroy, h)
        self.local_rows = self.plan.local_rows
        self.n_ext = self.plan.local_rows + self.plan.n_halo
        self._send = torch.empty(max(1, int(sum(self.plan.send_splits))), dtype=self.dtype,
                                 device=f"cuda:{self.device}")
        self._x_p2p = None
        if exchange == "p2p":
            self._setup_p2p()

    def _setup_p2p(self):
        """IPC handles of the handle-owned x_ext and flag block go to every
        rank; each rank maps its peers' and hands the pull plan (source rank
        and offset of every halo slot) to the device handle."""
        import torch
        import torch.distributed as dist

        xp, fp = C.c_void_p(), C.c_void_p()
        L.call("ehyb_dev_p2p_alloc", self._h, C.byref(xp), C.byref(fp))

        class _Buf:  # zero-copy torch view of the handle-owned x_ext
            def __init__(self, ptr, n, typestr):
                self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr,
                                                 "data": (ptr, False), "version": 3,
                                                 "strides": None}

        self._x_p2p = torch.as_tensor(
            _Buf(xp.value, self.n_ext, "<f4" if self.tau == 4 else "<f8"),
            device=f"cuda:{self.device}")

        def handle(ptr):
            buf = (C.c_char * 64)()
            L.call("ehyb_ipc_handle", C.c_void_p(ptr), buf)
            return bytes(buf)

        mine = (handle(xp.value), handle(fp.value))
        world, rank = self.plan.world, self.plan.rank
        allh = [None] * world
        dist.all_gather_object(allh, mine, group=self.group)
        self._peer_ptrs = []
        px = (C.c_void_p * world)()
        pf = (C.c_void_p * world)()
        for q in range(world):
            if q == rank:
                continue
            for arr, hb in ((px, allh[q][0]), (pf, allh[q][1])):
                ptr = C.c_void_p()
                L.call("ehyb_ipc_open", C.create_string_buffer(hb, 64), self.device,
                       C.byref(ptr))
                arr[q] = ptr.value
                self._peer_ptrs.append(ptr.value)
        vec = self.plan.vec
        ranges = [part_range(self.plan_n_parts, world, q) for q in range(world)]
        starts = np.array([r0 * vec for r0, _ in ranges], np.int64)
        halo = np.asarray(self.plan.halo_cols, np.int64)
        src = (np.searchsorted(starts, halo, side="right") - 1).astype(np.int32)
        off = (halo - starts[src]).astype(np.int64)
        L.call("ehyb_dev_p2p_setup", self._h, world, rank, px, pf, C.c_void_p(src.ctypes.data),
               C.c_void_p(off.ctypes.data), int(sum(self.plan.send_splits)))
        self._p2p_keep = (src, off)
        lib = L.lib()
        self._p2p_finalizer = weakref.finalize(
            self, lambda ptrs: [lib.ehyb_ipc_close(C.c_void_p(p)) for p in ptrs],
            list(self._peer_ptrs))

    def info(self) -> dict:
        """ehyb_dev_info of this rank's handle (grid, work units, split, ...)."""
        out = L.DevInfo()
        L.call("ehyb_dev_info_get", self._h, C.byref(out))
        return {f: getattr(out, f) for f, _ in L.DevInfo._fields_}

    def new_ext(self):
        """A fresh zeroed x in the [owned | halo] layout the SpMV reads."""
        import torch

        return torch.zeros(self.n_ext, dtype=self.dtype, device=f"cuda:{self.device}")

    def ext_buffer(self):
        """The x_ext the SpMV reads without a copy. p2p: the handle-owned,
        peer-mapped buffer (one per handle: write the owned part, the halo
        part is pulled by the kernel; spmv on any other x_ext first copies its
        owned part here). NCCL: a fresh buffer like new_ext()."""
        if self._x_p2p is not None:
            return self._x_p2p
        return self.new_ext()

    def spmv_local(self, x_ext, y_local, *, fma: bool = False, exact: bool = False):
        """Both phases on an x_ext whose halo is already filled (no exchange)."""
        import torch

        mode = L.mode(fma, exact)
        st = C.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)
        xp, yp = C.c_void_p(x_ext.data_ptr()), C.c_void_p(y_local.data_ptr())
        L.call("ehyb_dev_spmv_ell", self._h, xp, yp, mode, st)
        L.call("ehyb_dev_spmv_er", self._h, xp, yp, mode, st)
        return y_local

    def spmv(self, x_ext, y_local, *, fma: bool = False, exact: bool = False,
             overlap: bool = True):
        """y_local = A[owned rows, :] x. x_ext[:local_rows] holds the owned x;
        the halo part is exchanged here, overlapped with the ELL phase."""
        import torch

        mode = L.mode(fma, exact)
        st = C.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)
        if self._x_p2p is not None:
            # one fused launch: ELL, local ER, halo pull from peer memory, halo rows
            if x_ext.data_ptr() != self._x_p2p.data_ptr():
                self._x_p2p[: self.local_rows].copy_(x_ext[: self.local_rows])
            L.call("ehyb_dev_spmv_p2p", self._h, C.c_void_p(y_local.data_ptr()), mode, st)
            return y_local
        xp, yp = C.c_void_p(x_ext.data_ptr()), C.c_void_p(y_local.data_ptr())
        if self.plan.world == 1:
            L.call("ehyb_dev_spmv", self._h, xp, yp, mode, st)
            return y_local
        work = halo_exchange(x_ext, self.plan, self.group, send_buf=self._send[: int(sum(
            self.plan.send_splits))], async_op=True)
        if overlap:
            L.call("ehyb_dev_spmv_ell", self._h, xp, yp, mode, st)
            work.wait()
        else:
            work.wait()
            L.call("ehyb_dev_spmv_ell", self._h, xp, yp, mode, st)
        L.call("ehyb_dev_spmv_er", self._h, xp, yp, mode, st)
        return y_local


    def spmv_host(self, x_local, y_local, *, fma: bool = False, exact: bool = False):
        """Host arrays in and out (pinned for the full PCIe rate): copy the
        owned x slice in, exchange the halo, multiply, copy the owned y out,
        synchronise — the end-to-end call of one rank."""
        import torch

        if not hasattr(self, "_x_ext"):
            self._x_ext = self.ext_buffer()
            self._y_loc = torch.empty(self.local_rows, dtype=self.dtype,
                                      device=f"cuda:{self.device}")
        self._x_ext[: self.local_rows].copy_(torch.as_tensor(x_local), non_blocking=True)
        self.spmv(self._x_ext, self._y_loc, fma=fma, exact=exact)
        out = torch.as_tensor(y_local)
        out.copy_(self._y_loc, non_blocking=True)
        torch.cuda.current_stream(self.device).synchronize()
        return y_local


def dot(a, b, out, n: int):
    """Local fp64 dot product of the first n entries into out (device)."""
    import torch

    tau = 4 if a.dtype == torch.float32 else 8
    L.call("ehyb_dev_dot", C.c_void_p(a.data_ptr()), C.c_void_p(b.data_ptr()), int(n), tau,
           C.c_void_p(out.data_ptr()),
           C.c_void_p(torch.cuda.current_stream(a.device).cuda_stream))


def cg(A: DistributedEhyb, b_local, maxiter: int = 100, tol: float = 0.0,
       method: str = "chronopoulos-gear"):
    """Conjugate gradients on the sharded operator, every vector and scalar on
    the device. method "chronopoulos-gear" (default): one SpMV and ONE fused
    all-reduce of two fp64 scalars per iteration; "classic": textbook CG with
    two all-reduces. Returns (x_local, info)."""
    if method == "chronopoulos-gear":
        return _cg_cg(A, b_local, maxiter, tol)
    if method != "classic":
        raise ValueError("method must be 'chronopoulos-gear' or 'classic'")
    import torch
    import torch.distributed as dist

    dev = f"cuda:{A.device}"
    n = A.local_rows
    st = C.c_void_p(torch.cuda.current_stream(A.device).cuda_stream)
    tau = A.tau
    x = torch.zeros(n, dtype=A.dtype, device=dev)
    r = b_local.clone()
    p = A.ext_buffer()
    p[:n].copy_(r)
    q = torch.empty(n, dtype=A.dtype, device=dev)
    sc = torch.zeros(4, dtype=torch.float64, device=dev)  # rr, pq, rr_new, |b|^2
    dot(r, r, sc[0:1], n)
    if A.plan.world > 1:
        dist.all_reduce(sc[0:1], group=A.group)
    sc[3] = sc[0]
    its = 0
    for its in range(1, maxiter + 1):
        A.spmv(p, q)
        dot(p, q, sc[1:2], n)
        if A.plan.world > 1:
            dist.all_reduce(sc[1:2], group=A.group)
        L.call("ehyb_dev_cg_xr", C.c_void_p(x.data_ptr()), C.c_void_p(r.data_ptr()),
               C.c_void_p(p.data_ptr()), C.c_void_p(q.data_ptr()), C.c_void_p(sc[0:1].data_ptr()),
               C.c_void_p(sc[1:2].data_ptr()), n, tau, C.c_void_p(sc[2:3].data_ptr()), st)
        if A.plan.world > 1:
            dist.all_reduce(sc[2:3], group=A.group)
        L.call("ehyb_dev_cg_p", C.c_void_p(p.data_ptr()), C.c_void_p(r.data_ptr()),
               C.c_void_p(sc[2:3].data_ptr()), C.c_void_p(sc[0:1].data_ptr()), n, tau, st)
        sc[0:1].copy_(sc[2:3])
        if tol > 0 and its % 10 == 0:
            if float(sc[0]) <= tol * tol * float(sc[3]):
                break
    info = {"iterations": its, "method": "classic",
            "rel_residual": float(np.sqrt(float(sc[0]) / max(float(sc[3]), 1e-300)))}
    return x, info


def _cg_cg(A: DistributedEhyb, b_local, maxiter: int, tol: float):
    """Chronopoulos-Gear CG (s-step 1): w = A r, (gamma, delta) = ((r,r),
    (w,r)) in one pass and one all-reduce; beta = gamma/gamma_old, alpha =
    gamma/(delta - beta*gamma/alpha_old); p = r + beta p, s = w + beta s,
    x += alpha p, r -= alpha s (one fused kernel, scalars on the device)."""
    import torch
    import torch.distributed as dist

    dev = f"cuda:{A.device}"
    n = A.local_rows
    st = C.c_void_p(torch.cuda.current_stream(A.device).cuda_stream)
    tau = A.tau
    x = torch.zeros(n, dtype=A.dtype, device=dev)
    r = A.ext_buffer()  # r lives in the [owned | halo] layout the SpMV reads
    r[:n].copy_(b_local)
    p = torch.zeros(n, dtype=A.dtype, device=dev)
    s = torch.zeros(n, dtype=A.dtype, device=dev)
    w = torch.empty(n, dtype=A.dtype, device=dev)
    sc = torch.zeros(8, dtype=torch.float64, device=dev)  # gamma, delta, gamma_old, alpha, beta
    multi = A.plan.world > 1

    def ptr(t):
        return C.c_void_p(t.data_ptr())

    def reduce_gamma_delta():
        A.spmv(r, w)
        L.call("ehyb_dev_dot2", ptr(r), ptr(r), ptr(w), ptr(r), n, tau, ptr(sc), st)
        if multi:
            dist.all_reduce(sc[0:2], group=A.group)

    reduce_gamma_delta()
    bb = float(sc[0])
    its = 0
    for its in range(1, maxiter + 1):
        L.call("ehyb_dev_cgcg_step", ptr(x), ptr(r), ptr(p), ptr(s), ptr(w), ptr(sc),
               1 if its == 1 else 0, n, tau, st)
        reduce_gamma_delta()
        if tol > 0 and its % 10 == 0:
            if float(sc[0]) <= tol * tol * bb:
                break
    info = {"iterations": its, "method": "chronopoulos-gear",
            "rel_residual": float(np.sqrt(float(sc[0]) / max(bb, 1e-300)))}
    return x, info


# --------------------------------------------------------------------------
# multi-GPU bench (bench.py --gpus N under torchrun)
# --------------------------------------------------------------------------

def weak_config(world: int):
    """N-GPU weak-scaling workload: 27-point stencil 128 x 128 x (128*N),
    random symmetric permutation (seed 1), fp64, P = 148*N partitions.
    N = 1 is exactly cfg2; N = 8 has cfg5's 16.7M rows."""
    from . import workloads as W

    return W.permute_symmetric(*W.stencil27(128 * world, 128, 128), seed=1)


def dist_workload(name: str, world: int):
    """The multi-rank bench workload: (n, rows, cols, vals, tau, profile, desc).
    A named config (default cfg5, BASELINE configs[4]) keeps its 1-GPU
    profile at every GPU count, so every N streams the same structure and
    bytes (SURVEY.md 8e option (i)); ranks that own fewer partitions than
    SMs split them into work units. "weak": the 128*N x 128 x 128 permuted
    stencil with P = 148*N (N = 1 is cfg2)."""
    from . import workloads as W
    from .format import DeviceProfile, b200_profile

    if name == "weak":
        n, r, c, v = weak_config(world)
        return (n, r, c, v, 8, b200_profile(world),
                f"27-point stencil {128 * world}x128x128, random symmetric permutation, "
                f"P=148x{world} (weak scaling; N=1: cfg2)")
    if name not in W.CONFIGS:
        raise ValueError(f"unknown config {name!r}")
    n, r, c, v, tau = W.build_config(name)
    prof = W.CONFIG_PROFILES.get(name)
    return (n, r, c, v, tau, DeviceProfile(*prof) if prof else b200_profile(1),
            f"{name}: {W.CONFIGS[name][0]}")


def single_gpu_reference(e, device: int, args):
    """The same matrix on this one GPU (rank 0, before sharding): the T_1 of
    the strong-scaling run, CUDA-event time per SpMV."""
    import torch

    from .device import DeviceMatrix
    from .format import permute_vector
    from . import workloads as W

    dm = DeviceMatrix(e, device)
    xr = torch.from_numpy(permute_vector(W.deterministic_vector(e.dimension, 0), e.plan)).to(
        f"cuda:{device}", dm.torch_dtype)
    y = torch.empty_like(xr)
    for _ in range(max(3, args.warmup)):
        dm.spmv(xr, y)
    torch.cuda.synchronize()
    k = max(10, min(args.steps, 100))
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(k):
        dm.spmv(xr, y)
    b.record()
    b.synchronize()
    t = a.elapsed_time(b) / 1e3 / k
    out = {"ms_per_step": t * 1e3, "value": 2 * e.nnz / t / 1e9, "unit": "GFLOP/s",
           "ctas": dm.info()["ctas"], "how": "the same assembled matrix on rank 0's GPU alone "
                                             "(T_1 of this strong-scaling run)"}
    dm.close()
    del xr, y
    torch.cuda.empty_cache()
    return out


def measured_hbm_peak():
    """MEASURED_PEAKS.json hbm_gbs (driver-written), else the B200 recipe's
    fallback."""
    import json

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    try:
        with open(os.path.join(root, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:  # noqa: BLE001 - absent on a fresh box
        return 6650.0, "fallback (B200_PROFILING.md)"


def bench_main(args, clock_cls=None):
    import json

    import torch
    import torch.distributed as dist

    from . import engine
    from .format import b200_profile, build_ehyb
    from .matrix_io import CooMatrix, read_ehyb_container, write_ehyb_container

    for k, v in (("MASTER_ADDR", "127.0.0.1"), ("MASTER_PORT", "29517"), ("RANK", "0"),
                 ("WORLD_SIZE", "1")):
        os.environ.setdefault(k, v)  # allow a single-process run without torchrun
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    # EHYB_DIST_BACKEND=gloo: a functional check of the multi-rank flow with
    # several ranks sharing one GPU (NCCL needs one GPU per rank)
    backend = os.environ.get("EHYB_DIST_BACKEND", "nccl")
    local = int(os.environ.get("LOCAL_RANK", str(rank))) % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    # the driver parses one JSON line from stdout: keep NCCL's banner off it
    if os.environ.get("NCCL_DEBUG", "").upper() in ("", "VERSION"):
        os.environ["NCCL_DEBUG"] = "WARN"
    sys.stdout.flush()
    saved = os.dup(1)
    os.dup2(2, 1)
    try:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
        else:
            dist.init_process_group(backend)
        dist.barrier()
    finally:
        sys.stdout.flush()
        os.dup2(saved, 1)
        os.close(saved)
    name = getattr(args, "config", None) or "cfg5"
    path = os.path.join(os.environ.get("EHYB_SCRATCH", "/tmp"), f"ehyb_{name}_{world}.ehyb")
    t0 = time.perf_counter()
    nnz = None
    single = None
    if rank == 0:
        n, r, c, v, tau, prof, desc = dist_workload(name, world)
        m = CooMatrix(n, n, r, c, v)
        nnz = m.nnz
        del r, c, v
        from .gpu_prep import build_ehyb_gpu

        e = build_ehyb_gpu(m, tau=tau, profile=prof, device=local)
        del m
        if world > 1 and name != "weak":
            single = single_gpu_reference(e, local, args)
        # contiguous rank blocks of a quotient-graph ordering of the partitions
        e = renumber_partitions(e, group_partitions(e, world))
        write_ehyb_container(e, path)
    else:
        desc = None
    obj = [nnz, desc]
    dist.broadcast_object_list(obj, src=0)
    nnz, desc = obj
    dist.barrier()
    if rank != 0:
        e = read_ehyb_container(path)
    t_prep = time.perf_counter() - t0
    # exchange: the fused peer-memory pull (one launch per SpMV) by default at
    # N > 1, NCCL if any rank cannot map its peers (decided collectively)
    exchange = os.environ.get("EHYB_EXCHANGE", "p2p" if world > 1 else "nccl")
    A = None
    if exchange == "p2p":
        ok = torch.ones(1, dtype=torch.int64,
                        device=f"cuda:{local}" if backend == "nccl" else "cpu")
        try:
            A = DistributedEhyb(e, device=local, exchange="p2p")
        except Exception as ex:  # noqa: BLE001 - reported, then the NCCL path
            print(f"p2p exchange unavailable on rank {rank}: {ex}", file=sys.stderr)
            ok.zero_()
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        if int(ok) == 0:
            A, exchange = None, "nccl"
    if A is None:
        A = DistributedEhyb(e, device=local)
    # the other exchange, timed beside it (N > 1)
    A_nccl = DistributedEhyb(e, device=local) if (exchange == "p2p" and world > 1) else None
    bmin_total = engine.min_bytes(e)
    n_parts = e.n_parts
    info0 = A.info()
    peak, peak_src = measured_hbm_peak()
    e_full = e if rank == 0 else None  # the single-GPU product checks the sharded one
    from . import workloads as W

    xg = W.deterministic_vector(e.dimension, 0)
    from .format import permute_vector

    xr = permute_vector(xg, e.plan)
    lo, hi = A.plan.p0 * A.plan.vec, A.plan.p1 * A.plan.vec
    x_ext = A.ext_buffer()
    x_ext[: A.local_rows].copy_(torch.from_numpy(xr[lo:hi]))
    y = torch.empty(A.local_rows, dtype=A.dtype, device=x_ext.device)
    del e
    for _ in range(args.warmup):
        A.spmv(x_ext, y)
    torch.cuda.synchronize()
    dist.barrier()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    clocks = None
    if rank == 0 and clock_cls is not None:
        clocks = clock_cls(local)
        clocks.__enter__()
    ev0.record()
    for _ in range(args.steps):
        A.spmv(x_ext, y)
    ev1.record()
    ev1.synchronize()

    torch.cuda.synchronize()
    dist.barrier()
    t = torch.tensor([ev0.elapsed_time(ev1) / 1e3 / args.steps], dtype=torch.float64,
                     device=x_ext.device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    t_step = float(t)
    t_nccl = None
    if A_nccl is not None:
        xn = A_nccl.new_ext()
        xn[: A_nccl.local_rows].copy_(torch.from_numpy(xr[lo:hi]))
        yn = torch.empty_like(y)
        for _ in range(args.warmup):
            A_nccl.spmv(xn, yn)
        torch.cuda.synchronize()
        dist.barrier()
        ev0.record()
        for _ in range(args.steps):
            A_nccl.spmv(xn, yn)
        ev1.record()
        ev1.synchronize()
        tn = torch.tensor([ev0.elapsed_time(ev1) / 1e3 / args.steps], dtype=torch.float64,
                          device=x_ext.device)
        dist.all_reduce(tn, op=dist.ReduceOp.MAX)
        t_nccl = float(tn)
        del A_nccl, xn, yn
    # end to end: per step the owned x slice H2D (pinned), exchange + product,
    # owned y slice D2H, synchronised; max over ranks
    x_pin = torch.from_numpy(np.ascontiguousarray(xr[lo:hi])).pin_memory()
    y_pin = torch.empty(A.local_rows, dtype=A.dtype).pin_memory()
    for _ in range(3):
        A.spmv_host(x_pin, y_pin)
    k_e2e = max(5, min(args.steps, 100))
    dist.barrier()
    te0 = time.perf_counter()
    for _ in range(k_e2e):
        A.spmv_host(x_pin, y_pin)
    te = torch.tensor([(time.perf_counter() - te0) / k_e2e], dtype=torch.float64,
                      device=x_ext.device)
    dist.all_reduce(te, op=dist.ReduceOp.MAX)
    t_e2e = float(te)
    nb = torch.tensor([A.local_rows * A.dtype.itemsize], dtype=torch.int64, device=x_ext.device)
    dist.all_reduce(nb)
    # CG: 100 iterations on b = A*1
    b = torch.empty(A.local_rows, dtype=A.dtype, device=x_ext.device)
    ones = A.new_ext()
    ones[: A.local_rows].fill_(1.0)
    A.spmv(ones, b)
    torch.cuda.synchronize()
    cg_res = {}
    for method in ("chronopoulos-gear", "classic"):
        cg(A, b, maxiter=3, method=method)  # warm-up
        torch.cuda.synchronize()
        dist.barrier()
        c0 = torch.cuda.Event(enable_timing=True)
        c1 = torch.cuda.Event(enable_timing=True)
        tw0 = time.perf_counter()
        c0.record()
        _, info = cg(A, b, maxiter=100, method=method)
        c1.record()
        c1.synchronize()
        tw = time.perf_counter() - tw0
        tc = torch.tensor([c0.elapsed_time(c1) / 1e3, tw], dtype=torch.float64,
                          device=x_ext.device)
        dist.all_reduce(tc, op=dist.ReduceOp.MAX)
        cg_res[method] = {"iterations": info["iterations"],
                          "ms_per_iter": float(tc[0]) / info["iterations"] * 1e3,
                          "wall_ms_per_iter": float(tc[1]) / info["iterations"] * 1e3,
                          "rel_residual": info["rel_residual"],
                          "allreduces_per_iter": 1 if method == "chronopoulos-gear" else 2}
    if clocks is not None:
        clocks.__exit__(None, None, None)
    # parity: the gathered sharded y against one single-GPU launch (rank 0);
    # x_ext is rewritten (p2p: CG used the same handle-owned buffer)
    x_ext[: A.local_rows].copy_(torch.from_numpy(xr[lo:hi]))
    A.spmv(x_ext, y)
    torch.cuda.synchronize()
    parts = [None] * world if rank == 0 else None
    dist.gather_object(y.cpu().numpy(), parts, dst=0)
    parity = None
    if rank == 0:
        from .device import DeviceMatrix

        dm = DeviceMatrix(e_full, local)
        y_one = dm.spmv(torch.from_numpy(xr).to(f"cuda:{local}", dm.torch_dtype)).cpu().numpy()
        y_all = np.concatenate(parts)
        ok = y_all.tobytes() == y_one.tobytes()
        parity = "bitwise == single-GPU product" if ok else "MISMATCH"
        if not ok:
            bad = np.flatnonzero(y_all.view(np.int64) != y_one.view(np.int64))
            print(f"parity: {bad.size} rows differ, first {bad[:8].tolist()}, "
                  f"values {[(float(y_all[i]), float(y_one[i])) for i in bad[:4]]}",
                  file=sys.stderr)
        del dm
    e_full = None
    if rank == 0:
        flops = 2 * nnz
        out = {
            "metric": "SpMV GFLOP/s (2*nnz/t) and achieved HBM GB/s vs peak",
            "value": flops / t_step / 1e9, "unit": "GFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_step * 1e3,
            "higher_is_better": True, "scaling": "weak" if name == "weak" else "strong",
            "vs_baseline": None, "dtype": "f64" if A.tau == 8 else "f32",
            "data": "synthetic",
            "config": {"workload": desc, "n": int(A.plan.vec * n_parts), "nnz": nnz,
                       "n_parts": n_parts, "work_units_rank0": info0["work_units"],
                       "split_rank0": info0["split"], "parallelism": (
                           f"row shards x{world}, halo pulled from peer memory inside one "
                           f"fused launch" if exchange == "p2p" else
                           f"row shards x{world}, NCCL halo all-to-all overlapped with the "
                           f"local launch"),
                       "l2_policy": "inputs larger than L2"},
            "roofline": {"bound": "hbm", "achieved": bmin_total / t_step / 1e9 / world,
                         "peak": peak, "unit": "GB/s (per GPU)", "peak_source": peak_src,
                         "frac": bmin_total / t_step / 1e9 / world / peak, "traffic": None,
                         "algorithmic_bytes_per_step": bmin_total},
            "same_matrix_1gpu": single,
            "e2e": {"value": flops / t_e2e / 1e9, "unit": "GFLOP/s",
                    "h2d_bytes_per_step": int(nb), "d2h_bytes_per_step": int(nb),
                    "ms_per_step": t_e2e * 1e3,
                    "api": "DistributedEhyb.spmv_host per rank: pinned H2D of the owned x "
                           "slice, NCCL halo exchange + fused kernels, D2H of the owned y "
                           "slice, synchronised (max over ranks)"},
            "clocks": clocks.summary() if clocks is not None else None,
            "halo_values_rank0": A.plan.n_halo,
            "parity": parity, "backend": backend, "exchange": exchange,
            "nccl_exchange": None if t_nccl is None else {
                "ms_per_step": t_nccl * 1e3, "value": flops / t_nccl / 1e9,
                "how": "pack kernel + NCCL all_to_all overlapped with the local launch, "
                       "then the halo launch"},
            "cg": cg_res,
            "preprocessing_s": t_prep,
            "gpu_launches": (1 if (world == 1 or exchange == "p2p") else 3) * args.steps,
        }
        print(json.dumps(out), flush=True)
    dist.barrier()
    dist.destroy_process_group()
    return 0
