/*
 * ehyb_b200.h — C ABI of the B200-native EHYB SpMV path (libehyb_b200.so).
 *
 * Drop-in boundary for the reference package `ehyb` 0.1.0
 * (arXiv 2204.06666, /root/reference/pkg/src/ehyb). Each entry point names
 * the reference function it replaces (file:line). The reference is pure
 * Python, so its "FFI" for this path is the Python API itself; the Python
 * shim in paper_2204_06666_b200/ binds these symbols with ctypes and keeps
 * the reference's signatures, dataclasses and error wording
 * (see INTEGRATION.md for the binding a maintainer would add to `ehyb`).
 *
 * Conventions
 *  - Every function returns 0 on success. A nonzero return is an error whose
 *    message (the reference's ValueError wording where one exists) is
 *    available from ehyb_last_error() on the calling thread:
 *      EHYB_EINVAL (1)  -> ValueError in Python
 *      EHYB_ENOMEM (2)  -> MemoryError
 *      EHYB_ECUDA  (3)  -> RuntimeError (CUDA / cuSPARSE failure)
 *  - Plain pointers and sizes only; no caller pointer is retained past the
 *    call except by a device handle, which owns device copies of the matrix
 *    (uploaded once in ehyb_dev_create, freed by ehyb_dev_destroy).
 *  - Arrays the library allocates (marked "lib-alloc") are released with
 *    ehyb_free().
 *  - Device entry points take CUDA device pointers and a cudaStream_t passed
 *    as void*; launches are stream-ordered and never synchronise the host
 *    unless stated.
 *  - A handle keeps per-launch counters on the device (alternating by a
 *    device-side launch epoch, so captured CUDA graphs replay correctly):
 *    launches of one handle must be ordered (one stream, or events between
 *    streams); different handles are independent.
 */
#ifndef EHYB_B200_H
#define EHYB_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define EHYB_API __attribute__((visibility("default")))

#define EHYB_EINVAL 1
#define EHYB_ENOMEM 2
#define EHYB_ECUDA 3

#define EHYB_MAX_LOCAL_INDEX 65536 /* format.py:21 MAX_LOCAL_INDEX */

/* SpMV arithmetic modes */
#define EHYB_MODE_STRICT 0 /* separately rounded mul + add, k ascending: bitwise == reference */
#define EHYB_MODE_FMA 1    /* fused multiply-add; within 1e-12 (fp64) / 1e-5 (fp32) */
#define EHYB_MODE_DEFAULT 2 /* STRICT for every slice row; rows wider than the long-row
                               threshold (EHYB_LONG_ROW, 128 entries) are summed in fixed
                               4096-entry segments (deterministic, reassociated: within
                               1e-12 (fp64) / 1e-5 (fp32)). == STRICT when no row is long */

/* ------------------------------------------------------------ utilities */
EHYB_API const char* ehyb_last_error(void);
EHYB_API int ehyb_abi_version(void); /* bumps on any signature change */
EHYB_API void ehyb_free(void* p);
EHYB_API int ehyb_num_threads(void); /* OpenMP threads used by host preprocessing */

/* ------------------------------------------------- host preprocessing */

/* compute_params (format.py:83-107, Eq.1-2): smallest k with the
 * warp-aligned window vec = align_up(ceil(dimension/(k*procs)), warp)
 * satisfying vec*tau <= shm and vec <= 65536. */
EHYB_API int ehyb_compute_params(int64_t dimension, int32_t tau, int64_t procs, int64_t warp,
                                 int64_t shm, int64_t* out_k, int64_t* out_n_parts,
                                 int64_t* out_vec);

/* build_graph (partition.py:77-98): symmetrised off-diagonal adjacency,
 * sorted duplicate-free neighbour lists. adj_ptr: caller-alloc int64[n+1];
 * *out_adj: lib-alloc int32[*out_n_adj]. */
EHYB_API int ehyb_build_graph(int64_t n, int64_t nnz, const int64_t* rows, const int64_t* cols,
                              int64_t* adj_ptr, int32_t** out_adj, int64_t* out_n_adj);

/* partition_graph (partition.py:101-204): BFS region growing seeded at
 * min-degree vertices (CPython random.Random(seed) tie draws), leftover
 * regions, round-robin isolated vertices, one refinement pass.
 * assignment: caller-alloc int64[n]; sizes: caller-alloc int64[n_parts]. */
EHYB_API int ehyb_partition_graph(int64_t n, const int64_t* adj_ptr, const int32_t* adj,
                                  int64_t n_parts, int64_t capacity, int64_t seed,
                                  int64_t* assignment, int64_t* sizes);

/* rebalance_partition (partition.py:224-262). */
EHYB_API int ehyb_rebalance_partition(int64_t n, const int64_t* adj_ptr, const int32_t* adj,
                                      int64_t n_parts, int64_t capacity,
                                      const int64_t* assignment_in, int64_t* assignment,
                                      int64_t* sizes);

/* classify_rows (format.py:123-137). inner/outer/row_order: caller-alloc
 * int64[n]; *out_er_row_order: lib-alloc int64[*out_n_er]. */
EHYB_API int ehyb_classify_rows(int64_t n, int64_t nnz, const int64_t* rows, const int64_t* cols,
                                const int64_t* assignment, int64_t n_parts, int64_t* inner,
                                int64_t* outer, int64_t* row_order, int64_t** out_er_row_order,
                                int64_t* out_n_er);

/* build_reorder_plan (format.py:161-199). reorder/inverse: int64[n_parts*vec];
 * arrange: int64[n]; y_idx_er: int64[n_er]; all caller-alloc. */
EHYB_API int ehyb_build_reorder_plan(int64_t n, int64_t n_parts, int64_t vec,
                                     const int64_t* assignment, const int64_t* part_sizes,
                                     const int64_t* row_order, const int64_t* er_row_order,
                                     int64_t n_er, int64_t* reorder, int64_t* inverse,
                                     int64_t* arrange, int64_t* y_idx_er);

/* assemble_ehyb (format.py:302-409). Caller-alloc (sizes known up front):
 * position_ell i32[padded/warp+1], width_ell i32[padded/warp],
 * ell_row_widths i32[padded], part_boundary i32[n_parts+1],
 * position_er i32[ceil(n_er/warp)+1], width_er i32[ceil(n_er/warp)],
 * er_row_widths i32[n_er]. Lib-alloc: val_ell (f32|f64)[slots_ell],
 * col_ell u16[slots_ell], val_er (f32|f64)[slots_er], col_er u32[slots_er]. */
EHYB_API int ehyb_assemble(int64_t n, int64_t nnz, const int64_t* rows, const int64_t* cols,
                           const double* values, const int64_t* assignment,
                           const int64_t* reorder, const int64_t* arrange, int64_t n_er,
                           int64_t warp, int64_t vec, int64_t n_parts, int32_t tau,
                           int32_t* position_ell, int32_t* width_ell, int32_t* ell_row_widths,
                           int32_t* part_boundary, int32_t* position_er, int32_t* width_er,
                           int32_t* er_row_widths, void** out_val_ell, uint16_t** out_col_ell,
                           int64_t* out_slots_ell, void** out_val_er, uint32_t** out_col_er,
                           int64_t* out_slots_er);

/* ---------------------------------------------- GPU preprocessing
 * The same results as ehyb_build_graph / ehyb_classify_rows /
 * ehyb_build_reorder_plan / ehyb_assemble (bit-exact), computed on a GPU:
 * the COO is uploaded once (ehyb_gprep_create; entries grouped by row,
 * column and entry index with a stable radix sort), build_graph returns the
 * adjacency like ehyb_build_graph, assemble takes the (host-computed)
 * partition and fills the outputs of the three host calls at once.
 * Caller-alloc: inner/outer/row_order/arrange i64[n], reorder/inverse
 * i64[padded], position_ell i32[padded/warp+1], width_ell i32[padded/warp],
 * ell_row_widths i32[padded], part_boundary i32[n_parts+1]. Lib-alloc
 * (ehyb_free): er_row_order, y_idx_er i64[n_er], position_er i32[n_er_sl+1],
 * width_er i32[n_er_sl], er_row_widths i32[n_er], the four slab arrays. */
typedef struct ehyb_gprep ehyb_gprep;
EHYB_API int ehyb_gprep_create(int64_t n, int64_t nnz, const int64_t* rows, const int64_t* cols,
                               const double* values, int device, ehyb_gprep** out);
EHYB_API int ehyb_gprep_destroy(ehyb_gprep* c);
EHYB_API int ehyb_gprep_build_graph(ehyb_gprep* c, int64_t* adj_ptr, int32_t** out_adj,
                                    int64_t* out_n_adj);
EHYB_API int ehyb_gprep_assemble(ehyb_gprep* c, const int64_t* assignment, int64_t n_parts,
                                 int64_t vec, int64_t warp, int32_t tau,
                                 int64_t* inner, int64_t* outer, int64_t* row_order,
                                 int64_t** out_er_row_order, int64_t* out_n_er,
                                 int64_t* reorder, int64_t* inverse, int64_t* arrange,
                                 int64_t** out_y_idx_er,
                                 int32_t* position_ell, int32_t* width_ell, int32_t* ell_row_widths,
                                 int32_t* part_boundary, int32_t** out_position_er,
                                 int32_t** out_width_er, int32_t** out_er_row_widths,
                                 void** out_val_ell, uint16_t** out_col_ell, int64_t* out_slots_ell,
                                 void** out_val_er, uint32_t** out_col_er, int64_t* out_slots_er);

/* Host view of an assembled EhybMatrix (format.py:202-248). Array lengths
 * travel beside their pointers so ehyb_check can validate them. */
typedef struct ehyb_host_matrix {
  int64_t dimension;
  int64_t padded_dimension;
  int64_t plan_padded_dimension;
  int64_t k;
  int64_t n_parts;
  int64_t vec_cache_size;
  int64_t warp_size;
  int64_t tau;
  int64_t n_er_rows;
  const int64_t* reorder; int64_t n_reorder;
  const int64_t* inverse; int64_t n_inverse;
  const int64_t* y_idx_er; int64_t n_y_idx_er;
  const int32_t* part_boundary; int64_t n_part_boundary;
  const int32_t* position_ell; int64_t n_position_ell;
  const int32_t* width_ell; int64_t n_width_ell;
  const int32_t* ell_row_widths; int64_t n_ell_row_widths;
  const uint16_t* col_ell; int64_t n_col_ell;
  const void* val_ell; int64_t slots_ell;
  const int32_t* position_er; int64_t n_position_er;
  const int32_t* width_er; int64_t n_width_er;
  const int32_t* er_row_widths; int64_t n_er_row_widths;
  const uint32_t* col_er; int64_t n_col_er;
  const void* val_er; int64_t slots_er;
} ehyb_host_matrix;

/* EhybMatrix.check (format.py:250-299): structural invariants, O(size). */
EHYB_API int ehyb_check(const ehyb_host_matrix* m);

/* ------------------------------------------------------ device (B200) */

typedef struct ehyb_dev ehyb_dev; /* opaque device handle */

typedef struct ehyb_dev_info {
  int64_t device_bytes;       /* total HBM held by the handle */
  int64_t er_slices;          /* per-partition ER slices (derived layout) */
  int64_t er_slots;           /* derived ER slots incl. padding */
  int64_t window_bytes;       /* x window staged per CTA */
  int32_t window_in_smem;     /* 1: window staged in shared memory by TMA bulk copy */
  int32_t threads_per_cta;
  int32_t ctas;               /* grid size of one SpMV launch */
  int32_t sm_count;
  int64_t pool_slices;        /* ER slices in the cross-CTA pool (0 = pool off) */
  int32_t er_buf_slices;      /* own ER slices buffered in shared memory per CTA */
  int32_t smem_bytes;         /* dynamic shared memory of a fused launch */
  int64_t long_rows;          /* rows computed by the long-row path (width > EHYB_LONG_ROW) */
  int64_t ring_bytes;         /* shared-memory ring the ELL stream is TMA-staged through (0 = off) */
  int64_t work_units;         /* CTA work units of a launch: partitions x split */
  int32_t split;              /* units per partition (chunk ranges of one window; EHYB_SPLIT) */
  int32_t reserved;
} ehyb_dev_info;

/* Upload an assembled matrix once (device = CUDA ordinal) and derive the
 * per-partition ER layout the fused kernel reads. Replaces the per-call
 * array traversal of spmv_ehyb (engine.py:108-216). */
EHYB_API int ehyb_dev_create(const ehyb_host_matrix* m, int device, ehyb_dev** out);
EHYB_API int ehyb_dev_destroy(ehyb_dev* h);
EHYB_API int ehyb_dev_info_get(const ehyb_dev* h, ehyb_dev_info* out);

/* Launch tuning of a handle (defaults are the measured best for B200):
 *   EHYB_TUNE_PREFETCH_ELL  ELL slices kept ahead of the warps by TMA bulk
 *                           L2 prefetch (0 = off)
 *   EHYB_TUNE_PREFETCH_ER   1 = bulk-prefetch each warp's next ER slice
 *   EHYB_TUNE_THREADS       threads per CTA (multiple of 32, <= 1024)
 *   EHYB_TUNE_TIMING        device pointer to n_parts*8 u64 %globaltimer
 *                           stamps per CTA (start, window ready, ELL
 *                           issue drained, end, own ER done, combine done,
 *                           pool done, ELL published), zeroed by the
 *                           caller, 0 = off */
#define EHYB_TUNE_PREFETCH_ELL 1
#define EHYB_TUNE_PREFETCH_ER 2
#define EHYB_TUNE_THREADS 3
#define EHYB_TUNE_TIMING 4
#define EHYB_TUNE_ER_WARPS 5 /* warps that compute own ER rows before ELL (default 6; half the CTA for small partitions) */
#define EHYB_TUNE_CLAIM_AHEAD 6 /* bit0: ELL chunks, bit1: ER slices claimed one ahead */
#define EHYB_TUNE_PHASES 7      /* measurement only: bit0 skips the ER work, bit1 the ELL
                                   stream (y is then incomplete) */
EHYB_API int ehyb_dev_tune(ehyb_dev* h, int key, int64_t value);

/* spmv_ehyb (engine.py:108-216) in reordered space: y[padded] = A x[padded].
 * x, y: device arrays of the stored precision (tau 4 -> float, 8 -> double),
 * non-aliasing. One fused kernel: per partition, TMA-staged x window ->
 * ELL slices -> the partition's ER rows. mode: EHYB_MODE_*. */
EHYB_API int ehyb_dev_spmv(ehyb_dev* h, const void* x_dev, void* y_dev, int mode, void* stream);

/* permute_vector (format.py:445-452) / unpermute_vector (format.py:455-460)
 * on device; x_user, y_user have `dimension` entries, x_r / y_r padded. */
EHYB_API int ehyb_dev_permute(ehyb_dev* h, const void* x_user, void* x_r, void* stream);
EHYB_API int ehyb_dev_unpermute(ehyb_dev* h, const void* y_r, void* y_user, void* stream);

/* spmv_ehyb_user (engine.py:219-227) on device buffers in user order:
 * permute -> fused SpMV -> unpermute, using handle-owned scratch. */
EHYB_API int ehyb_dev_spmv_user(ehyb_dev* h, const void* x_user, void* y_user, int mode,
                                void* stream);

/* The same from HOST memory: copy x in, run, copy y out, synchronise.
 * user_order=1: x,y have `dimension` entries (spmv_ehyb_user);
 * user_order=0: x,y are padded reordered vectors (spmv_ehyb).
 * Host buffers may be pageable or pinned (pinned is faster). */
EHYB_API int ehyb_dev_spmv_host(ehyb_dev* h, const void* x_host, void* y_host, int user_order,
                                int mode, void* stream);

/* A sequence of independent products from HOST memory (the same call as
 * ehyb_dev_spmv_host repeated `count` times: vector i is x_hosts[i] ->
 * y_hosts[i], user_order as above), pipelined on three device buffer pairs:
 * the copy-in of vector i+1 and the copy-out of vector i-1 overlap the
 * product of vector i (copy-in / copy-out on handle-owned streams, compute on
 * `stream`). Returns after the last copy-out; host buffers should be pinned.
 * Results are bitwise those of count single calls. */
EHYB_API int ehyb_dev_spmv_host_many(ehyb_dev* h, const void* const* x_hosts,
                                     void* const* y_hosts, int64_t count, int user_order,
                                     int mode, void* stream);

/* ------------------------------------------- cuSPARSE CSR comparator */
typedef struct ehyb_csr ehyb_csr;
/* CSR (coo_to_csr, matrix_io.py:255-268 layout) uploaded with int32 indices
 * and values at tau bytes. */
EHYB_API int ehyb_csr_create(int64_t n_rows, int64_t n_cols, int64_t nnz, const int64_t* row_ptr,
                             const int64_t* col_idx, const double* values, int32_t tau,
                             int device, ehyb_csr** out);
/* y = A x. alg 0 = the reference oracle's own order (replaces
 * engine.py:56-69 spmv_csr: fp64 products, np.add.reduceat row sums with
 * numpy's pairwise summation; bitwise the reference's y; tau must be 8);
 * alg 1 = cusparseSpMV CUSPARSE_SPMV_CSR_ALG1, 2 = ALG2 (the comparator). */
EHYB_API int ehyb_csr_spmv(ehyb_csr* h, const void* x_dev, void* y_dev, int alg, void* stream);
EHYB_API int ehyb_csr_destroy(ehyb_csr* h);

/* --------------------------------------------- multi-GPU row shards */

/* A shard owns a contiguous block of partitions [p0, p1) of a matrix that
 * was assembled once for the whole job; its x/y range is the new-row range
 * [p0*vec, p1*vec). ER columns outside that range are remapped into a halo
 * segment appended after the owned window: x_ext = [owned | halo]. */
typedef struct ehyb_shard_plan {
  int64_t p0, p1;          /* owned partitions */
  int64_t n_halo;          /* distinct remote columns referenced by owned ER rows */
  const int64_t* halo_cols;/* global new-order column of each halo slot (ascending) */
} ehyb_shard_plan;

/* Upload the owned part of the matrix; ER columns are remapped against
 * plan->halo_cols. The shard's SpMV reads x_ext[(p1-p0)*vec + n_halo]. */
EHYB_API int ehyb_dev_create_shard(const ehyb_host_matrix* m, const ehyb_shard_plan* plan,
                                   int device, ehyb_dev** out);

/* Split SpMV for overlap with the halo exchange.
 * ehyb_dev_spmv_ell: the local phase — ELL plus every ER row whose columns
 *   are all owned (own slices, shared-memory buffer, cross-CTA pool); reads
 *   only x_ext[0, local_rows), so it runs while the halo is in flight.
 * ehyb_dev_spmv_er: the halo phase — ER rows with a halo column and long
 *   rows; needs x_ext complete. Each ER row is added to y exactly once.
 * ehyb_dev_spmv on a shard handle runs all of it in one launch. */
EHYB_API int ehyb_dev_spmv_ell(ehyb_dev* h, const void* x_ext, void* y_local, int mode,
                               void* stream);
EHYB_API int ehyb_dev_spmv_er(ehyb_dev* h, const void* x_ext, void* y_local, int mode,
                              void* stream);

/* P2P halo exchange (one launch per SpMV, no NCCL): the shard handle owns
 * x_ext ([owned | halo], tau bytes each) and a 64-byte flag block, both
 * IPC-shareable. Every rank publishes IPC handles of both (ehyb_ipc_handle),
 * maps its peers' (ehyb_ipc_open) and passes them with its pull plan (per
 * halo slot: source rank and offset in that rank's x_ext) to
 * ehyb_dev_p2p_setup; served_per_spmv = values the peers pull from this rank
 * per SpMV. ehyb_dev_spmv_p2p then runs ELL, local ER, the halo pull from
 * peer memory and the halo rows in one launch; it returns (stream-ordered)
 * only after the peers have pulled from this rank, so the next kernel may
 * overwrite x_ext. All ranks must issue the same sequence of p2p SpMVs (in
 * lockstep: the n-th call on every rank is the same SpMV). A rank whose peer
 * never issues its matching call does not hang: each cross-rank wait traps
 * after EHYB_SPIN_TIMEOUT_S seconds (default 20), failing the launch with a
 * CUDA error, and a launch that fails to issue leaves the sequence number
 * unchanged. */
EHYB_API int ehyb_dev_p2p_alloc(ehyb_dev* h, void** x_ext, void** flags);
EHYB_API int ehyb_ipc_handle(const void* dev_ptr, void* out_handle /* 64 bytes */);
EHYB_API int ehyb_ipc_open(const void* handle, int device, void** out_ptr);
EHYB_API int ehyb_ipc_close(void* ptr);
EHYB_API int ehyb_dev_p2p_setup(ehyb_dev* h, int32_t world, int32_t rank, void* const* peer_x,
                                void* const* peer_flags, const int32_t* pull_src,
                                const int64_t* pull_off, int64_t served_per_spmv);
EHYB_API int ehyb_dev_spmv_p2p(ehyb_dev* h, void* y_local, int mode, void* stream);

/* Gather x_local[idx[i]] into a packed send buffer (halo pack). */
EHYB_API int ehyb_dev_gather(const void* src, const int64_t* idx_dev, int64_t count, void* dst,
                             int32_t tau, void* stream);

/* ------------------------------------------------ CG building blocks */
/* dot products of the CG loop, accumulated in fp64 into out_dev[0]
 * (deterministic two-level reduction, no atomics). */
EHYB_API int ehyb_dev_dot(const void* a, const void* b, int64_t n, int32_t tau, double* out_dev,
                          void* stream);
/* CG updates with device-resident scalars: alpha = rr[0]/pq[0];
 * x += alpha p; r -= alpha q; rr_new[0] = r.r (local part, deterministic). */
EHYB_API int ehyb_dev_cg_xr(void* x, void* r, const void* p, const void* q, const double* rr,
                            const double* pq, int64_t n, int32_t tau, double* rr_new,
                            void* stream);
/* p = r + (rr_new[0] / rr_old[0]) p. */
EHYB_API int ehyb_dev_cg_p(void* p, const void* r, const double* rr_new, const double* rr_old,
                           int64_t n, int32_t tau, void* stream);
/* y = a*x + y (a read from device memory, scaled by sign). */
/* Chronopoulos-Gear CG (one all-reduce per iteration): two fp64 dot
 * products in one pass, out2_dev = {a.b, c.d}; and one step's scalar update
 * (sc = {gamma, delta, gamma_old, alpha, beta} on the device) fused with
 * p = r + beta p, s = w + beta s, x += alpha p, r -= alpha s. */
EHYB_API int ehyb_dev_dot2(const void* a, const void* b, const void* c, const void* d, int64_t n,
                           int32_t tau, double* out2_dev, void* stream);
EHYB_API int ehyb_dev_cgcg_step(void* x, void* r, void* p, void* s, const void* w, double* sc,
                                int first, int64_t n, int32_t tau, void* stream);
EHYB_API int ehyb_dev_axpy(const double* a_dev, double sign, const void* x, void* y, int64_t n,
                           int32_t tau, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* EHYB_B200_H */
