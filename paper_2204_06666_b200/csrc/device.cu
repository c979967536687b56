// Device side of the C ABI: matrix upload (ehyb_dev_create / _create_shard),
// the derived per-partition ER layout, SpMV launches, permutation, the
// cuSPARSE comparator and the CG vector primitives.
//
// Derived layout (built once at upload, never a parity object): the
// reference stores ER rows globally sorted by outer count and sliced by
// warp_size (format.py:367-392); its engine runs them after a grid-wide
// barrier (engine.py:146-154, 172-173). Here the ER rows are regrouped by
// the partition that owns their output row (y_idx_er // vec), keeping the
// reference's relative order (so widths stay descending) and re-sliced in
// 32-row SELL slices, so the owning CTA finishes its own rows without a
// grid barrier or atomics. Each row keeps its entries in the reference's k
// order, so the accumulation is unchanged.

#include "ehyb_common.h"
#include "kernels.cuh"

#include <cuda_runtime.h>
#include <cusparse.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

using namespace ehyb;

#define CUDA_TRY(expr)                                                                       \
  do {                                                                                       \
    cudaError_t err__ = (expr);                                                              \
    if (err__ != cudaSuccess)                                                                \
      return ehyb::fail(std::string(#expr) + ": " + cudaGetErrorString(err__), EHYB_ECUDA); \
  } while (0)

#define CUSPARSE_TRY(expr)                                                                 \
  do {                                                                                     \
    cusparseStatus_t st__ = (expr);                                                        \
    if (st__ != CUSPARSE_STATUS_SUCCESS)                                                   \
      return ehyb::fail(std::string(#expr) + ": cusparse status " + std::to_string(int(st__)), \
                        EHYB_ECUDA);                                                       \
  } while (0)

namespace {

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

template <typename P>
cudaError_t upload(P** dst, const void* src, size_t bytes, size_t* total) {
  *dst = nullptr;
  cudaError_t e = cudaMalloc(reinterpret_cast<void**>(dst), std::max<size_t>(bytes, 16));
  if (e != cudaSuccess) return e;
  *total += std::max<size_t>(bytes, 16);
  // large arrays (the ELL slab: 4.5 GB for cfg5) through the pinned double
  // buffer: host copy of one half overlapped with the DMA of the other
  static const bool staged = [] {
    const char* v = std::getenv("EHYB_UPLOAD_STAGED");  // dev: 0 = plain cudaMemcpy
    return !(v && *v && std::atof(v) == 0.0);
  }();
  if (bytes) e = staged ? staged_h2d(*dst, src, bytes) : cudaMemcpy(*dst, src, bytes, cudaMemcpyHostToDevice);
  return e;
}

}  // namespace

struct ehyb_dev {
  int device = 0;
  int tau = 8;
  int64_t dimension = 0, padded = 0, n_parts = 0, vec = 0, warp = 32;
  int64_t local_rows = 0, n_halo = 0;  // shard geometry (full matrix: local_rows == padded)
  bool shard = false;
  // ELL parity arrays (re-based to the owned partitions)
  void* val_ell = nullptr;
  uint16_t* col_ell = nullptr;
  int32_t* pos_ell = nullptr;
  int32_t* width_ell = nullptr;
  // derived ER
  int64_t er_slices = 0, er_slots = 0;
  int32_t* er_part_ptr = nullptr;
  int32_t* er_part_mid = nullptr;  // first halo slice of each partition (shards)
  int64_t* er_pos = nullptr;
  int32_t* er_swidth = nullptr;
  int32_t* er_rows = nullptr;
  int32_t* er_lwidth = nullptr;
  void* er_val = nullptr;
  uint32_t* er_col = nullptr;
  // permutation (full matrix only)
  int32_t* reorder = nullptr;  // [dimension]
  int32_t* inverse = nullptr;  // [padded]
  // scratch
  void* xr = nullptr;
  void* yr = nullptr;
  void* xu = nullptr;
  void* yu = nullptr;
  // launch configuration
  int threads = 1024;
  size_t smem = 0;      // dynamic smem of a fused launch (window + ER buffer)
  size_t win_bytes = 0;  // window part
  bool window_in_smem = false, window_tma = false;
  int sm_count = 0;
  int64_t max_ctas = 1;  // co-resident CTAs of the fused kernel (occupancy x SMs)
  size_t bytes = 0;
  // tuning knobs (ehyb_dev_tune) and optional per-CTA timing buffer
  int pf_ell = 0, pf_er = 1;
  unsigned long long* timing = nullptr;
  // ER pool (cross-CTA load balance)
  int64_t pool_lo = 0, pool_hi = 0;
  unsigned int* pool_done = nullptr;
  int32_t* pool_own_ptr = nullptr;
  int32_t* pool_own_idx = nullptr;
  int32_t* unit_part = nullptr;  // persistent launches: unit -> partition (heaviest first)
  int32_t* part_unit = nullptr;  // its inverse
  void* pool_acc = nullptr;
  int32_t* pool_pos = nullptr;   // owner-major position of each pooled slice
  int32_t* pool_rows = nullptr;  // pooled slices' rows, owner-major
  void* own_acc = nullptr;  // own ER sums beyond the shared-memory buffer
  // P2P halo exchange (shards): x_ext and flags owned by the handle (IPC-able),
  // the pull plan and the peers' mapped buffers
  void* p2p_x = nullptr;
  unsigned long long* p2p_flags = nullptr;
  int32_t* pull_src = nullptr;
  int64_t* pull_off = nullptr;
  void** peer_x_dev = nullptr;
  unsigned long long** peer_flags_dev = nullptr;
  unsigned long long p2p_seq = 0, served_per_spmv = 0;
  bool p2p_ready = false, p2p_active = false;
  unsigned int* part_flag = nullptr;  // persistent mode: per-partition publication
  int32_t* pool_grp = nullptr;         // pooled-slice range per iteration group
  int32_t pool_groups = 0;
  int32_t pool_last_scratch = 0;  // last iteration group via scratch + owner add
  unsigned int* pool_gctr = nullptr;
  unsigned int* pool_ctr = nullptr;
  unsigned int* epoch_dev = nullptr;  // [2] launch epoch, CTAs finished (device-side: graph-safe)
  // own-ER shared-memory buffer
  int er_buf_slices = 0, er_buf_offset = 0, er_warps = 6;  // measured best: cfg2 102.5 vs 103.7 us at 8
  size_t ring_offset = 0, ring_bytes = 0;  // ELL staging ring (0 = register path)
  int ring_stages = 0, stage_bytes = 0, stage_vbytes = 0;
  bool ell_vec = false;  // ELL slices in the 128-bit interleaved layout
  int32_t* part_stage_ptr = nullptr;  // ring stage plan (see SpmvParams)
  int32_t* st_pos = nullptr;
  int32_t* st_slots = nullptr;
  int32_t* st_chunks = nullptr;
  uint2* ch_stage = nullptr;
  int ell_ahead = 1, er_ahead = 1;
  int32_t meta_off = -1;  // chunk metadata in dynamic smem (byte offset), -1 = global loads
  int phase_skip = 0;
  int32_t split = 1, unit_chunks = 0;  // work units per partition, chunks per unit
  int64_t n_units = 0;                 // launch work units (partitions x split)  // EHYB_TUNE_PHASES (dev): bit 0 skips the ER work, bit 1 the ELL stream
  // ER padding column (SURVEY.md 8a gotcha 4): x index of the column the
  // reference's padding slots hold; shards without it locally fix up later
  int64_t er_pad_idx = 0;
  int32_t* padfix_rows = nullptr;
  int64_t padfix_n = 0;
  unsigned long long spin_timeout_ns = 20000000000ull;  // cross-rank waits trap after this
  bool cooperative = true;  // launch the fused kernel cooperatively (EHYB_COOPERATIVE=0: plain)
  // long rows (derived): masked out of the slice paths, computed by warps
  uint32_t* long_bits = nullptr;
  int32_t lr_tasks = 0, lr_segs = 0;
  int64_t* lr_span = nullptr;
  int32_t* lr_row = nullptr;
  int64_t* lr_padcol = nullptr;
  void* lr_val = nullptr;
  uint32_t* lr_col = nullptr;
  int64_t* lr_seg = nullptr;
  int32_t* lr_task_seg = nullptr;
  int32_t* lr_task_nell = nullptr;
  void* lr_part = nullptr;
  unsigned int* lr_cnt = nullptr;
  unsigned int* lr_ctr = nullptr;
  // host-batch pipeline (ehyb_dev_spmv_host_many): copy-in / copy-out streams,
  // two device buffer pairs, per-buffer events
  static constexpr int kPipe = 3;  // device buffer pairs in flight
  cudaStream_t s_in = nullptr, s_out = nullptr;
  cudaEvent_t ev_in[kPipe] = {}, ev_comp[kPipe] = {}, ev_out[kPipe] = {};
  void* bx[kPipe] = {};
  void* by[kPipe] = {};

  ~ehyb_dev() {
    void* ptrs[] = {val_ell, col_ell, pos_ell, width_ell, er_part_ptr, er_part_mid, er_pos, er_swidth,
                    er_rows, er_lwidth, er_val, er_col, reorder, inverse, xr, yr, xu, yu,
                    pool_done, pool_own_ptr, pool_own_idx, unit_part, part_unit, pool_acc, pool_pos, pool_rows, own_acc, p2p_x, p2p_flags, pull_src, pull_off, peer_x_dev, peer_flags_dev,
                    pool_ctr, epoch_dev, part_flag, pool_grp, pool_gctr,
                    part_stage_ptr, st_pos, st_slots, st_chunks, ch_stage,
                    bx[2], by[2], bx[0], bx[1], by[0], by[1], long_bits, lr_span,
                    lr_row, lr_padcol, lr_val, lr_col, lr_seg, lr_task_seg, lr_task_nell,
                    lr_part, lr_cnt, lr_ctr, padfix_rows};
    for (void* p : ptrs)
      if (p) cudaFree(p);
    for (int b = 0; b < kPipe; ++b) {
      if (ev_in[b]) cudaEventDestroy(ev_in[b]);
      if (ev_comp[b]) cudaEventDestroy(ev_comp[b]);
      if (ev_out[b]) cudaEventDestroy(ev_out[b]);
    }
    if (s_in) cudaStreamDestroy(s_in);
    if (s_out) cudaStreamDestroy(s_out);
  }
};

namespace {

template <typename T, int MODE, bool C32>
cudaError_t launch_typed(const ehyb_dev* h, const void* x, void* y, bool do_ell, bool do_er,
                         cudaStream_t st) {
  SpmvParams<T> P;
  P.val_ell = static_cast<const T*>(h->val_ell);
  P.col_ell = h->col_ell;
  P.pos_ell = h->pos_ell;
  P.width_ell = h->width_ell;
  P.er_part_ptr = h->er_part_ptr;
  P.er_part_mid = h->er_part_mid;
  // launch kinds: full (ELL + all ER), local phase (ELL + ER rows whose columns
  // are all owned, pool included), halo phase (ER rows with a halo column and
  // long rows, after the exchange)
  P.er_sel = (do_ell && do_er) ? 0 : (do_ell ? 1 : 2);
  do_er = !(h->phase_skip & 1);  // dev measurement: EHYB_TUNE_PHASES bit 0 = no ER work
  P.er_pos = h->er_pos;
  P.er_swidth = h->er_swidth;
  P.er_rows = h->er_rows;
  P.er_lwidth = h->er_lwidth;
  P.er_val = static_cast<const T*>(h->er_val);
  P.er_col = h->er_col;
  P.x = static_cast<const T*>(x);
  P.er_pad_idx = h->er_pad_idx;
  P.y = static_cast<T*>(y);
  P.vec = h->vec;
  P.warp = int32_t(h->warp);
  P.window_in_smem = (do_ell && h->window_in_smem) ? 1 : 0;
  P.window_tma = h->window_tma ? 1 : 0;
  P.do_ell = (do_ell && !(h->phase_skip & 2)) ? 1 : 0;
  P.do_er = do_er ? 1 : 0;
  P.pf_ell = h->pf_ell;
  P.pf_er = h->pf_er;
  P.timing = h->timing;
  P.pool_lo = h->pool_lo;
  P.pool_hi = h->pool_hi;
  P.pool_ctr = h->pool_ctr;
  P.pool_done = h->pool_done;
  P.pool_own_ptr = h->pool_own_ptr;
  P.pool_own_idx = h->pool_own_idx;
  P.pool_acc = static_cast<T*>(h->pool_acc);
  P.pool_pos = h->pool_pos;
  P.pool_rows = h->pool_rows;
  P.own_acc = static_cast<T*>(h->own_acc);
  P.n_halo = h->n_halo;
  P.local_rows = h->local_rows;
  P.pull_src = h->pull_src;
  P.pull_off = h->pull_off;
  P.peer_x = reinterpret_cast<T* const*>(h->peer_x_dev);
  P.peer_flags = h->peer_flags_dev;
  P.my_flags = h->p2p_flags;
  P.seq = h->p2p_seq;
  P.spin_timeout_ns = h->spin_timeout_ns;
  P.served_per_spmv = h->served_per_spmv;
  P.part_flag = h->part_flag;
  P.pool_grp = h->pool_grp;
  P.pool_groups = h->pool_groups;
  P.pool_gctr = h->pool_gctr;
  P.pool_last_scratch = h->pool_last_scratch;
  P.epoch_dev = h->epoch_dev;
  P.er_buf_slices = h->er_buf_slices;
  P.er_buf_offset = h->er_buf_offset;
  P.er_warps = h->er_warps;
  P.n_parts = int32_t(h->n_units);
  P.split = h->split;
  P.unit_chunks = h->unit_chunks;
  P.meta_off = h->meta_off;
  P.unit_part = h->unit_part;
  P.part_unit = h->part_unit;
  P.ell_ahead = h->ell_ahead;
  P.er_ahead = h->er_ahead;
  P.long_bits = h->long_bits;
  P.ell_vec = h->ell_vec ? 1 : 0;
  P.lr_tasks = h->lr_tasks;
  P.lr_span = h->lr_span;
  P.lr_row = h->lr_row;
  P.lr_padcol = h->lr_padcol;
  P.lr_val = static_cast<const T*>(h->lr_val);
  P.lr_col = h->lr_col;
  P.lr_segs = h->lr_segs;
  P.lr_seg = h->lr_seg;
  P.lr_task_seg = h->lr_task_seg;
  P.lr_task_nell = h->lr_task_nell;
  P.lr_part = static_cast<T*>(h->lr_part);
  P.lr_cnt = h->lr_cnt;
  P.lr_ctr = h->lr_ctr;
  if (P.er_sel == 1) P.lr_tasks = 0;  // long rows may read the halo: halo phase
  if (P.er_sel == 2) {                 // the pool holds local rows only
    P.pool_lo = P.pool_hi;
    P.pool_own_ptr = nullptr;
    P.part_flag = nullptr;  // no group drains (the group counters still reset)
    P.pool_last_scratch = 0;
  }
  // work-unit split (several CTAs per partition): its own variant, so the
  // one-unit-per-partition kernel keeps the register allocation it had
  const bool split = h->split > 1;
#ifdef EHYB_DEV_ONE
  // dev experiments (EHYB_NVCC_FLAGS=-DEHYB_DEV_ONE=<tau> -DEHYB_DEV_MODE=<m>):
  // one kernel variant compiled, every other launch kind refused
  if (!(do_ell && h->window_in_smem) || split || h->p2p_active || h->ring_bytes > 0 || !C32)
    return cudaErrorNotSupported;
  size_t smem = (do_ell && (do_er || h->meta_off >= 0)) ? h->smem : (P.window_in_smem ? h->win_bytes : 0);
  void (*kern)(const SpmvParams<T>) = spmv_fused_kernel<T, MODE, true, true, false>;
  P.ring_offset = 0;
  P.ring_stages = P.stage_bytes = P.stage_vbytes = 0;
  P.part_stage_ptr = P.st_pos = P.st_slots = P.st_chunks = nullptr;
  P.ch_stage = nullptr;
#else
  void (*kern)(const SpmvParams<T>) =
      (do_ell && h->window_in_smem)
          ? (split ? spmv_fused_kernel<T, MODE, C32, true, false, false, true>
                   : spmv_fused_kernel<T, MODE, C32, true, false>)
          : (split ? spmv_fused_kernel<T, MODE, C32, false, false, false, true>
                   : spmv_fused_kernel<T, MODE, C32, false, false>);
  // dynamic smem: [window | own-ER buffer | ELL ring]; the buffer is only
  // used when one launch runs both phases, the ring by any ELL launch
  size_t smem = (do_ell && (do_er || h->meta_off >= 0)) ? h->smem : (P.window_in_smem ? h->win_bytes : 0);
  P.ring_offset = 0;
  P.ring_stages = P.stage_bytes = P.stage_vbytes = 0;
  P.part_stage_ptr = P.st_pos = P.st_slots = P.st_chunks = nullptr;
  P.ch_stage = nullptr;
  if constexpr (C32) {
    if (do_ell && h->window_in_smem && h->window_tma && h->ring_bytes > 0 && h->threads >= 64) {
      kern = spmv_fused_kernel<T, MODE, true, true, true>;
      P.ring_offset = int32_t(h->ring_offset);
      P.ring_stages = h->ring_stages;
      P.stage_bytes = h->stage_bytes;
      P.stage_vbytes = h->stage_vbytes;
      P.part_stage_ptr = h->part_stage_ptr;
      P.st_pos = h->st_pos;
      P.st_slots = h->st_slots;
      P.st_chunks = h->st_chunks;
      P.ch_stage = h->ch_stage;
      smem = h->ring_offset + h->ring_bytes;
    }
  }
  if constexpr (C32) {
    if (h->p2p_active)
      kern = split ? spmv_fused_kernel<T, MODE, true, true, false, true, true>
                   : spmv_fused_kernel<T, MODE, true, true, false, true>;
  }
#endif  // EHYB_DEV_ONE
  if (!(do_ell && do_er)) {
    P.er_buf_slices = 0;
  }
  if (smem > 48 * 1024) {
    // opt in once per (kernel, device) to the largest window any handle needs
    static std::mutex mu;
    static std::unordered_map<std::string, size_t> configured;
    const std::string key = std::to_string(reinterpret_cast<uintptr_t>(
                                reinterpret_cast<const void*>(kern))) + ":" + std::to_string(h->device);
    std::lock_guard<std::mutex> lock(mu);
    auto it = configured.find(key);
    if (it == configured.end() || it->second < smem) {
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
      if (e != cudaSuccess) return e;
      configured[key] = smem;
    }
  }
  // at most one wave of resident CTAs; each loops over its partitions
  const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(h->n_units, h->max_ctas));

  // cooperative launch: the runtime guarantees every CTA of the grid is
  // resident at once (or fails the launch) — the pool, persistent-group and
  // P2P protocols spin on flags other CTAs write, so a partially scheduled
  // grid (another kernel holding SMs, e.g. an overlapped NCCL collective)
  // must never start
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(unsigned(grid));
  cfg.blockDim = dim3(unsigned(h->threads));
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = h->cooperative ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, P);
}

template <typename T>
cudaError_t launch_mode(const ehyb_dev* h, const void* x, void* y, int mode, bool ell, bool er,
                        cudaStream_t st) {
  const bool c32 = h->warp == 32;
#ifdef EHYB_DEV_ONE
  if constexpr (sizeof(T) == EHYB_DEV_ONE) {
    if (mode == EHYB_DEV_MODE && c32) return launch_typed<T, EHYB_DEV_MODE, true>(h, x, y, ell, er, st);
  }
  return cudaErrorNotSupported;
#else
  if (mode == EHYB_MODE_FMA)
    return c32 ? launch_typed<T, EHYB_MODE_FMA, true>(h, x, y, ell, er, st)
               : launch_typed<T, EHYB_MODE_FMA, false>(h, x, y, ell, er, st);
  if (mode == EHYB_MODE_DEFAULT)
    return c32 ? launch_typed<T, EHYB_MODE_DEFAULT, true>(h, x, y, ell, er, st)
               : launch_typed<T, EHYB_MODE_DEFAULT, false>(h, x, y, ell, er, st);
  return c32 ? launch_typed<T, EHYB_MODE_STRICT, true>(h, x, y, ell, er, st)
             : launch_typed<T, EHYB_MODE_STRICT, false>(h, x, y, ell, er, st);
#endif
}

cudaError_t launch_spmv(ehyb_dev* h, const void* x, void* y, int mode, bool ell, bool er,
                        cudaStream_t st) {
  if (mode != EHYB_MODE_STRICT && mode != EHYB_MODE_FMA && mode != EHYB_MODE_DEFAULT)
    return cudaErrorInvalidValue;
  cudaError_t e = h->tau == 4 ? launch_mode<float>(h, x, y, mode, ell, er, st)
                              : launch_mode<double>(h, x, y, mode, ell, er, st);
  if (e != cudaSuccess || !er || h->padfix_n == 0) return e;
  // ER finished: the padding products of rows whose padding column is remote
  const int blocks = int(std::min<int64_t>((h->padfix_n + 255) / 256, int64_t(h->sm_count) * 4));
  if (h->tau == 4)
    pad_fixup_kernel<float><<<blocks, 256, 0, st>>>(static_cast<float*>(y), h->padfix_rows,
                                                     h->padfix_n,
                                                     static_cast<const float*>(x) + h->er_pad_idx);
  else
    pad_fixup_kernel<double><<<blocks, 256, 0, st>>>(static_cast<double*>(y), h->padfix_rows,
                                                      h->padfix_n,
                                                      static_cast<const double*>(x) + h->er_pad_idx);
  return cudaGetLastError();
}

double env_double(const char* name, double dflt) {
  const char* v = std::getenv(name);
  if (!v || !*v) return dflt;
  return std::atof(v);
}

template <typename T, int MODE>
const void* fused_variant(bool c32, bool smem) {
#ifdef EHYB_DEV_ONE
  if constexpr (sizeof(T) == EHYB_DEV_ONE) return (const void*)spmv_fused_kernel<T, EHYB_DEV_MODE, true, true, false>;
  return nullptr;
#else
  return c32 ? (smem ? (const void*)spmv_fused_kernel<T, MODE, true, true, false>
                     : (const void*)spmv_fused_kernel<T, MODE, true, false, false>)
             : (smem ? (const void*)spmv_fused_kernel<T, MODE, false, true, false>
                     : (const void*)spmv_fused_kernel<T, MODE, false, false, false>);
#endif
}

// resident CTAs per SM of the fused kernel for this handle's configuration:
// the minimum over the arithmetic-mode variants, so every launch mode fits
// the one grid the persistent-group layout was built for
cudaError_t occupancy(const ehyb_dev* h, int* per_sm) {
  const bool c32 = h->warp == 32;
  const void* ks[3];
  if (h->tau == 4) {
    ks[0] = fused_variant<float, EHYB_MODE_STRICT>(c32, h->window_in_smem);
    ks[1] = fused_variant<float, EHYB_MODE_FMA>(c32, h->window_in_smem);
    ks[2] = fused_variant<float, EHYB_MODE_DEFAULT>(c32, h->window_in_smem);
  } else {
    ks[0] = fused_variant<double, EHYB_MODE_STRICT>(c32, h->window_in_smem);
    ks[1] = fused_variant<double, EHYB_MODE_FMA>(c32, h->window_in_smem);
    ks[2] = fused_variant<double, EHYB_MODE_DEFAULT>(c32, h->window_in_smem);
  }
  *per_sm = 1 << 30;
  for (const void* k : ks) {
    if (!k) continue;
    if (h->smem > 48 * 1024) {
      cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(h->smem));
      if (e != cudaSuccess) return e;
    }
    int n = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k, h->threads, h->smem);
    if (e != cudaSuccess) return e;
    *per_sm = std::min(*per_sm, n);
  }
  return cudaSuccess;
}

int grid_for(int64_t n, int threads, int sms) {
  int64_t g = (n + threads - 1) / threads;
  return int(std::max<int64_t>(1, std::min<int64_t>(g, int64_t(sms) * 16)));
}

// Build the device copy of partitions [p0, p1). ER columns are remapped:
// owned columns -> c - p0*vec, halo columns -> local_rows + slot in halo_cols.
int create_impl(const ehyb_host_matrix* m, int64_t p0, int64_t p1, const int64_t* halo_cols,
                int64_t n_halo, bool shard, int device, ehyb_dev** out) {
  if (!m || !out) return fail("null argument");
  if (m->tau != 4 && m->tau != 8) return fail("tau must be 4 or 8");
  if (p0 < 0 || p1 > m->n_parts || p0 >= p1) return fail("bad shard partition range");
  const int64_t vec = m->vec_cache_size, C = m->warp_size;
  const int64_t padded = m->padded_dimension;
  if (padded >= (int64_t(1) << 30)) return fail("padded dimension exceeds the 2^30 device row range");
  const size_t tb = size_t(m->tau);

  int ndev = 0;
  CUDA_TRY(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) return fail("invalid CUDA device ordinal", EHYB_ECUDA);
  DeviceGuard guard(device);
  auto h = std::make_unique<ehyb_dev>();
  h->device = device;
  h->tau = int(m->tau);
  h->dimension = m->dimension;
  h->padded = padded;
  h->n_parts = m->n_parts;
  h->vec = vec;
  h->warp = C;
  h->shard = shard;
  h->local_rows = (p1 - p0) * vec;
  h->n_halo = n_halo;
  const int64_t row_lo = p0 * vec, row_hi = p1 * vec;

  // ---- ELL: slices of the owned rows, positions re-based
  const int64_t s_lo = row_lo / C, s_hi = row_hi / C;
  const int64_t base = m->position_ell[s_lo];
  const int64_t slots = int64_t(m->position_ell[s_hi]) - base;
  std::vector<int32_t> pos(size_t(s_hi - s_lo) + 1);
  for (int64_t s = s_lo; s <= s_hi; ++s) pos[size_t(s - s_lo)] = int32_t(m->position_ell[s] - base);
  CUDA_TRY(upload(&h->pos_ell, pos.data(), pos.size() * 4, &h->bytes));

  // ---- long rows: ELL or ER width above the threshold. They leave the slice
  // paths (lane masked, slice narrowed to its widest remaining lane) and are
  // computed whole by warps (include/ehyb_b200.h, "long rows").
  const int64_t long_w = std::max<int64_t>(1, int64_t(env_double("EHYB_LONG_ROW", 128.0)));
  std::vector<int64_t> long_rows;
  std::unordered_map<int64_t, int64_t> long_er;  // row -> ER row j
  for (int64_t r = row_lo; r < row_hi; ++r)
    if (m->ell_row_widths[r] > long_w) long_rows.push_back(r);
  for (int64_t j = 0; j < m->n_er_rows; ++j) {
    const int64_t r = m->y_idx_er[j];
    if (r < row_lo || r >= row_hi) continue;
    if (m->er_row_widths[j] > long_w || m->ell_row_widths[r] > long_w) {
      if (m->er_row_widths[j] > long_w && m->ell_row_widths[r] <= long_w) long_rows.push_back(r);
      long_er[r] = j;
    }
  }
  std::sort(long_rows.begin(), long_rows.end());
  std::vector<uint32_t> lbits(size_t((h->local_rows + 31) / 32) + 1, 0u);
  int64_t max_chunk_bytes = 0;  // widest ELL slice (after long rows), ring sizing
  for (int64_t r : long_rows) lbits[size_t((r - row_lo) >> 5)] |= 1u << ((r - row_lo) & 31);
  std::vector<int32_t> eff(static_cast<size_t>(s_hi - s_lo));
  {
    for (int64_t s = s_lo; s < s_hi; ++s) {
      const int32_t W = m->width_ell[s];
      int32_t wmax = 0;
      bool has_long = false;
      for (int64_t r = s * C; r < (s + 1) * C; ++r) {
        const int64_t lr = r - row_lo;
        if ((lbits[size_t(lr >> 5)] >> (lr & 31)) & 1u) has_long = true;
        else wmax = std::max<int32_t>(wmax, m->ell_row_widths[r]);
      }
      int32_t e = has_long ? wmax : W;
      if (e > kEffWidth) return fail("ELL slice width exceeds the device limit");
      if (has_long) e |= kEffHasLong | (wmax < W ? kEffPadTail : 0);
      eff[size_t(s - s_lo)] = e;
      max_chunk_bytes = std::max<int64_t>(
          max_chunk_bytes, (int64_t(e & kEffWidth) * int64_t(C) * int64_t(tb + 2) + 127) / 128 * 128);
    }
  }
  CUDA_TRY(upload(&h->long_bits, lbits.data(), lbits.size() * 4, &h->bytes));

  // ---- ELL slab. C == 32: each slice is re-laid so a lane's 4 consecutive k
  // are contiguous (one 128-bit value load per 4 (fp32) or 2 (fp64) entries,
  // one 64-bit load per 4 columns; the W % 4 tail keeps the SELL layout).
  // Same slots, same per-slice positions; slices narrowed by a long row keep
  // the reference layout. A derived device layout, never a parity object.
  // default: fp32 slabs interleaved (4-byte values and 2-byte columns fetch 128 /
  // 64 B per warp instruction in the SELL layout, below the rate the HBM
  // stream needs: profiles/stream_probe_r2.txt; cfg3 fp32 114.9 vs 119.2 us),
  // fp64 interleaved when one wave of CTAs covers the partitions (cfg2 104.3
  // vs 106.5 us) and in the reference's SELL layout for persistent CTAs (cfg5
  // 963 vs 990 us)
  int sms = 0;
  CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  const bool one_wave = (p1 - p0) <= int64_t(sms);  // one CTA per SM covers every partition
  h->ell_vec = C == 32 && env_double("EHYB_VEC", (tb == 4 || one_wave) ? 1.0 : 0.0) != 0.0 &&
               env_double("EHYB_RING", 0.0) == 0.0;
  if (h->ell_vec) {
    std::vector<char> pv(size_t(std::max<int64_t>(slots, 1)) * tb);
    std::vector<uint16_t> pc(size_t(std::max<int64_t>(slots, 1)));
    const char* sv = static_cast<const char*>(m->val_ell) + size_t(base) * tb;
    const uint16_t* sc = m->col_ell + base;
#pragma omp parallel for schedule(dynamic, 256)
    for (int64_t s = s_lo; s < s_hi; ++s) {
      const int64_t p0 = pos[size_t(s - s_lo)];
      const int64_t W = m->width_ell[s];
      const bool keep = (eff[size_t(s - s_lo)] & kEffHasLong) != 0;
      const int64_t nb = W / 4;
      for (int64_t k = 0; k < W; ++k)
        for (int64_t lane = 0; lane < 32; ++lane) {
          const int64_t src = p0 + lane + 32 * k;
          const int64_t dst = keep ? src
                                   : p0 + (k < 4 * nb ? (k / 4) * 128 + lane * 4 + (k % 4)
                                                      : 128 * nb + (k - 4 * nb) * 32 + lane);
          std::memcpy(&pv[size_t(dst) * tb], sv + size_t(src) * tb, tb);
          pc[size_t(dst)] = sc[src];
        }
    }
    CUDA_TRY(upload(&h->val_ell, pv.data(), size_t(slots) * tb, &h->bytes));
    CUDA_TRY(upload(&h->col_ell, pc.data(), size_t(slots) * 2, &h->bytes));
  } else {
    CUDA_TRY(upload(&h->val_ell, static_cast<const char*>(m->val_ell) + size_t(base) * tb,
                    size_t(slots) * tb, &h->bytes));
    CUDA_TRY(upload(&h->col_ell, m->col_ell + base, size_t(slots) * 2, &h->bytes));
  }

  // ---- ER regrouped per owning partition
  const int64_t n_loc_parts = p1 - p0;
  // shards: rows with a column outside the shard ("halo rows") form their own
  // slices, run by the halo launch after the exchange; all other ER rows run
  // in the first launch together with ELL
  std::vector<std::vector<int64_t>> members(static_cast<size_t>(n_loc_parts)),
      hmembers(static_cast<size_t>(n_loc_parts));
  for (int64_t j = 0; j < m->n_er_rows; ++j) {
    const int64_t r = m->y_idx_er[j];
    if (r < row_lo || r >= row_hi || ((lbits[size_t((r - row_lo) >> 5)] >> ((r - row_lo) & 31)) & 1u))
      continue;
    bool halo = false;
    if (shard) {
      const int64_t src0 = int64_t(m->position_er[j / C]) + j % C;
      for (int64_t k = 0; k < m->er_row_widths[j] && !halo; ++k) {
        const int64_t c = m->col_er[src0 + C * k];
        halo = c < row_lo || c >= row_hi;
      }
    }
    (halo ? hmembers : members)[size_t(r / vec - p0)].push_back(j);
  }
  // slices holding an ER row publish their completion (the ER add waits on
  // it); the others skip the fence and the shared-memory atomic (C == 32)
  if (C == 32) {
    for (const auto* grp : {&members, &hmembers})
      for (const auto& mem : *grp)
        for (int64_t j : mem) eff[size_t((m->y_idx_er[j] - row_lo) / C)] |= kEffHasEr;
  } else {
    for (auto& e : eff) e |= kEffHasEr;
  }
  CUDA_TRY(upload(&h->width_ell, eff.data(), eff.size() * 4, &h->bytes));
  std::unordered_map<int64_t, int64_t> halo_index;
  halo_index.reserve(size_t(n_halo) * 2 + 1);
  for (int64_t i = 0; i < n_halo; ++i) halo_index[halo_cols[i]] = h->local_rows + i;
  // the ER padding column: what the reference's padding slots hold (global
  // column 0, format.py:379-380; a renumbered shard layout moves it). A
  // handle that owns it multiplies it inline (kPadFlag); a shard that does
  // not reads it from its halo in the fix-up pass after the ER phase
  int64_t pad_col = -1;
  for (int64_t j = 0; j < m->n_er_rows; ++j)
    if (m->er_row_widths[j] < m->width_er[j / C]) {
      pad_col = m->col_er[int64_t(m->position_er[j / C]) + j % C + C * int64_t(m->er_row_widths[j])];
      break;
    }
  const bool pad_local = pad_col < 0 || (pad_col >= row_lo && pad_col < row_hi);
  std::vector<int32_t> padfix;
  if (pad_col >= 0) {
    if (pad_local) {
      h->er_pad_idx = pad_col - row_lo;
    } else {
      auto it = halo_index.find(pad_col);
      h->er_pad_idx = it == halo_index.end() ? -1 : it->second;
    }
  }
  // launch configuration first: the ER pool is only safe when every CTA of
  // the grid is resident at once (pool rows wait on other CTAs' ELL chunks)
  int optin = 0;
  CUDA_TRY(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
  CUDA_TRY(cudaDeviceGetAttribute(&h->sm_count, cudaDevAttrMultiProcessorCount, device));
  const size_t win = size_t(vec) * tb;
  const size_t win_al = (win + 127) / 128 * 128;
  constexpr size_t kStaticReserve = 2048;  // mbarrier, counters, done bitmaps
  h->window_in_smem = win_al + kStaticReserve <= size_t(optin);
  h->win_bytes = h->window_in_smem ? win_al : 0;
  h->window_tma = h->window_in_smem && (win % 16 == 0);  // TMA needs 16 B multiples
  h->er_buf_offset = int(h->win_bytes);
  const size_t buf_slot = size_t(tb);  // own-ER buffer: one sum per buffered row
  h->er_buf_slices = int(std::min<size_t>(
      kMaxErBuf, (size_t(optin) - h->win_bytes - kStaticReserve) / (32 * buf_slot)));
  h->smem = h->win_bytes + size_t(h->er_buf_slices) * 32 * buf_slot;
  const int64_t chunks = (vec + 31) / 32;
  // one warp per chunk up to 1024 threads, plus the ring producer warp
  h->threads = int(std::min<int64_t>(max_threads_for(int(tb)), std::max<int64_t>(64, chunks * 32 + 32)));
  int per_sm = 0;
  CUDA_TRY(occupancy(h.get(), &per_sm));
  h->max_ctas = std::max<int64_t>(1, int64_t(per_sm) * h->sm_count);
  h->cooperative = env_double("EHYB_COOPERATIVE", 1.0) != 0.0;
  h->spin_timeout_ns = (unsigned long long)(env_double("EHYB_SPIN_TIMEOUT_S", 20.0) * 1e9);
  // the launch never exceeds one resident wave, so pooled rows (which wait on
  // other CTAs' ELL publication) cannot deadlock
  const bool pool_ok = true;

  // work units: a shard with fewer partitions than resident CTAs (a rank that
  // owns 74 of cfg5's 592 partitions on 148 SMs) splits each partition's
  // 32-row chunks into `split` contiguous units, one CTA each; every unit
  // stages the partition's window (SURVEY.md 8e option (i): the structure
  // stays that of the 1-GPU profile at every GPU count)
  int64_t split = 1;
  if (C == 32 && env_double("EHYB_RING", 0.0) == 0.0) {
    const double forced = env_double("EHYB_SPLIT", 0.0);
    if (forced >= 1.0) split = int64_t(forced);
    else if (n_loc_parts < h->max_ctas)
      split = std::min<int64_t>(std::min<int64_t>(4, h->max_ctas / n_loc_parts), chunks / 8);
    split = std::max<int64_t>(1, std::min<int64_t>(split, chunks));
  }
  const int64_t unit_chunks = (chunks + split - 1) / split;
  split = (chunks + unit_chunks - 1) / unit_chunks;  // no empty unit
  h->split = int32_t(split);
  h->unit_chunks = int32_t(unit_chunks);
  const int64_t n_units = n_loc_parts * split;
  h->n_units = n_units;
  if (split > 1) {  // regroup the per-partition ER members by unit (order kept)
    auto unit_of = [&](int64_t lr) {
      const int64_t q = lr / vec;
      return q * split + std::min<int64_t>(((lr - q * vec) >> 5) / unit_chunks, split - 1);
    };
    for (auto* grp : {&members, &hmembers}) {
      std::vector<std::vector<int64_t>> by_unit(static_cast<size_t>(n_units));
      for (const auto& mem : *grp)
        for (int64_t j : mem) by_unit[size_t(unit_of(m->y_idx_er[j] - row_lo))].push_back(j);
      grp->swap(by_unit);
    }
  }

  // persistent launches (more units than resident CTAs, one unit per
  // partition), EHYB_ORDER_UNITS=1: units run in decreasing modelled cost
  // (ELL slots + er_cost * ER entries), so the last iteration holds the
  // lightest partitions. A derived launch order only (rows, x and y keep the
  // reference layout; bitwise the same y). Measured off by default
  // (profiles/ab_order_r3.jsonl: cfg3 fp64 172.0 vs 172.2 us, cfg5 978 vs 967)
  std::vector<int32_t> upart;
  if (split == 1 && C == 32 && n_units > h->max_ctas && env_double("EHYB_ORDER_UNITS", 0.0) != 0.0) {
    const double ec = env_double("EHYB_ER_COST", 5.0);
    std::vector<double> cost(static_cast<size_t>(n_units), 0.0);
    for (int64_t q = 0; q < n_units; ++q) {
      const int64_t a = (q * vec) / C, b = ((q + 1) * vec) / C;
      cost[size_t(q)] = double(pos[size_t(b)] - pos[size_t(a)]);
      for (int64_t j : members[size_t(q)]) cost[size_t(q)] += ec * m->er_row_widths[j];
    }
    upart.resize(static_cast<size_t>(n_units));
    for (int64_t q = 0; q < n_units; ++q) upart[size_t(q)] = int32_t(q);
    std::stable_sort(upart.begin(), upart.end(),
                     [&](int32_t a, int32_t b) { return cost[size_t(a)] > cost[size_t(b)]; });
    for (auto* grp : {&members, &hmembers}) {
      std::vector<std::vector<int64_t>> by_unit(static_cast<size_t>(n_units));
      for (int64_t u = 0; u < n_units; ++u) by_unit[size_t(u)].swap((*grp)[size_t(upart[size_t(u)])]);
      grp->swap(by_unit);
    }
    std::vector<int32_t> pu(static_cast<size_t>(n_units));
    for (int64_t u = 0; u < n_units; ++u) pu[size_t(upart[size_t(u)])] = int32_t(u);
    CUDA_TRY(upload(&h->unit_part, upart.data(), upart.size() * 4, &h->bytes));
    CUDA_TRY(upload(&h->part_unit, pu.data(), pu.size() * 4, &h->bytes));
  }

  // per-partition 32-row ER slices (members in reference order), then the
  // own / pool split: partition q keeps the prefix of its ER slices that fits
  // its share of the mean per-CTA cost (ELL slots + er_cost * ER entries);
  // the rest joins a pool any CTA may claim once its own work is done
  // small partitions (at most two ELL chunks per warp, e.g. cfg1): the pool's
  // extra round trips cost more than the balance it buys; more ER-first
  // warps and no claim-ahead (profiles/sweep_r2_small_cfg1.txt)
  const bool small = chunks <= 2 * int64_t(h->threads / 32);
  if (tb == 4) h->ell_ahead = h->er_ahead = 0;  // fp32: measured 1.5% better without
  if (small) {
    h->er_warps = h->threads / 64;  // half the warps (16 of 32 at 1024 threads)
    h->ell_ahead = h->er_ahead = 0;
  }
  if (const double a = env_double("EHYB_CLAIM_AHEAD", -1.0); a >= 0.0) {  // dev override
    h->ell_ahead = int(a) & 1;
    h->er_ahead = (int(a) >> 1) & 1;
  }
  h->pf_ell = int(env_double("EHYB_PF_ELL", double(h->pf_ell)));
  const double pool_factor = env_double("EHYB_POOL_FACTOR", small ? 1e30 : 0.9);
  const double er_cost = env_double("EHYB_ER_COST", 5.0);
  std::vector<double> ell_cost(static_cast<size_t>(n_units)), er_total(static_cast<size_t>(n_units), 0.0);
  double total = 0.0;
  for (int64_t q = 0; q < n_units; ++q) {
    const int64_t qp = upart.empty() ? q / split : int64_t(upart[size_t(q)]),
                  c0 = (q % split) * unit_chunks;
    const int64_t a = (qp * vec) / C + c0 * (32 / C),
                  b = std::min<int64_t>(((qp + 1) * vec) / C, a + unit_chunks * (32 / C));
    ell_cost[size_t(q)] = double(pos[size_t(b)] - pos[size_t(a)]);
    for (int64_t j : members[size_t(q)]) er_total[size_t(q)] += er_cost * m->er_row_widths[j];
    total += ell_cost[size_t(q)] + er_total[size_t(q)];
  }
  const double budget_mean = n_units ? total / double(n_units) : 0.0;
  // ER-heavy matrices (ER > 40% of the modelled work): ER-first warps in
  // proportion to the ER share, so more of the latency-bound ER chains run
  // under the stream (profiles/ab_erw_r3.jsonl: cfg4, share 0.55, 69.2 us at
  // 6 warps -> 60.7 / 59.9 us at 12 / 14 of 24; below the threshold the
  // measured optimum stays 6: cfg2 (0.32) 100.4 us at 6 vs 100.7 at 8, cfg3
  // and cfg5 flat)
  if (!small && total > 0.0) {
    double er_sum = 0.0;
    for (double v : er_total) er_sum += v;
    const double share = er_sum / total;
    const int nw = h->threads / 32;
    if (share > 0.4)
      h->er_warps = std::max(h->er_warps, std::min(int(std::lround(double(nw) * share)), nw - 8));
  }
  h->er_warps = int(env_double("EHYB_ER_WARPS", double(h->er_warps)));  // dev override
  struct SliceRef { int64_t q, i0; bool halo; };
  std::vector<std::vector<SliceRef>> own(static_cast<size_t>(n_units)), spill(static_cast<size_t>(n_units));
  // persistent CTAs: units of the last iteration may keep a different share
  // (their pooled slices can only be finished after the loop)
  const int64_t last_it0 = n_units > h->max_ctas ? (n_units - 1) / h->max_ctas * h->max_ctas : n_units;
  const double pool_factor_last = env_double("EHYB_POOL_FACTOR_LAST", pool_factor);
  for (int64_t q = 0; q < n_units; ++q) {
    const auto& mem = members[size_t(q)];
    const double pf = q >= last_it0 ? pool_factor_last : pool_factor;
    double left = (pool_ok && pf > 0.0) ? pf * budget_mean - ell_cost[size_t(q)] : 1e300;
    bool spilling = false;
    for (size_t i0 = 0; i0 < mem.size(); i0 += 32) {
      double c = 0.0;
      for (size_t i = i0; i < std::min(mem.size(), i0 + 32); ++i) c += er_cost * m->er_row_widths[mem[i]];
      if (!spilling && c <= left) {
        left -= c;
        own[size_t(q)].push_back({q, int64_t(i0), false});
      } else {
        spilling = true;
        spill[size_t(q)].push_back({q, int64_t(i0), false});
      }
    }
  }
  std::vector<int32_t> part_ptr(size_t(n_units) + 1, 0), part_mid(static_cast<size_t>(n_units), 0);
  std::vector<SliceRef> order;
  for (int64_t q = 0; q < n_units; ++q) {
    for (const auto& r : own[size_t(q)]) order.push_back(r);
    part_mid[size_t(q)] = int32_t(order.size());
    for (size_t i0 = 0; i0 < hmembers[size_t(q)].size(); i0 += 32) order.push_back({q, int64_t(i0), true});
    part_ptr[size_t(q) + 1] = int32_t(order.size());
  }
  h->pool_lo = int64_t(order.size());
  for (size_t round = 0;; ++round) {  // pool: round-robin over the heavy partitions
    bool any = false;
    for (int64_t q = 0; q < n_units; ++q)
      if (round < spill[size_t(q)].size()) {
        order.push_back(spill[size_t(q)][round]);
        any = true;
      }
    if (!any) break;
  }
  h->pool_hi = int64_t(order.size());
  // several partitions per CTA: the pool is reordered (stable) into groups by
  // the iteration in which the owner partition runs on its CTA (q / grid)
  std::vector<int32_t> pool_gptr;
  bool own_scratch = false;
  if (n_units > h->max_ctas && h->pool_hi > h->pool_lo &&
      env_double("EHYB_POOL_DIRECT", 1.0) != 0.0) {
    const int64_t grid = h->max_ctas;
    const int64_t ng = (n_units + grid - 1) / grid;
    std::stable_sort(order.begin() + h->pool_lo, order.end(),
                     [&](const SliceRef& a, const SliceRef& b) { return a.q / grid < b.q / grid; });
    pool_gptr.assign(static_cast<size_t>(ng) + 1, 0);
    for (int64_t i = h->pool_lo; i < h->pool_hi; ++i) pool_gptr[size_t(order[size_t(i)].q / grid) + 1] += 1;
    pool_gptr[0] = int32_t(h->pool_lo);
    for (int64_t g = 0; g < ng; ++g) pool_gptr[size_t(g) + 1] += pool_gptr[size_t(g)];
  }
  {
    int64_t max_own = 0;
    for (int64_t q = 0; q < n_units; ++q) max_own = std::max<int64_t>(max_own, int64_t(own[size_t(q)].size()));
    h->er_buf_slices = int(std::min<int64_t>(h->er_buf_slices, max_own));
    // partitions with more own ER slices than the shared-memory buffer holds
    // (large windows, e.g. cfg5) spill the rest to a global scratch, so the
    // ER-first warps still finish them during the ELL phase
    own_scratch = max_own > h->er_buf_slices && env_double("EHYB_OWN_SCRATCH", 0.0) != 0.0;
    h->smem = h->win_bytes + size_t(h->er_buf_slices) * 32 * buf_slot;
    // ELL ring (C == 32, TMA-staged window): shared memory left after the
    // window, at least 2 chunks of the widest slice; the own-ER buffer gives
    // way so the ring keeps >= EHYB_RING_KB (default 64 KB)
    h->ring_bytes = 0;
#ifdef EHYB_DEV_ONE
    if (false) {
#else
    if (C == 32 && h->window_tma && env_double("EHYB_RING", 0.0) != 0.0) {
#endif
      cudaFuncAttributes fa{};
      if (tb == 4)
        CUDA_TRY(cudaFuncGetAttributes(&fa, spmv_fused_kernel<float, EHYB_MODE_STRICT, true, true, true>));
      else
        CUDA_TRY(cudaFuncGetAttributes(&fa, spmv_fused_kernel<double, EHYB_MODE_STRICT, true, true, true>));
      const int64_t dyn = int64_t(optin) - int64_t(fa.sharedSizeBytes) - 256;
      const int64_t avail = dyn - int64_t(h->win_bytes);
      const int64_t want = std::max<int64_t>(2 * max_chunk_bytes,
                                             int64_t(env_double("EHYB_RING_KB", 64.0) * 1024.0));
      if (avail >= 2 * max_chunk_bytes && avail >= 16 * 1024) {
        int64_t buf = int64_t(h->er_buf_slices) * 32 * int64_t(buf_slot);
        if (avail - buf < want) buf = std::max<int64_t>(0, avail - want);
        h->er_buf_slices = int(buf / (32 * int64_t(buf_slot)));
        buf = int64_t(h->er_buf_slices) * 32 * int64_t(buf_slot);
        h->ring_offset = (size_t(h->win_bytes) + size_t(buf) + 127) / 128 * 128;
        const int64_t total = (dyn - int64_t(h->ring_offset)) / 128 * 128;
        // stages of ~EHYB_STAGE_KB (default 16 KB), 2..kRingNS-1 of them; each
        // region must hold the widest chunk
        const int64_t target = int64_t(env_double("EHYB_STAGE_KB", 16.0) * 1024.0);
        int64_t ns = std::min<int64_t>(kRingNS - 1, std::max<int64_t>(2, total / std::max<int64_t>(target, 1)));
        int64_t sb = total / ns / 128 * 128;
        int64_t svb = sb * int64_t(tb) / int64_t(tb + 2) / 128 * 128;
        const int64_t wmax = max_chunk_bytes / (32 * int64_t(tb + 2)) + 1;
        if (ns >= 2 && svb >= 32 * wmax * int64_t(tb) && sb - svb >= 64 * wmax) {
          h->ring_stages = int(ns);
          h->stage_bytes = int(sb);
          h->stage_vbytes = int(svb);
          h->ring_bytes = size_t(ns * sb);
        }
        h->smem = h->win_bytes + size_t(buf);
      }
    }
    // per-unit chunk metadata {pos, eff} in shared memory after the own-ER
    // buffer (32-row slices, staged window, no ring) when it fits the
    // per-CTA budget the grid was sized for
    // measured (profiles/ab_meta_r3.jsonl): fp32 (no claim-ahead) 114.7 ->
    // 112.7 us on cfg3; persistent fp64 180.0 -> 176.5 us on cfg3 fp64; the
    // one-wave fp64 path already hides the metadata behind its claim-ahead
    // (cfg2 100.5 vs 102.5 us with it), so it keeps the global loads
    h->meta_off = -1;
    const bool meta_default = tb == 4 || n_units > h->max_ctas;
    if (C == 32 && h->window_in_smem && h->ring_bytes == 0 &&
        env_double("EHYB_META_SMEM", meta_default ? 1.0 : 0.0) != 0.0) {
      const size_t off = (h->smem + 15) / 16 * 16;
      const size_t bytes = size_t(unit_chunks) * 8;
      if (off + bytes + kStaticReserve <= size_t(optin)) {
        h->meta_off = int32_t(off);
        h->smem = off + bytes;
      }
    }
    if (h->ring_stages > 0) {
      // stage plan: runs of consecutive chunks whose slab slots fit a stage's
      // value and column regions; a slice narrowed by a long row ends its stage
      // (its long lane's slots beyond the narrowed width are not copied)
      const int64_t cpp = vec / 32;  // chunks per partition
      const int64_t svb = h->stage_vbytes, scb = int64_t(h->stage_bytes) - h->stage_vbytes;
      std::vector<int32_t> sptr(static_cast<size_t>(n_loc_parts) + 1, 0), spos, sslots, schunks;
      std::vector<uint2> chs(static_cast<size_t>(n_loc_parts * cpp));
      for (int64_t q = 0; q < n_loc_parts; ++q) {
        sptr[size_t(q)] = int32_t(spos.size());
        bool open = false;
        int32_t cur_pos = 0, cur_slots = 0, cur_n = 0;
        auto close = [&]() {
          if (!open) return;
          spos.push_back(cur_pos);
          sslots.push_back(cur_slots);
          schunks.push_back(cur_n);
          open = false;
        };
        for (int64_t c = 0; c < cpp; ++c) {
          const int64_t sl = q * cpp + c;
          const int32_t e = eff[size_t(sl)];
          const int64_t w = e & kEffWidth;
          const int32_t p = pos[size_t(sl)];
          int64_t rel = open ? int64_t(p) - cur_pos : 0;
          if (open && ((rel + 32 * w) * int64_t(tb) > svb || (rel + 32 * w) * 2 > scb || cur_n >= 64)) {
            close();
            rel = 0;
          }
          if (!open) {
            open = true;
            cur_pos = p;
            cur_n = 0;
          }
          chs[size_t(sl)] = make_uint2(uint32_t(int64_t(spos.size()) - sptr[size_t(q)]), uint32_t(rel));
          cur_slots = int32_t(rel + 32 * w);
          ++cur_n;
          if (e & kEffHasLong) close();
        }
        close();
      }
      sptr[size_t(n_loc_parts)] = int32_t(spos.size());
      CUDA_TRY(upload(&h->part_stage_ptr, sptr.data(), sptr.size() * 4, &h->bytes));
      CUDA_TRY(upload(&h->st_pos, spos.data(), spos.size() * 4, &h->bytes));
      CUDA_TRY(upload(&h->st_slots, sslots.data(), sslots.size() * 4, &h->bytes));
      CUDA_TRY(upload(&h->st_chunks, schunks.data(), schunks.size() * 4, &h->bytes));
      CUDA_TRY(upload(&h->ch_stage, chs.data(), chs.size() * 8, &h->bytes));
    }
  }
  const int64_t n_sl = int64_t(order.size());
  std::vector<int64_t> epos(size_t(n_sl) + 1, 0);
  std::vector<int32_t> eswidth(size_t(n_sl), 0), erows(size_t(n_sl) * 32, -1),
      elwidth(size_t(n_sl) * 32, 0);
  for (int64_t sl = 0; sl < n_sl; ++sl) {
    const auto& ref = order[size_t(sl)];
    const auto& mem = ref.halo ? hmembers[size_t(ref.q)] : members[size_t(ref.q)];
    for (int64_t i = ref.i0; i < std::min<int64_t>(int64_t(mem.size()), ref.i0 + 32); ++i) {
      const int64_t j = mem[size_t(i)];
      const int32_t w = m->er_row_widths[j];
      const int64_t ref_w = m->width_er[j / C];
      const int64_t lr = m->y_idx_er[j] - row_lo;
      int32_t row = int32_t(lr);
      if (w < ref_w) {
        if (pad_local) row |= kPadFlag;
        else padfix.push_back(int32_t(lr));
      }
      erows[size_t(sl) * 32 + (i - ref.i0)] = row;
      elwidth[size_t(sl) * 32 + (i - ref.i0)] = w;
      eswidth[size_t(sl)] = std::max(eswidth[size_t(sl)], w);
    }
  }
  for (int64_t s = 0; s < n_sl; ++s) epos[size_t(s) + 1] = epos[size_t(s)] + 32 * int64_t(eswidth[size_t(s)]);
  const int64_t eslots = epos[size_t(n_sl)];
  std::vector<char> evals(size_t(std::max<int64_t>(eslots, 1)) * tb, 0);
  std::vector<uint32_t> ecols(size_t(std::max<int64_t>(eslots, 1)), 0);
  for (int64_t sl = 0; sl < n_sl; ++sl) {
    const auto& ref = order[size_t(sl)];
    const auto& mem = ref.halo ? hmembers[size_t(ref.q)] : members[size_t(ref.q)];
    for (int64_t i = ref.i0; i < std::min<int64_t>(int64_t(mem.size()), ref.i0 + 32); ++i) {
      const int64_t j = mem[size_t(i)];
      const int64_t w = m->er_row_widths[j];
      const int64_t src0 = int64_t(m->position_er[j / C]) + j % C;
      const int64_t dst0 = epos[size_t(sl)] + (i - ref.i0);
      for (int64_t k = 0; k < w; ++k) {
        const int64_t src = src0 + k * C, dst = dst0 + k * 32;
        std::memcpy(&evals[size_t(dst) * tb], static_cast<const char*>(m->val_er) + size_t(src) * tb, tb);
        const int64_t c = m->col_er[src];
        int64_t lc;
        if (c >= row_lo && c < row_hi) {
          lc = c - row_lo;
        } else {
          auto it = halo_index.find(c);
          if (it == halo_index.end()) return fail("ER column missing from the shard halo plan");
          lc = it->second;
        }
        ecols[size_t(dst)] = uint32_t(lc);
      }
    }
  }
  h->er_slices = n_sl;
  h->er_slots = eslots;
  if (own_scratch) {
    CUDA_TRY(cudaMalloc(&h->own_acc, size_t(std::max<int64_t>(n_sl, 1)) * 32 * tb));
    h->bytes += size_t(std::max<int64_t>(n_sl, 1)) * 32 * tb;
  }
  CUDA_TRY(upload(&h->er_part_ptr, part_ptr.data(), part_ptr.size() * 4, &h->bytes));
  CUDA_TRY(upload(&h->er_part_mid, part_mid.data(), part_mid.size() * 4, &h->bytes));
  CUDA_TRY(upload(&h->er_pos, epos.data(), epos.size() * 8, &h->bytes));
  CUDA_TRY(upload(&h->er_swidth, eswidth.data(), eswidth.size() * 4, &h->bytes));
  CUDA_TRY(upload(&h->er_rows, erows.data(), erows.size() * 4, &h->bytes));
  CUDA_TRY(upload(&h->er_lwidth, elwidth.data(), elwidth.size() * 4, &h->bytes));
  CUDA_TRY(upload(&h->er_val, evals.data(), size_t(eslots) * tb, &h->bytes));
  CUDA_TRY(upload(&h->er_col, ecols.data(), size_t(eslots) * 4, &h->bytes));

  // ---- long-row tasks: entries in the reference's k order with x indices
  // (ELL window columns made shard-local), longest first; FMA-mode segments
  if (!long_rows.empty()) {
    struct Task { int64_t row, n_ell, n_er; };
    std::vector<Task> tasks;
    for (int64_t r : long_rows) {
      auto it = long_er.find(r);
      tasks.push_back({r, m->ell_row_widths[r], it == long_er.end() ? 0 : m->er_row_widths[it->second]});
    }
    std::stable_sort(tasks.begin(), tasks.end(), [](const Task& a, const Task& b) {
      return a.n_ell + a.n_er > b.n_ell + b.n_er;
    });
    const int64_t n_t = int64_t(tasks.size());
    const int64_t seg_len = std::max<int64_t>(256, int64_t(env_double("EHYB_LONG_SEG", 4096.0)));
    std::vector<int64_t> span(static_cast<size_t>(3 * n_t)), padcol(static_cast<size_t>(n_t)), seg;
    std::vector<int32_t> lrow(static_cast<size_t>(n_t)), tseg(static_cast<size_t>(n_t) + 1, 0),
        tnell(static_cast<size_t>(n_t), 0);
    int64_t total = 0;
    for (const auto& t : tasks) total += t.n_ell + t.n_er;
    std::vector<char> lval(size_t(std::max<int64_t>(total, 1)) * tb, 0);
    std::vector<uint32_t> lcol(size_t(std::max<int64_t>(total, 1)), 0);
    int64_t at = 0;
    for (int64_t i = 0; i < n_t; ++i) {
      const auto& t = tasks[size_t(i)];
      const int64_t r = t.row, s = r / C, lane = r % C;
      const int64_t win0 = (r / vec) * vec - row_lo;  // shard-local index of window column 0
      span[size_t(3 * i)] = at;
      for (int64_t k = 0; k < t.n_ell; ++k, ++at) {
        const int64_t src = int64_t(m->position_ell[s]) + lane + C * k;
        std::memcpy(&lval[size_t(at) * tb], static_cast<const char*>(m->val_ell) + size_t(src) * tb, tb);
        lcol[size_t(at)] = uint32_t(win0 + m->col_ell[src]);
      }
      span[size_t(3 * i + 1)] = at;
      int32_t flags = 0;
      if (t.n_ell < m->width_ell[s]) flags |= kLrEllPad;
      padcol[size_t(i)] = win0;
      if (auto it = long_er.find(r); it != long_er.end()) {
        const int64_t j = it->second;
        flags |= kLrHasEr;
        if (t.n_er < m->width_er[j / C]) {
          if (pad_local) flags |= kLrErPad;
          else padfix.push_back(int32_t(r - row_lo));
        }
        const int64_t src0 = int64_t(m->position_er[j / C]) + j % C;
        for (int64_t k = 0; k < t.n_er; ++k, ++at) {
          const int64_t src = src0 + C * k;
          std::memcpy(&lval[size_t(at) * tb], static_cast<const char*>(m->val_er) + size_t(src) * tb, tb);
          const int64_t c = m->col_er[src];
          int64_t lc;
          if (c >= row_lo && c < row_hi) {
            lc = c - row_lo;
          } else {
            auto hit = halo_index.find(c);
            if (hit == halo_index.end()) return fail("ER column missing from the shard halo plan");
            lc = hit->second;
          }
          lcol[size_t(at)] = uint32_t(lc);
        }
      }
      span[size_t(3 * i + 2)] = at;
      lrow[size_t(i)] = int32_t(r - row_lo) | flags;
      tseg[size_t(i)] = int32_t(seg.size() / 3);
      for (int part_i = 0; part_i < 2; ++part_i) {
        const int64_t lo = span[size_t(3 * i + part_i)], hi = span[size_t(3 * i + part_i + 1)];
        for (int64_t a = lo; a < hi; a += seg_len) {
          seg.push_back(i);
          seg.push_back(a);
          seg.push_back(std::min(hi, a + seg_len));
          if (part_i == 0) tnell[size_t(i)] += 1;
        }
      }
    }
    tseg[size_t(n_t)] = int32_t(seg.size() / 3);
    h->lr_tasks = int32_t(n_t);
    h->lr_segs = int32_t(seg.size() / 3);
    CUDA_TRY(upload(&h->lr_span, span.data(), span.size() * 8, &h->bytes));
    CUDA_TRY(upload(&h->lr_row, lrow.data(), lrow.size() * 4, &h->bytes));
    CUDA_TRY(upload(&h->lr_padcol, padcol.data(), padcol.size() * 8, &h->bytes));
    CUDA_TRY(upload(&h->lr_val, lval.data(), size_t(total) * tb, &h->bytes));
    CUDA_TRY(upload(&h->lr_col, lcol.data(), size_t(total) * 4, &h->bytes));
    CUDA_TRY(upload(&h->lr_seg, seg.data(), seg.size() * 8, &h->bytes));
    CUDA_TRY(upload(&h->lr_task_seg, tseg.data(), tseg.size() * 4, &h->bytes));
    CUDA_TRY(upload(&h->lr_task_nell, tnell.data(), tnell.size() * 4, &h->bytes));
    CUDA_TRY(cudaMalloc(&h->lr_part, size_t(std::max<int32_t>(h->lr_segs, 1)) * tb));
    CUDA_TRY(cudaMalloc(&h->lr_cnt, size_t(n_t) * 4));
    CUDA_TRY(cudaMemset(h->lr_cnt, 0, size_t(n_t) * 4));
    CUDA_TRY(cudaMalloc(&h->lr_ctr, 16));
    CUDA_TRY(cudaMemset(h->lr_ctr, 0, 16));
    h->bytes += size_t(std::max<int32_t>(h->lr_segs, 1)) * tb + size_t(n_t) * 4 + 16;
  }

  if (!padfix.empty()) {
    if (h->er_pad_idx < 0) return fail("ER padding column missing from the shard halo plan");
    std::sort(padfix.begin(), padfix.end());
    h->padfix_n = int64_t(padfix.size());
    CUDA_TRY(upload(&h->padfix_rows, padfix.data(), padfix.size() * 4, &h->bytes));
  }

  // ---- permutation tables (int32) for the user-order entry points
  if (!shard) {
    std::vector<int32_t> ro(static_cast<size_t>(m->dimension)), inv(static_cast<size_t>(padded));
    for (int64_t i = 0; i < m->dimension; ++i) ro[size_t(i)] = int32_t(m->reorder[i]);
    for (int64_t i = 0; i < padded; ++i) inv[size_t(i)] = int32_t(m->inverse[i]);
    CUDA_TRY(upload(&h->reorder, ro.data(), ro.size() * 4, &h->bytes));
    CUDA_TRY(upload(&h->inverse, inv.data(), inv.size() * 4, &h->bytes));
  }

  // ---- launch epoch on the device (starts at 1; the kernel advances it)
  {
    const unsigned int init[2] = {1u, 0u};
    CUDA_TRY(upload(&h->epoch_dev, init, sizeof(init), &h->bytes));
  }
  // ---- ER pool state: claim counters, per-owner lists, scratch, counts
  if (h->pool_hi > h->pool_lo) {
    std::vector<int32_t> optr(static_cast<size_t>(n_units) + 1, 0), oidx;
    for (int64_t sl = h->pool_lo; sl < h->pool_hi; ++sl) optr[size_t(order[size_t(sl)].q) + 1] += 1;
    for (int64_t q = 0; q < n_units; ++q) optr[size_t(q) + 1] += optr[size_t(q)];
    oidx.resize(size_t(h->pool_hi - h->pool_lo));
    std::vector<int32_t> fill(optr.begin(), optr.end() - 1);
    for (int64_t sl = h->pool_lo; sl < h->pool_hi; ++sl)
      oidx[size_t(fill[size_t(order[size_t(sl)].q)]++)] = int32_t(sl);
    CUDA_TRY(upload(&h->pool_own_ptr, optr.data(), optr.size() * 4, &h->bytes));
    CUDA_TRY(upload(&h->pool_own_idx, oidx.data(), oidx.size() * 4, &h->bytes));
    // owner-major scratch: pooled slice s writes its sums at position pos[s]
    // of its owner's list; the owner reads rows and sums contiguously
    {
      std::vector<int32_t> ppos(oidx.size()), prow(oidx.size() * 32);
      for (size_t i = 0; i < oidx.size(); ++i) {
        const int64_t sl = oidx[i];
        ppos[size_t(sl - h->pool_lo)] = int32_t(i);
        std::memcpy(&prow[i * 32], &erows[size_t(sl) * 32], 32 * 4);
      }
      CUDA_TRY(upload(&h->pool_pos, ppos.data(), ppos.size() * 4, &h->bytes));
      CUDA_TRY(upload(&h->pool_rows, prow.data(), prow.size() * 4, &h->bytes));
    }
    const size_t acc_bytes = size_t(h->pool_hi - h->pool_lo) * 32 * tb;
    CUDA_TRY(cudaMalloc(&h->pool_acc, acc_bytes));
    CUDA_TRY(cudaMalloc(&h->pool_done, size_t(n_units) * 8 + 16));
    CUDA_TRY(cudaMemset(h->pool_done, 0, size_t(n_units) * 8 + 16));
    CUDA_TRY(cudaMalloc(&h->pool_ctr, 16));
    CUDA_TRY(cudaMemset(h->pool_ctr, 0, 16));
    h->bytes += acc_bytes + size_t(n_units) * 8 + 32;
    if (!pool_gptr.empty()) {
      const int64_t ng = int64_t(pool_gptr.size()) - 1;
      h->pool_groups = int32_t(ng);
      h->pool_last_scratch = ng > 1 && env_double("EHYB_POOL_LAST_SCRATCH", 0.0) != 0.0;
      CUDA_TRY(upload(&h->pool_grp, pool_gptr.data(), pool_gptr.size() * 4, &h->bytes));
      CUDA_TRY(cudaMalloc(&h->pool_gctr, size_t(ng) * 8 + 16));
      CUDA_TRY(cudaMemset(h->pool_gctr, 0, size_t(ng) * 8 + 16));
      CUDA_TRY(cudaMalloc(&h->part_flag, size_t(n_units) * 4 + 16));
      CUDA_TRY(cudaMemset(h->part_flag, 0, size_t(n_units) * 4 + 16));
      h->bytes += size_t(ng) * 12 + size_t(n_units) * 4 + 48;
    }
  }
  *out = h.release();
  return 0;
}

}  // namespace

extern "C" {

EHYB_API int ehyb_dev_create(const ehyb_host_matrix* m, int device, ehyb_dev** out) {
  EHYB_TRY {
    int rc = ehyb_check(m);
    if (rc) return rc;
    return create_impl(m, 0, m->n_parts, nullptr, 0, false, device, out);
  }
  EHYB_CATCH
}

EHYB_API int ehyb_dev_create_shard(const ehyb_host_matrix* m, const ehyb_shard_plan* plan,
                                   int device, ehyb_dev** out) {
  EHYB_TRY {
    if (!plan) return fail("null shard plan");
    int rc = ehyb_check(m);
    if (rc) return rc;
    return create_impl(m, plan->p0, plan->p1, plan->halo_cols, plan->n_halo, true, device, out);
  }
  EHYB_CATCH
}

EHYB_API int ehyb_dev_destroy(ehyb_dev* h) {
  if (!h) return 0;
  DeviceGuard guard(h->device);
  delete h;
  return 0;
}

EHYB_API int ehyb_dev_tune(ehyb_dev* h, int key, int64_t value) {
  if (!h) return fail("null handle");
  switch (key) {
    case EHYB_TUNE_PREFETCH_ELL: h->pf_ell = int(std::max<int64_t>(0, value)); return 0;
    case EHYB_TUNE_PREFETCH_ER: h->pf_er = value ? 1 : 0; return 0;
    case EHYB_TUNE_THREADS:
      if (value < 32 || value > max_threads_for(h->tau) || value % 32)
        return fail("threads must be a multiple of 32 in [32, " +
                    std::to_string(max_threads_for(h->tau)) + "]");
      h->threads = int(value);
      return 0;
    case EHYB_TUNE_ER_WARPS: h->er_warps = int(std::max<int64_t>(0, value)); return 0;
    case EHYB_TUNE_CLAIM_AHEAD:
      h->ell_ahead = int(value & 1);
      h->er_ahead = int((value >> 1) & 1);
      return 0;
    case EHYB_TUNE_PHASES: h->phase_skip = int(value & 3); return 0;
    case EHYB_TUNE_TIMING:
      h->timing = reinterpret_cast<unsigned long long*>(static_cast<uintptr_t>(value));
      return 0;
    default:
      return fail("unknown tuning key");
  }
}

EHYB_API int ehyb_dev_info_get(const ehyb_dev* h, ehyb_dev_info* out) {
  if (!h || !out) return fail("null argument");
  out->device_bytes = int64_t(h->bytes);
  out->er_slices = h->er_slices;
  out->er_slots = h->er_slots;
  out->window_bytes = h->vec * h->tau;
  out->window_in_smem = h->window_in_smem ? 1 : 0;
  out->threads_per_cta = h->threads;
  out->ctas = int32_t(std::min<int64_t>(h->n_units, h->max_ctas));
  out->work_units = h->n_units;
  out->split = h->split;
  out->reserved = 0;
  out->sm_count = h->sm_count;
  out->pool_slices = h->pool_hi - h->pool_lo;
  out->er_buf_slices = h->er_buf_slices;
  out->smem_bytes = int32_t(h->ring_bytes ? h->ring_offset + h->ring_bytes : h->smem);
  out->ring_bytes = int64_t(h->ring_bytes);
  out->long_rows = h->lr_tasks;
  return 0;
}

EHYB_API int ehyb_dev_spmv(ehyb_dev* h, const void* x_dev, void* y_dev, int mode, void* stream) {
  EHYB_TRY {
    if (!h || !x_dev || !y_dev) return fail("null argument");
    if (x_dev == y_dev) return fail("x and y must not alias");
    DeviceGuard guard(h->device);
    CUDA_TRY(launch_spmv(h, x_dev, y_dev, mode, true, true, static_cast<cudaStream_t>(stream)));
    return 0;
  }
  EHYB_CATCH
}

EHYB_API int ehyb_dev_spmv_ell(ehyb_dev* h, const void* x_ext, void* y_local, int mode,
                               void* stream) {
  EHYB_TRY {
    if (!h || !x_ext || !y_local) return fail("null argument");
    DeviceGuard guard(h->device);
    CUDA_TRY(launch_spmv(h, x_ext, y_local, mode, true, false, static_cast<cudaStream_t>(stream)));
    return 0;
  }
  EHYB_CATCH
}

EHYB_API int ehyb_dev_spmv_er(ehyb_dev* h, const void* x_ext, void* y_local, int mode,
                              void* stream) {
  EHYB_TRY {
    if (!h || !x_ext || !y_local) return fail("null argument");
    DeviceGuard guard(h->device);
    CUDA_TRY(launch_spmv(h, x_ext, y_local, mode, false, true, static_cast<cudaStream_t>(stream)));
    return 0;
  }
  EHYB_CATCH
}

EHYB_API int ehyb_dev_permute(ehyb_dev* h, const void* x_user, void* x_r, void* stream) {
  EHYB_TRY {
    if (!h || h->shard) return fail("permute needs a full-matrix handle");
    DeviceGuard guard(h->device);
    auto st = static_cast<cudaStream_t>(stream);
    const int g = grid_for(h->padded, 256, h->sm_count);
    if (h->tau == 4)
      permute_kernel<float><<<g, 256, 0, st>>>(static_cast<const float*>(x_user), h->inverse,
                                                h->dimension, h->padded, static_cast<float*>(x_r));
    else
      permute_kernel<double><<<g, 256, 0, st>>>(static_cast<const double*>(x_user), h->inverse,
                                                 h->dimension, h->padded, static_cast<double*>(x_r));
    CUDA_TRY(cudaGetLastError());
    return 0;
  }
  EHYB_CATCH
}

EHYB_API int ehyb_dev_unpermute(ehyb_dev* h, const void* y_r, void* y_user, void* stream) {
  EHYB_TRY {
    if (!h || h->shard) return fail("unpermute needs a full-matrix handle");
    DeviceGuard guard(h->device);
    auto st = static_cast<cudaStream_t>(stream);
    const int g = grid_for(h->dimension, 256, h->sm_count);
    if (h->tau == 4)
      unpermute_kernel<float><<<g, 256, 0, st>>>(static_cast<const float*>(y_r), h->reorder,
                                                  h->dimension, static_cast<float*>(y_user));
    else
      unpermute_kernel<double><<<g, 256, 0, st>>>(static_cast<const double*>(y_r), h->reorder,
                                                   h->dimension, static_cast<double*>(y_user));
    CUDA_TRY(cudaGetLastError());
    return 0;
  }
  EHYB_CATCH
}

static int ensure_scratch(ehyb_dev* h) {
  const size_t tb = size_t(h->tau);
  if (!h->xr) {
    CUDA_TRY(cudaMalloc(&h->xr, size_t(h->padded) * tb));
    CUDA_TRY(cudaMalloc(&h->yr, size_t(h->padded) * tb));
    CUDA_TRY(cudaMalloc(&h->xu, std::max<size_t>(size_t(h->dimension) * tb, 16)));
    CUDA_TRY(cudaMalloc(&h->yu, std::max<size_t>(size_t(h->dimension) * tb, 16)));
    h->bytes += 2 * size_t(h->padded) * tb + 2 * size_t(h->dimension) * tb;
  }
  return 0;
}

EHYB_API int ehyb_dev_spmv_user(ehyb_dev* h, const void* x_user, void* y_user, int mode,
                                void* stream) {
  EHYB_TRY {
    if (!h || h->shard) return fail("spmv_user needs a full-matrix handle");
    DeviceGuard guard(h->device);
    int rc = ensure_scratch(h);
    if (rc) return rc;
    rc = ehyb_dev_permute(h, x_user, h->xr, stream);
    if (rc) return rc;
    CUDA_TRY(launch_spmv(h, h->xr, h->yr, mode, true, true, static_cast<cudaStream_t>(stream)));
    return ehyb_dev_unpermute(h, h->yr, y_user, stream);
  }
  EHYB_CATCH
}

EHYB_API int ehyb_dev_spmv_host(ehyb_dev* h, const void* x_host, void* y_host, int user_order,
                                int mode, void* stream) {
  EHYB_TRY {
    if (!h || h->shard) return fail("spmv_host needs a full-matrix handle");
    DeviceGuard guard(h->device);
    int rc = ensure_scratch(h);
    if (rc) return rc;
    auto st = static_cast<cudaStream_t>(stream);
    const size_t tb = size_t(h->tau);
    if (user_order) {
      const size_t nb = size_t(h->dimension) * tb;
      CUDA_TRY(cudaMemcpyAsync(h->xu, x_host, nb, cudaMemcpyHostToDevice, st));
      rc = ehyb_dev_spmv_user(h, h->xu, h->yu, mode, stream);
      if (rc) return rc;
      CUDA_TRY(cudaMemcpyAsync(y_host, h->yu, nb, cudaMemcpyDeviceToHost, st));
    } else {
      const size_t pb = size_t(h->padded) * tb;
      CUDA_TRY(cudaMemcpyAsync(h->xr, x_host, pb, cudaMemcpyHostToDevice, st));
      CUDA_TRY(launch_spmv(h, h->xr, h->yr, mode, true, true, st));
      CUDA_TRY(cudaMemcpyAsync(y_host, h->yr, pb, cudaMemcpyDeviceToHost, st));
    }
    CUDA_TRY(cudaStreamSynchronize(st));
    return 0;
  }
  EHYB_CATCH
}

static int ensure_pipeline(ehyb_dev* h) {
  if (h->s_in) return 0;
  const size_t pb = size_t(h->padded) * size_t(h->tau);
  for (int b = 0; b < ehyb_dev::kPipe; ++b) {
    CUDA_TRY(cudaMalloc(&h->bx[b], pb));
    CUDA_TRY(cudaMalloc(&h->by[b], pb));
    CUDA_TRY(cudaEventCreateWithFlags(&h->ev_in[b], cudaEventDisableTiming));
    CUDA_TRY(cudaEventCreateWithFlags(&h->ev_comp[b], cudaEventDisableTiming));
    CUDA_TRY(cudaEventCreateWithFlags(&h->ev_out[b], cudaEventDisableTiming));
  }
  h->bytes += 2 * ehyb_dev::kPipe * pb;
  CUDA_TRY(cudaStreamCreateWithFlags(&h->s_out, cudaStreamNonBlocking));
  CUDA_TRY(cudaStreamCreateWithFlags(&h->s_in, cudaStreamNonBlocking));
  return 0;
}

EHYB_API int ehyb_dev_spmv_host_many(ehyb_dev* h, const void* const* x_hosts,
                                     void* const* y_hosts, int64_t count, int user_order,
                                     int mode, void* stream) {
  EHYB_TRY {
    if (!h || h->shard) return fail("spmv_host_many needs a full-matrix handle");
    if (count < 0 || (count > 0 && (!x_hosts || !y_hosts))) return fail("null argument");
    if (count == 0) return 0;
    DeviceGuard guard(h->device);
    int rc = ensure_scratch(h);
    if (rc) return rc;
    rc = ensure_pipeline(h);
    if (rc) return rc;
    auto st = static_cast<cudaStream_t>(stream);
    const size_t tb = size_t(h->tau);
    const size_t nb = size_t(user_order ? h->dimension : h->padded) * tb;
    // the copy-in stream starts after whatever the caller queued on `st`
    cudaEvent_t ev_start = h->ev_out[0];
    CUDA_TRY(cudaEventRecord(ev_start, st));
    CUDA_TRY(cudaStreamWaitEvent(h->s_in, ev_start, 0));
    constexpr int K = ehyb_dev::kPipe;
    for (int64_t i = 0; i < count; ++i) {
      const int b = int(i % K);
      // copy-in: buffer b is free once the compute of vector i-K has read it
      if (i >= K) CUDA_TRY(cudaStreamWaitEvent(h->s_in, h->ev_comp[b], 0));
      CUDA_TRY(cudaMemcpyAsync(h->bx[b], x_hosts[i], nb, cudaMemcpyHostToDevice, h->s_in));
      CUDA_TRY(cudaEventRecord(h->ev_in[b], h->s_in));
      // compute on the caller's stream; by[b] is free once the copy-out of i-K ended
      CUDA_TRY(cudaStreamWaitEvent(st, h->ev_in[b], 0));
      if (i >= K) CUDA_TRY(cudaStreamWaitEvent(st, h->ev_out[b], 0));
      if (user_order) {
        rc = ehyb_dev_spmv_user(h, h->bx[b], h->by[b], mode, stream);
        if (rc) return rc;
      } else {
        CUDA_TRY(launch_spmv(h, h->bx[b], h->by[b], mode, true, true, st));
      }
      CUDA_TRY(cudaEventRecord(h->ev_comp[b], st));
      // copy-out overlaps the next vector's copy-in (PCIe is full duplex)
      CUDA_TRY(cudaStreamWaitEvent(h->s_out, h->ev_comp[b], 0));
      CUDA_TRY(cudaMemcpyAsync(y_hosts[i], h->by[b], nb, cudaMemcpyDeviceToHost, h->s_out));
      CUDA_TRY(cudaEventRecord(h->ev_out[b], h->s_out));
    }
    CUDA_TRY(cudaStreamSynchronize(h->s_out));
    CUDA_TRY(cudaStreamSynchronize(st));
    return 0;
  }
  EHYB_CATCH
}

// ------------------------------------------------ P2P halo exchange
EHYB_API int ehyb_dev_p2p_alloc(ehyb_dev* h, void** x_ext, void** flags) {
  EHYB_TRY {
    if (!h || !h->shard) return fail("p2p buffers need a shard handle");
    DeviceGuard guard(h->device);
    if (!h->p2p_x) {
      const size_t xb = size_t(h->local_rows + h->n_halo) * size_t(h->tau);
      CUDA_TRY(cudaMalloc(&h->p2p_x, std::max<size_t>(xb, 16)));
      CUDA_TRY(cudaMemset(h->p2p_x, 0, std::max<size_t>(xb, 16)));
      CUDA_TRY(cudaMalloc(&h->p2p_flags, 64));
      CUDA_TRY(cudaMemset(h->p2p_flags, 0, 64));
      h->bytes += xb + 64;
    }
    if (x_ext) *x_ext = h->p2p_x;
    if (flags) *flags = h->p2p_flags;
    return 0;
  }
  EHYB_CATCH
}

EHYB_API int ehyb_ipc_handle(const void* dev_ptr, void* out_handle) {
  EHYB_TRY {
    if (!dev_ptr || !out_handle) return fail("null argument");
    cudaIpcMemHandle_t hd;
    CUDA_TRY(cudaIpcGetMemHandle(&hd, const_cast<void*>(dev_ptr)));
    std::memcpy(out_handle, &hd, sizeof(hd));
    return 0;
  }
  EHYB_CATCH
}

EHYB_API int ehyb_ipc_open(const void* handle, int device, void** out_ptr) {
  EHYB_TRY {
    if (!handle || !out_ptr) return fail("null argument");
    DeviceGuard guard(device);
    cudaIpcMemHandle_t hd;
    std::memcpy(&hd, handle, sizeof(hd));
    CUDA_TRY(cudaIpcOpenMemHandle(out_ptr, hd, cudaIpcMemLazyEnablePeerAccess));
    return 0;
  }
  EHYB_CATCH
}

EHYB_API int ehyb_ipc_close(void* ptr) {
  EHYB_TRY {
    if (ptr) CUDA_TRY(cudaIpcCloseMemHandle(ptr));
    return 0;
  }
  EHYB_CATCH
}

EHYB_API int ehyb_dev_p2p_setup(ehyb_dev* h, int32_t world, int32_t rank, void* const* peer_x,
                                void* const* peer_flags, const int32_t* pull_src,
                                const int64_t* pull_off, int64_t served_per_spmv) {
  EHYB_TRY {
    if (!h || !h->p2p_x) return fail("call ehyb_dev_p2p_alloc first");
    if (h->warp != 32 || !h->window_in_smem || !h->window_tma || h->ring_bytes)
      return fail("p2p exchange needs 32-row slices and a TMA-staged window");
    if (world < 1 || rank < 0 || rank >= world) return fail("bad world / rank");
    DeviceGuard guard(h->device);
    std::vector<void*> px(static_cast<size_t>(world)), pf(static_cast<size_t>(world));
    for (int q = 0; q < world; ++q) {
      px[size_t(q)] = q == rank ? h->p2p_x : peer_x[q];
      pf[size_t(q)] = q == rank ? static_cast<void*>(h->p2p_flags) : peer_flags[q];
    }
    if (h->peer_x_dev) cudaFree(h->peer_x_dev);
    if (h->peer_flags_dev) cudaFree(h->peer_flags_dev);
    if (h->pull_src) cudaFree(h->pull_src);
    if (h->pull_off) cudaFree(h->pull_off);
    h->peer_x_dev = nullptr;
    h->peer_flags_dev = nullptr;
    h->pull_src = nullptr;
    h->pull_off = nullptr;
    size_t dummy = 0;
    CUDA_TRY(upload(&h->peer_x_dev, px.data(), px.size() * sizeof(void*), &dummy));
    CUDA_TRY(upload(&h->peer_flags_dev, pf.data(), pf.size() * sizeof(void*), &dummy));
    CUDA_TRY(upload(&h->pull_src, pull_src, size_t(h->n_halo) * 4, &dummy));
    CUDA_TRY(upload(&h->pull_off, pull_off, size_t(h->n_halo) * 8, &dummy));
    h->served_per_spmv = (unsigned long long)served_per_spmv;
    h->p2p_ready = true;
    return 0;
  }
  EHYB_CATCH
}

EHYB_API int ehyb_dev_spmv_p2p(ehyb_dev* h, void* y_local, int mode, void* stream) {
  EHYB_TRY {
    if (!h || !h->p2p_ready) return fail("p2p exchange not set up (ehyb_dev_p2p_setup)");
    if (!y_local) return fail("null argument");
    DeviceGuard guard(h->device);
    // the sequence number advances only with a launch that was issued: a
    // failed launch must not put this rank out of step with its peers
    h->p2p_seq += 1;
    h->p2p_active = true;
    const cudaError_t e = launch_spmv(h, h->p2p_x, y_local, mode, true, true,
                                      static_cast<cudaStream_t>(stream));
    h->p2p_active = false;
    if (e != cudaSuccess) h->p2p_seq -= 1;
    CUDA_TRY(e);
    return 0;
  }
  EHYB_CATCH
}

EHYB_API int ehyb_dev_gather(const void* src, const int64_t* idx_dev, int64_t count, void* dst,
                             int32_t tau, void* stream) {
  EHYB_TRY {
    if (count <= 0) return 0;
    auto st = static_cast<cudaStream_t>(stream);
    const int g = int(std::min<int64_t>((count + 255) / 256, 148 * 16));
    if (tau == 4)
      gather_kernel<float><<<g, 256, 0, st>>>(static_cast<const float*>(src), idx_dev, count,
                                               static_cast<float*>(dst));
    else
      gather_kernel<double><<<g, 256, 0, st>>>(static_cast<const double*>(src), idx_dev, count,
                                                static_cast<double*>(dst));
    CUDA_TRY(cudaGetLastError());
    return 0;
  }
  EHYB_CATCH
}

EHYB_API int ehyb_dev_dot(const void* a, const void* b, int64_t n, int32_t tau, double* out_dev,
                          void* stream) {
  EHYB_TRY {
    auto st = static_cast<cudaStream_t>(stream);
    constexpr int kBlocks = 592, kThreads = 512;
    static thread_local std::unordered_map<int, double*> partials;
    int dev = 0;
    CUDA_TRY(cudaGetDevice(&dev));
    double*& part = partials[dev];
    if (!part) CUDA_TRY(cudaMalloc(&part, kBlocks * sizeof(double)));
    if (tau == 4)
      dot_partial_kernel<float><<<kBlocks, kThreads, 0, st>>>(
          static_cast<const float*>(a), static_cast<const float*>(b), n, part);
    else
      dot_partial_kernel<double><<<kBlocks, kThreads, 0, st>>>(
          static_cast<const double*>(a), static_cast<const double*>(b), n, part);
    dot_final_kernel<<<1, 1024, 0, st>>>(part, kBlocks, out_dev);
    CUDA_TRY(cudaGetLastError());
    return 0;
  }
  EHYB_CATCH
}

EHYB_API int ehyb_dev_cg_xr(void* x, void* r, const void* p, const void* q, const double* rr,
                            const double* pq, int64_t n, int32_t tau, double* rr_new,
                            void* stream) {
  EHYB_TRY {
    auto st = static_cast<cudaStream_t>(stream);
    constexpr int kBlocks = 592, kThreads = 512;
    static thread_local std::unordered_map<int, double*> partials;
    int dev = 0;
    CUDA_TRY(cudaGetDevice(&dev));
    double*& part = partials[dev];
    if (!part) CUDA_TRY(cudaMalloc(&part, kBlocks * sizeof(double)));
    if (tau == 4)
      cg_xr_kernel<float><<<kBlocks, kThreads, 0, st>>>(
          static_cast<float*>(x), static_cast<float*>(r), static_cast<const float*>(p),
          static_cast<const float*>(q), rr, pq, n, part);
    else
      cg_xr_kernel<double><<<kBlocks, kThreads, 0, st>>>(
          static_cast<double*>(x), static_cast<double*>(r), static_cast<const double*>(p),
          static_cast<const double*>(q), rr, pq, n, part);
    dot_final_kernel<<<1, 1024, 0, st>>>(part, kBlocks, rr_new);
    CUDA_TRY(cudaGetLastError());
    return 0;
  }
  EHYB_CATCH
}

EHYB_API int ehyb_dev_cg_p(void* p, const void* r, const double* rr_new, const double* rr_old,
                           int64_t n, int32_t tau, void* stream) {
  EHYB_TRY {
    auto st = static_cast<cudaStream_t>(stream);
    const int g = int(std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 16)));
    if (tau == 4)
      cg_p_kernel<float><<<g, 256, 0, st>>>(static_cast<float*>(p), static_cast<const float*>(r),
                                             rr_new, rr_old, n);
    else
      cg_p_kernel<double><<<g, 256, 0, st>>>(static_cast<double*>(p),
                                              static_cast<const double*>(r), rr_new, rr_old, n);
    CUDA_TRY(cudaGetLastError());
    return 0;
  }
  EHYB_CATCH
}

EHYB_API int ehyb_dev_dot2(const void* a, const void* b, const void* c, const void* d, int64_t n,
                           int32_t tau, double* out2_dev, void* stream) {
  EHYB_TRY {
    auto st = static_cast<cudaStream_t>(stream);
    constexpr int kBlocks = 592, kThreads = 512;
    static thread_local std::unordered_map<int, double*> partials;
    int dev = 0;
    CUDA_TRY(cudaGetDevice(&dev));
    double*& part = partials[dev];
    if (!part) CUDA_TRY(cudaMalloc(&part, 2 * kBlocks * sizeof(double)));
    if (tau == 4)
      dot2_partial_kernel<float><<<kBlocks, kThreads, 0, st>>>(
          static_cast<const float*>(a), static_cast<const float*>(b), static_cast<const float*>(c),
          static_cast<const float*>(d), n, part);
    else
      dot2_partial_kernel<double><<<kBlocks, kThreads, 0, st>>>(
          static_cast<const double*>(a), static_cast<const double*>(b),
          static_cast<const double*>(c), static_cast<const double*>(d), n, part);
    dot2_final_kernel<<<1, 1024, 0, st>>>(part, kBlocks, out2_dev);
    CUDA_TRY(cudaGetLastError());
    return 0;
  }
  EHYB_CATCH
}

EHYB_API int ehyb_dev_cgcg_step(void* x, void* r, void* p, void* s, const void* w, double* sc,
                                int first, int64_t n, int32_t tau, void* stream) {
  EHYB_TRY {
    auto st = static_cast<cudaStream_t>(stream);
    cgcg_scalars_kernel<<<1, 1, 0, st>>>(sc, first);
    const int g = int(std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 16)));
    if (tau == 4)
      cgcg_update_kernel<float><<<g, 256, 0, st>>>(
          static_cast<float*>(x), static_cast<float*>(r), static_cast<float*>(p),
          static_cast<float*>(s), static_cast<const float*>(w), sc, n);
    else
      cgcg_update_kernel<double><<<g, 256, 0, st>>>(
          static_cast<double*>(x), static_cast<double*>(r), static_cast<double*>(p),
          static_cast<double*>(s), static_cast<const double*>(w), sc, n);
    CUDA_TRY(cudaGetLastError());
    return 0;
  }
  EHYB_CATCH
}

EHYB_API int ehyb_dev_axpy(const double* a_dev, double sign, const void* x, void* y, int64_t n,
                           int32_t tau, void* stream) {
  EHYB_TRY {
    auto st = static_cast<cudaStream_t>(stream);
    const int g = int(std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 16)));
    if (tau == 4)
      axpy_kernel<float><<<g, 256, 0, st>>>(a_dev, sign, static_cast<const float*>(x),
                                             static_cast<float*>(y), n);
    else
      axpy_kernel<double><<<g, 256, 0, st>>>(a_dev, sign, static_cast<const double*>(x),
                                              static_cast<double*>(y), n);
    CUDA_TRY(cudaGetLastError());
    return 0;
  }
  EHYB_CATCH
}

}  // extern "C"

// ------------------------------------------------------------ cuSPARSE CSR
struct ehyb_csr {
  int device = 0;
  int tau = 8;
  int64_t n_rows = 0, n_cols = 0, nnz = 0;
  int32_t* row_ptr = nullptr;
  int32_t* col_idx = nullptr;
  void* vals = nullptr;
  void* buffer = nullptr;
  size_t buffer_bytes = 0;
  cusparseHandle_t handle = nullptr;
  cusparseSpMatDescr_t mat = nullptr;
  ~ehyb_csr() {
    if (mat) cusparseDestroySpMat(mat);
    if (handle) cusparseDestroy(handle);
    void* ptrs[] = {row_ptr, col_idx, vals, buffer};
    for (void* p : ptrs)
      if (p) cudaFree(p);
  }
};

extern "C" {

EHYB_API int ehyb_csr_create(int64_t n_rows, int64_t n_cols, int64_t nnz, const int64_t* row_ptr,
                             const int64_t* col_idx, const double* values, int32_t tau,
                             int device, ehyb_csr** out) {
  EHYB_TRY {
    if (nnz >= (int64_t(1) << 31)) return fail("CSR comparator needs nnz < 2^31");
    DeviceGuard guard(device);
    auto h = std::make_unique<ehyb_csr>();
    h->device = device;
    h->tau = tau;
    h->n_rows = n_rows;
    h->n_cols = n_cols;
    h->nnz = nnz;
    std::vector<int32_t> rp(size_t(n_rows) + 1), ci(size_t(std::max<int64_t>(nnz, 1)));
    for (int64_t i = 0; i <= n_rows; ++i) rp[size_t(i)] = int32_t(row_ptr[i]);
    for (int64_t i = 0; i < nnz; ++i) ci[size_t(i)] = int32_t(col_idx[i]);
    size_t total = 0;
    CUDA_TRY(upload(&h->row_ptr, rp.data(), rp.size() * 4, &total));
    CUDA_TRY(upload(&h->col_idx, ci.data(), size_t(nnz) * 4, &total));
    if (tau == 4) {
      std::vector<float> v(size_t(std::max<int64_t>(nnz, 1)));
      for (int64_t i = 0; i < nnz; ++i) v[size_t(i)] = float(values[i]);
      CUDA_TRY(upload(&h->vals, v.data(), size_t(nnz) * 4, &total));
    } else {
      CUDA_TRY(upload(&h->vals, values, size_t(nnz) * 8, &total));
    }
    CUSPARSE_TRY(cusparseCreate(&h->handle));
    const cudaDataType dt = tau == 4 ? CUDA_R_32F : CUDA_R_64F;
    CUSPARSE_TRY(cusparseCreateCsr(&h->mat, n_rows, n_cols, nnz, h->row_ptr, h->col_idx, h->vals,
                                   CUSPARSE_INDEX_32I, CUSPARSE_INDEX_32I,
                                   CUSPARSE_INDEX_BASE_ZERO, dt));
    *out = h.release();
    return 0;
  }
  EHYB_CATCH
}

EHYB_API int ehyb_csr_spmv(ehyb_csr* h, const void* x_dev, void* y_dev, int alg, void* stream) {
  EHYB_TRY {
    if (!h) return fail("null handle");
    DeviceGuard guard(h->device);
    if (alg == 0) {  // the reference's own summation order (engine.py:56-69), fp64
      if (h->tau != 8) return fail("reference-order CSR product needs float64 values");
      const int threads = 256;
      const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((h->n_rows + threads - 1) / threads,
                                                                     int64_t(1) << 20));
      csr_ref_kernel<<<unsigned(blocks), threads, 0, static_cast<cudaStream_t>(stream)>>>(
          h->row_ptr, h->col_idx, static_cast<const double*>(h->vals),
          static_cast<const double*>(x_dev), h->n_rows, static_cast<double*>(y_dev));
      CUDA_TRY(cudaGetLastError());
      return 0;
    }
    const cudaDataType dt = h->tau == 4 ? CUDA_R_32F : CUDA_R_64F;
    cusparseDnVecDescr_t vx, vy;
    CUSPARSE_TRY(cusparseCreateDnVec(&vx, h->n_cols, const_cast<void*>(x_dev), dt));
    CUSPARSE_TRY(cusparseCreateDnVec(&vy, h->n_rows, y_dev, dt));
    CUSPARSE_TRY(cusparseSetStream(h->handle, static_cast<cudaStream_t>(stream)));
    const cusparseSpMVAlg_t a = alg == 2 ? CUSPARSE_SPMV_CSR_ALG2 : CUSPARSE_SPMV_CSR_ALG1;
    double one_d = 1.0, zero_d = 0.0;
    float one_f = 1.0f, zero_f = 0.0f;
    const void* alpha = h->tau == 4 ? static_cast<const void*>(&one_f) : &one_d;
    const void* beta = h->tau == 4 ? static_cast<const void*>(&zero_f) : &zero_d;
    size_t need = 0;
    CUSPARSE_TRY(cusparseSpMV_bufferSize(h->handle, CUSPARSE_OPERATION_NON_TRANSPOSE, alpha, h->mat,
                                         vx, beta, vy, dt, a, &need));
    if (need > h->buffer_bytes) {
      if (h->buffer) cudaFree(h->buffer);
      h->buffer = nullptr;
      CUDA_TRY(cudaMalloc(&h->buffer, need));
      h->buffer_bytes = need;
    }
    CUSPARSE_TRY(cusparseSpMV(h->handle, CUSPARSE_OPERATION_NON_TRANSPOSE, alpha, h->mat, vx, beta,
                              vy, dt, a, h->buffer));
    cusparseDestroyDnVec(vx);
    cusparseDestroyDnVec(vy);
    return 0;
  }
  EHYB_CATCH
}

EHYB_API int ehyb_csr_destroy(ehyb_csr* h) {
  if (!h) return 0;
  DeviceGuard guard(h->device);
  delete h;
  return 0;
}

}  // extern "C"
