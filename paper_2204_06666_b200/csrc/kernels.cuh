// EHYB SpMV kernels for B200 (sm_100a).
//
// One CTA per partition (Alg.3; reference simulation
// engine.py:134-154):
//   1. the partition's x window x[p*vec, (p+1)*vec) is staged into shared
//      memory by TMA bulk copies (cp.async.bulk ... mbarrier::complete_tx);
//      meanwhile TMA bulk L2 prefetches (cp.async.bulk.prefetch.L2) start
//      streaming the partition's contiguous ELL slab, and every claimed slice
//      keeps the stream pf_ell slices ahead of the warps;
//   2. warps claim 32-row chunks (= SELL slices for warp_size 32) from a
//      shared-memory counter (the paper's in-block slice stealing) and read
//      val/col with coalesced evict-first loads, 2*kUnroll loads in flight per
//      lane, gathering x from the staged window through the u16 local columns;
//   3. a warp that finds the ELL counter empty moves straight on to the
//      partition's ER rows (derived per-partition SELL layout, x through the
//      read-only path) and finishes y[r] = y_ell[r] + er_acc once r's ELL
//      chunk has published its done bit — the reference's phase-2
//      "y[y_idx] += acc" without a grid-wide barrier or atomics (each ER row
//      belongs to exactly one partition, so only its own CTA touches it).
// STRICT arithmetic is the reference's: acc starts at +0.0 and every slot is
// a separately rounded multiply then add, k ascending, padding slots
// included — bitwise identical y. FMA mode fuses the two roundings.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace ehyb {

constexpr int kUnroll = 8;        // slots per lane in flight
#ifndef EHYB_POOL_BATCH_F64
#define EHYB_POOL_BATCH_F64 1
#endif
// fused-kernel CTA size cap per value type = its register budget (one CTA per
// SM): fp32 1024 threads x 64 registers, fp64 768 x 80 (the fp64 kernel
// wants ~78 registers; at 64 it spills, and the persistent K > 1 path runs
// 3% faster with the fatter warps: DESIGN.md §8)
#ifndef EHYB_MAX_THREADS_F32
#define EHYB_MAX_THREADS_F32 1024
#endif
#ifndef EHYB_MAX_THREADS_F64
#define EHYB_MAX_THREADS_F64 768
#endif
constexpr int max_threads_for(int tau) { return tau == 4 ? EHYB_MAX_THREADS_F32 : EHYB_MAX_THREADS_F64; }
constexpr int kMaxThreads = EHYB_MAX_THREADS_F32 > EHYB_MAX_THREADS_F64 ? EHYB_MAX_THREADS_F32
                                                                        : EHYB_MAX_THREADS_F64;
constexpr int kTmaChunk = 32768;  // bytes per cp.async.bulk instruction

template <typename T>
struct SpmvParams {
  // ELL body (parity arrays, re-based for shards)
  const T* __restrict__ val_ell;
  const uint16_t* __restrict__ col_ell;
  const int32_t* __restrict__ pos_ell;
  const int32_t* __restrict__ width_ell;
  // derived per-partition ER (32-row SELL slices)
  const int32_t* __restrict__ er_part_ptr;  // [n_parts+1] slice ranges
  const int32_t* __restrict__ er_part_mid;  // [n_parts] first slice with a halo column (shards)
  int32_t er_sel;                           // 0: all own slices, 1: [ptr, mid), 2: [mid, ptr+1)
  const int64_t* __restrict__ er_pos;       // [n_slices] slot offset of each slice
  const int32_t* __restrict__ er_swidth;    // [n_slices] slice width
  const int32_t* __restrict__ er_rows;      // [n_slices*32] row | kPadFlag, -1 = empty lane
  const int32_t* __restrict__ er_lwidth;    // [n_slices*32] lane width
  const T* __restrict__ er_val;
  const uint32_t* __restrict__ er_col;
  const T* __restrict__ x;  // reordered (or [owned | halo]) input
  int64_t er_pad_idx;       // x index of the column the reference's ER padding slots hold
                            // (global column 0; kPadFlag rows multiply it once)
  T* __restrict__ y;        // reordered (or owned) output
  int64_t vec;
  int32_t warp;             // slice height C of the ELL body
  int32_t window_in_smem;
  int32_t window_tma;
  int32_t do_ell;
  int32_t do_er;
  int32_t pf_ell;            // ELL slices kept in flight ahead of the warps by L2 bulk prefetch (0 = off)
  int32_t pf_er;             // 1 = L2 bulk prefetch of the next ER slice per warp
  unsigned long long* timing;  // optional per-CTA %globaltimer stamps [start, window, ell issue
                               // end, end, own ER, combine, pool, ell published] (8 per CTA)
  // ER work pool shared by all CTAs (load balance across partitions): any
  // warp computes pooled slices into a global scratch at any time; the
  // owning CTA adds them to its rows once all of them are in
  int64_t pool_lo, pool_hi;         // global slice range of the pool
  unsigned int* pool_ctr;           // [2] claim counters, alternating by epoch
  unsigned int* pool_done;          // [2][n_parts] computed pooled slices per owner, by epoch
  const int32_t* __restrict__ pool_own_ptr;  // [n_parts+1] pooled slices of each partition
  const int32_t* __restrict__ pool_own_idx;  // their slice indices
  T* pool_acc;                      // [(pool_hi-pool_lo)*32] pooled row sums, owner-major order
  const int32_t* __restrict__ pool_pos;   // [pool slices] owner-major position of each pooled slice
  const int32_t* __restrict__ pool_rows;  // [pool slices*32] their rows, owner-major order
  T* own_acc;                       // [er_slices*32] own ER row sums beyond the smem buffer (or null)
  // P2P halo (shards, exchange = peer memory): the launch itself pulls the
  // halo from the peers' x buffers over NVLink and finishes halo rows once
  // its pulls are complete — one launch per SpMV, no NCCL
  int64_t n_halo;                   // halo slots, x_ext[local_rows + i]
  int64_t local_rows;
  const int32_t* __restrict__ pull_src;   // [n_halo] peer rank of each halo slot
  const int64_t* __restrict__ pull_off;   // [n_halo] offset in that peer's x
  T* const* peer_x;                       // [world] peers' x buffers (own entry unused)
  unsigned long long* const* peer_flags;  // [world] peers' flag blocks
  unsigned long long* my_flags;           // {ready seq, served (cum.), pulled (cum.)}
  unsigned long long seq;                 // SpMV sequence number (>= 1)
  unsigned long long served_per_spmv;     // values peers pull from this rank per SpMV
  unsigned long long spin_timeout_ns;     // a cross-rank wait longer than this traps (a peer
                                          // out of lockstep or dead): the launch fails loudly
  // several partitions per CTA: pooled slices grouped by the iteration in
  // which their owner partition runs (p / grid); group g is drained by the
  // ER-first warps during iteration g+1, rows finished in place once the
  // owner partition is published (part_flag == epoch)
  unsigned int* part_flag;          // [n_parts] epoch in which the partition's rows are final
  const int32_t* __restrict__ pool_grp;  // [n_groups+1] pooled-slice range of each group
  int32_t pool_groups;
  unsigned int* pool_gctr;          // [2][n_groups] group claim counters by epoch
  int32_t pool_last_scratch;        // 1: the last group is computed early into pool_acc and
                                    // added by its owners after the loop (no in-place wait)
  unsigned int* epoch_dev;          // [2]: launch sequence number (>= 1), CTAs finished; kept
                                    // on the device so a captured CUDA graph replays correctly
  // own-ER shared-memory buffer (overlap of ER gathers with the ELL stream)
  int32_t er_buf_slices;            // buffered own ER slices (<= kMaxErBuf)
  int32_t er_buf_offset;            // byte offset of the buffer in dynamic smem
  int32_t er_warps;                 // warps that start on ER before ELL
  int32_t n_parts;                  // work units of this launch (grid may be smaller: CTAs loop)
  int32_t split;                    // units per partition (a partition's 32-row chunks split
                                    // into `split` contiguous ranges, each its own CTA that
                                    // stages the same window; 1 = one unit per partition)
  int32_t unit_chunks;              // chunks per unit (the last unit of a partition may be short)
  int32_t ell_vec;                  // 1: ELL slices in the 128-bit interleaved layout
  int32_t ring_offset;              // RING variant: ELL staging ring in dynamic smem,
  int32_t ring_stages, stage_bytes, stage_vbytes;  // stages x stage_bytes (values first)
  // stage plan (host-built): stage t copies slab slots [st_pos[t], +st_slots[t])
  // and holds st_chunks[t] consecutive chunks; chunk c of a partition lives in
  // its local stage ch_stage[c].x at slot offset ch_stage[c].y
  const int32_t* __restrict__ part_stage_ptr;  // [n_parts+1]
  const int32_t* __restrict__ st_pos;
  const int32_t* __restrict__ st_slots;
  const int32_t* __restrict__ st_chunks;
  const uint2* __restrict__ ch_stage;          // [local_rows/32]
  const int32_t* __restrict__ unit_part;  // persistent launches: partition of each unit (null =
  const int32_t* __restrict__ part_unit;  // identity; units run heaviest first) and its inverse
  int32_t meta_off;                 // >= 0: byte offset in dynamic smem of the unit's chunk
                                    // metadata {pos, eff} (loaded once per partition; the
                                    // per-chunk claims then read shared memory), -1 = global
  int32_t ell_ahead;                // 1 = claim the next ELL chunk (and its metadata) one ahead
  int32_t er_ahead;                 // 1 = same for ER slices
  // long rows (derived at upload): rows whose ELL or ER width exceeds the long
  // threshold leave the slice paths (their lanes are masked) and are computed
  // by whole warps claimed at kernel start
  const uint32_t* __restrict__ long_bits;  // [local_rows/32] bit per masked row
  int32_t lr_tasks;                        // long rows
  const int64_t* __restrict__ lr_span;     // [3*tasks] lo, mid (ELL|ER split), hi
  const int32_t* __restrict__ lr_row;      // [tasks] row | kLrEllPad | kLrErPad | kLrHasEr
  const int64_t* __restrict__ lr_padcol;   // [tasks] x index of the ELL padding product
  const T* __restrict__ lr_val;
  const uint32_t* __restrict__ lr_col;     // x indices (window columns made global)
  int32_t lr_segs;                         // FMA mode: segments of the long rows
  const int64_t* __restrict__ lr_seg;      // [3*segs] task, lo, hi
  const int32_t* __restrict__ lr_task_seg; // [tasks+1] segment range of each task
  const int32_t* __restrict__ lr_task_nell;// [tasks] ELL segments of each task
  T* __restrict__ lr_part;                 // [segs] segment partial sums
  unsigned int* lr_cnt;                    // [tasks] finished segments (self-resetting)
  unsigned int* lr_ctr;                    // [2] task / segment claim counters by epoch
};

// The work unit that owns (local) row r: partition r / vec, chunk range by
// unit_chunks (SpmvParams::split).
template <bool SPLIT, typename T>
__device__ __forceinline__ uint32_t unit_of_row(const SpmvParams<T>& P, uint32_t r) {
  const uint32_t q = r / uint32_t(P.vec);
  if constexpr (!SPLIT) return P.part_unit ? uint32_t(__ldg(P.part_unit + q)) : q;
  const uint32_t h = ((r - q * uint32_t(P.vec)) >> 5) / uint32_t(P.unit_chunks);
  return q * uint32_t(P.split) + (h < uint32_t(P.split) ? h : uint32_t(P.split) - 1u);
}

// ell_eff (the slice widths the kernel reads) = effective width | flags
constexpr int32_t kEffWidth = 0x00ffffff;
constexpr int32_t kEffHasEr = 1 << 28;    // a row of the slice has ER entries (publish its completion)
constexpr int32_t kEffPadTail = 1 << 29;  // lanes owe the reference's padding products 0*win[0]
constexpr int32_t kEffHasLong = 1 << 30;  // a lane of the slice is a long row (long_bits)
// lr_row flags
constexpr int32_t kLrRowMask = 0x0fffffff;
constexpr int32_t kLrEllPad = 1 << 28;
constexpr int32_t kLrErPad = 1 << 29;
constexpr int32_t kLrHasEr = 1 << 30;

constexpr int32_t kPadFlag = 0x40000000;  // row had reference ER padding slots
constexpr int32_t kRowMask = 0x3fffffff;

// ------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// one lane's shared-memory counter claim: a plain atom.shared (the compiler
// turns atomicAdd under `lane == 0` into a warp-aggregated sequence)
__device__ __forceinline__ int atom_add_shared(int* p, int v) {
  int r;
  asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(r) : "r"(smem_addr(p)), "r"(v) : "memory");
  return r;
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void tma_bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                             uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "EHYB_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra EHYB_WAIT_%=;\n}" ::"r"(smem_addr(bar)),
      "r"(phase)
      : "memory");
}

template <bool STRICT>
__device__ __forceinline__ double madd(double acc, double v, double x) {
  if constexpr (STRICT) return __dadd_rn(acc, __dmul_rn(v, x));
  else return fma(v, x, acc);
}
template <bool STRICT>
__device__ __forceinline__ float madd(float acc, float v, float x) {
  if constexpr (STRICT) return __fadd_rn(acc, __fmul_rn(v, x));
  else return fmaf(v, x, acc);
}
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ void st_release_gpu(unsigned int* p, unsigned int v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned int ld_acquire_gpu(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void bulk_prefetch_l2(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}


// TMA bulk prefetch of one 32-row SELL slice (vals + cols) into L2. Slice
// offsets are multiples of 32 slots, so both ranges are 64 B aligned and a
// multiple of 16 bytes long, as cp.async.bulk requires.
template <typename T>
__device__ __forceinline__ void prefetch_slice(const T* val, const uint16_t* col, int64_t p0,
                                               int64_t p1) {
  if (p1 > p0) {
    bulk_prefetch_l2(val + p0, uint32_t((p1 - p0) * int64_t(sizeof(T))));
    bulk_prefetch_l2(col + p0, uint32_t((p1 - p0) * 2));
  }
}

// One 32-row SELL slice, one row per lane, slots pos + 32k. Full batches of
// U slots issue all column and value loads before the first gather so every
// lane keeps 2U independent loads in flight (U = 8 for fp64, 16 for fp32:
// the same bytes in flight per lane); the tail batch is predicated. The
// accumulation order is k ascending (reference order).
// ELL stream loads. EHYB_LD_HINT selects the PTX form (measured in
// DESIGN.md §8): 0 = ld.global.cs (evict-first), 1/2 = ld.global.cs with an
// L2 prefetch size of 128/256 B, 3 = ld.global.nc.L1::no_allocate.L2::256B
#ifndef EHYB_LD_HINT
#define EHYB_LD_HINT 0
#endif
#if EHYB_LD_HINT == 1
#define EHYB_LD_Q "ld.global.cs.L2::128B"
#elif EHYB_LD_HINT == 2
#define EHYB_LD_Q "ld.global.cs.L2::256B"
#elif EHYB_LD_HINT == 3
#define EHYB_LD_Q "ld.global.nc.L1::no_allocate.L2::256B"
#endif
__device__ __forceinline__ uint32_t ld_stream(const uint16_t* p) {
#if EHYB_LD_HINT == 0
  return __ldcs(p);
#else
  unsigned short v;
  asm volatile(EHYB_LD_Q ".u16 %0, [%1];" : "=h"(v) : "l"(p));
  return v;
#endif
}
__device__ __forceinline__ double ld_stream(const double* p) {
#if EHYB_LD_HINT == 0
  return __ldcs(p);
#else
  double v;
  asm volatile(EHYB_LD_Q ".f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
#endif
}
__device__ __forceinline__ float ld_stream(const float* p) {
#if EHYB_LD_HINT == 0
  return __ldcs(p);
#else
  float v;
  asm volatile(EHYB_LD_Q ".f32 %0, [%1];" : "=f"(v) : "l"(p));
  return v;
#endif
}

#ifndef EHYB_UNROLL_F32
#define EHYB_UNROLL_F32 8
#endif
#ifndef EHYB_UNROLL_F64
#define EHYB_UNROLL_F64 8
#endif
template <typename T>
struct EllUnroll {
  static constexpr int value = sizeof(T) == 4 ? EHYB_UNROLL_F32 : EHYB_UNROLL_F64;
};

template <typename T, bool STRICT, bool WAIT>
__device__ __forceinline__ T ell_slice32(const T* __restrict__ val,
                                         const uint16_t* __restrict__ col, int64_t pos, int w,
                                         const T* win, uint64_t* win_bar, uint32_t win_phase) {
  constexpr int U = EllUnroll<T>::value;
  T acc = T(0);
  int k = 0;
  for (; k + U <= w; k += U) {
    uint32_t c[U];
    T v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) c[u] = ld_stream(col + pos + int64_t(k + u) * 32);
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = ld_stream(val + pos + int64_t(k + u) * 32);
    // a warp's first chunk issues its stream loads before the window has
    // landed: the TMA copy and the first HBM round trip overlap
    if constexpr (WAIT) {
      if (k == 0) mbar_wait(win_bar, win_phase);
    }
    T xv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) xv[u] = win[c[u]];
#pragma unroll
    for (int u = 0; u < U; ++u) acc = madd<STRICT>(acc, v[u], xv[u]);
  }
  if (k < w) {
    uint32_t c[U];
    T v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      c[u] = 0;
      v[u] = T(0);
      if (k + u < w) {
        c[u] = ld_stream(col + pos + int64_t(k + u) * 32);
        v[u] = ld_stream(val + pos + int64_t(k + u) * 32);
      }
    }
    if constexpr (WAIT) {
      if (k == 0) mbar_wait(win_bar, win_phase);
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (k + u < w) acc = madd<STRICT>(acc, v[u], win[c[u]]);
  }
  return acc;
}

// One 32-row SELL slice staged in shared memory by the ring producer (TMA):
// values and columns are read with conflict-free LDS, x gathered from the
// window; k ascending as in the reference.
template <typename T, bool STRICT>
__device__ __forceinline__ T ell_slice32_smem(const T* sv, const uint16_t* sc, int w,
                                              const T* win) {
  constexpr int U = 8;
  T acc = T(0);
  int k = 0;
  for (; k + U <= w; k += U) {
    uint32_t c[U];
    T v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) c[u] = sc[32 * (k + u)];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = sv[32 * (k + u)];
    T xv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) xv[u] = win[c[u]];
#pragma unroll
    for (int u = 0; u < U; ++u) acc = madd<STRICT>(acc, v[u], xv[u]);
  }
  for (; k < w; ++k) acc = madd<STRICT>(acc, sv[32 * k], win[sc[32 * k]]);
  return acc;
}

constexpr int kRingNS = 8;   // max ring data slots
constexpr int kRingFB = 64;  // full barriers, by stage number mod 64: a consumer (at most 31
                             // chunks ahead of the oldest unconsumed one) never waits on a
                             // barrier whose previous phase is still pending

// One 32-row slice in the interleaved layout (device.cu): k blocks of 4 hold
// a lane's 4 consecutive entries contiguously — one 16-byte value load per 4
// (fp32) or 2 (fp64) entries and one 8-byte load per 4 columns, 512 B per warp
// instruction — then the W % 4 tail in SELL order. UB blocks per batch keep
// the same bytes in flight as the scalar path with fewer registers and a
// quarter of the load instructions. Accumulation is k ascending.
#ifndef EHYB_VEC_UB_F32
#define EHYB_VEC_UB_F32 4
#endif
#ifndef EHYB_VEC_UB_F64
#define EHYB_VEC_UB_F64 2
#endif
template <typename T>
struct VecBlocks {
  static constexpr int value = sizeof(T) == 4 ? EHYB_VEC_UB_F32 : EHYB_VEC_UB_F64;
};

template <typename T>
__device__ __forceinline__ void ld_block4(const T* p, T* v);
template <>
__device__ __forceinline__ void ld_block4<float>(const float* p, float* v) {
  const float4 q = __ldcs(reinterpret_cast<const float4*>(p));
  v[0] = q.x;
  v[1] = q.y;
  v[2] = q.z;
  v[3] = q.w;
}
template <>
__device__ __forceinline__ void ld_block4<double>(const double* p, double* v) {
  const double2 a = __ldcs(reinterpret_cast<const double2*>(p));
  const double2 b = __ldcs(reinterpret_cast<const double2*>(p) + 1);
  v[0] = a.x;
  v[1] = a.y;
  v[2] = b.x;
  v[3] = b.y;
}

template <typename T, bool STRICT, bool WAIT>
__device__ __forceinline__ T ell_slice32_vec(const T* __restrict__ val,
                                             const uint16_t* __restrict__ col, int64_t pos, int w,
                                             int lane, const T* win, uint64_t* win_bar,
                                             uint32_t win_phase) {
  constexpr int UB = VecBlocks<T>::value;
  T acc = T(0);
  const int nb = w >> 2;
  const int nt = w & 3;
  const T* vb = val + pos + 4 * lane;
  const uint16_t* cb = col + pos + 4 * lane;
  bool waited = false;
  auto gather_blocks = [&](const uint2* c, T* xv) {
#pragma unroll
    for (int u = 0; u < UB; ++u) {
      xv[4 * u + 0] = win[c[u].x & 0xffffu];
      xv[4 * u + 1] = win[c[u].x >> 16];
      xv[4 * u + 2] = win[c[u].y & 0xffffu];
      xv[4 * u + 3] = win[c[u].y >> 16];
    }
  };
  int b = 0;
  // full batches: UB blocks each, while more than UB blocks remain
  for (; b + UB < nb; b += UB) {
    T v[4 * UB];
    uint2 c[UB];
#pragma unroll
    for (int u = 0; u < UB; ++u) c[u] = __ldcs(reinterpret_cast<const uint2*>(cb + 128 * (b + u)));
#pragma unroll
    for (int u = 0; u < UB; ++u) ld_block4<T>(vb + 128 * (b + u), v + 4 * u);
    if constexpr (WAIT) {
      if (!waited) {
        mbar_wait(win_bar, win_phase);
        waited = true;
      }
    }
    T xv[4 * UB];
    gather_blocks(c, xv);
#pragma unroll
    for (int j = 0; j < 4 * UB; ++j) acc = madd<STRICT>(acc, v[j], xv[j]);
  }
  // last batch: the remaining (<= UB) blocks AND the W % 4 tail (SELL order
  // after the blocks) issued together, so a narrow slice costs one round trip
  {
    const int rb = nb - b;
    T v[4 * UB];
    uint2 c[UB];
    T tv[3];
    uint32_t tc[3];
#pragma unroll
    for (int u = 0; u < UB; ++u) {
      c[u] = make_uint2(0u, 0u);
      if (u < rb) c[u] = __ldcs(reinterpret_cast<const uint2*>(cb + 128 * (b + u)));
    }
    const int64_t tpos = pos + 128 * int64_t(nb) + lane;
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      tc[j] = 0;
      if (j < nt) tc[j] = __ldcs(col + tpos + 32 * j);
    }
#pragma unroll
    for (int u = 0; u < UB; ++u) {
      if (u < rb) {
        ld_block4<T>(vb + 128 * (b + u), v + 4 * u);
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) v[4 * u + j] = T(0);
      }
    }
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      tv[j] = T(0);
      if (j < nt) tv[j] = __ldcs(val + tpos + 32 * j);
    }
    if constexpr (WAIT) {
      if (!waited) mbar_wait(win_bar, win_phase);
    }
    T xv[4 * UB];
    gather_blocks(c, xv);
    T tx[3];
#pragma unroll
    for (int j = 0; j < 3; ++j) tx[j] = win[tc[j]];
#pragma unroll
    for (int u = 0; u < UB; ++u)
      if (u < rb) {
#pragma unroll
        for (int j = 0; j < 4; ++j) acc = madd<STRICT>(acc, v[4 * u + j], xv[4 * u + j]);
      }
#pragma unroll
    for (int j = 0; j < 3; ++j)
      if (j < nt) acc = madd<STRICT>(acc, tv[j], tx[j]);
  }
  return acc;
}

// Generic slice height C (the reference tests use 1, 4, 8): one row per
// thread, slots pos + C k.
template <typename T, bool STRICT>
__device__ __forceinline__ T ell_row_generic(const T* __restrict__ val,
                                             const uint16_t* __restrict__ col, int64_t pos, int w,
                                             int64_t C, const T* win) {
  T acc = T(0);
  for (int k = 0; k < w; k += kUnroll) {
    T v[kUnroll];
    uint32_t c[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      c[u] = 0;
      v[u] = T(0);
      if (k + u < w) {
        v[u] = __ldcs(val + pos + int64_t(k + u) * C);
        c[u] = __ldcs(col + pos + int64_t(k + u) * C);
      }
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u)
      if (k + u < w) acc = madd<STRICT>(acc, v[u], win[c[u]]);
  }
  return acc;
}

// Derived ER slice metadata of one lane: target row (-1 = empty lane, with
// kPadFlag), lane width, slice width and the lane's first slot.
struct ErMeta {
  int32_t rw;
  int lw;
  int sw;
  int64_t pos;
};

template <typename T>
__device__ __forceinline__ ErMeta er_slice_meta(const SpmvParams<T>& P, int64_t s, int lane) {
  ErMeta m;
  m.rw = __ldg(P.er_rows + s * 32 + lane);
  m.lw = __ldg(P.er_lwidth + s * 32 + lane);
  m.sw = __ldg(P.er_swidth + s);
  m.pos = __ldg(P.er_pos + s) + lane;
  return m;
}

// Metadata of a claimed ER slice (s >= s_end: an empty claim) plus a precise
// L2 bulk prefetch of its values and columns.
template <typename T>
__device__ __forceinline__ ErMeta er_claimed_meta(const SpmvParams<T>& P, int64_t s,
                                                  int64_t s_end, int lane) {
  ErMeta m{-1, 0, 0, 0};
  if (s < s_end) {
    m = er_slice_meta(P, s, lane);
    if (lane == 0 && P.pf_er && m.sw > 0) {
      bulk_prefetch_l2(P.er_val + m.pos - lane, uint32_t(32 * int64_t(m.sw) * int64_t(sizeof(T))));
      bulk_prefetch_l2(P.er_col + m.pos - lane, uint32_t(32 * int64_t(m.sw) * 4));
    }
  }
  return m;
}

// Products of one ER row in k order, x through the read-only path; the
// reference's ER padding products 0*x[0] (engine.py:148-151) are inert for
// finite x and NaN-propagating otherwise — reproduced with one product.
template <typename T, bool STRICT>
__device__ __forceinline__ T er_slice_compute(const SpmvParams<T>& P, const ErMeta& m) {
  T acc = T(0);
  for (int k = 0; k < m.sw; k += kUnroll) {
    T v[kUnroll];
    uint32_t c[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      c[u] = 0;
      v[u] = T(0);
      if (k + u < m.lw) {
        c[u] = __ldcs(P.er_col + m.pos + int64_t(k + u) * 32);
        v[u] = __ldcs(P.er_val + m.pos + int64_t(k + u) * 32);
      }
    }
    T xv[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) xv[u] = (k + u < m.lw) ? __ldg(P.x + c[u]) : T(0);
#pragma unroll
    for (int u = 0; u < kUnroll; ++u)
      if (k + u < m.lw) acc = madd<STRICT>(acc, v[u], xv[u]);
  }
  if (m.rw >= 0 && (m.rw & kPadFlag)) acc = add_rn(acc, mul_rn(T(0), __ldg(P.x + P.er_pad_idx)));
  return acc;
}

#ifndef EHYB_ER_PAIRS_F64_GROUP
#define EHYB_ER_PAIRS_F64_GROUP 1  // fp64: pairs in the persistent group drain (cfg3 fp64 177.6 -> 173.7 us)
#endif
#ifndef EHYB_ER_PAIRS_F64
#define EHYB_ER_PAIRS_F64 0  // fp64: pairs in the pool drain and own-ER passes too
#endif
#ifndef EHYB_ER_PAIRS
#define EHYB_ER_PAIRS 1
#endif
// Two ER slices at once (one warp, lane = row in each): their loads and x
// gathers are issued together, so a latency-bound slice costs half the warp
// time. b may be an empty claim (rw = -1, widths 0). Per row the order is the
// reference's k order; the padding products as in er_slice_compute.
template <typename T, bool STRICT>
__device__ __forceinline__ void er_pair_compute(const SpmvParams<T>& P, const ErMeta& a,
                                                const ErMeta& b, T& acc_a, T& acc_b) {
  constexpr int U = 4;
  acc_a = T(0);
  acc_b = T(0);
  const int sw = a.sw > b.sw ? a.sw : b.sw;
  for (int k = 0; k < sw; k += U) {
    T va[U], vb[U];
    uint32_t ca[U], cb[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      ca[u] = cb[u] = 0;
      va[u] = vb[u] = T(0);
      if (k + u < a.lw) {
        ca[u] = __ldcs(P.er_col + a.pos + int64_t(k + u) * 32);
        va[u] = __ldcs(P.er_val + a.pos + int64_t(k + u) * 32);
      }
      if (k + u < b.lw) {
        cb[u] = __ldcs(P.er_col + b.pos + int64_t(k + u) * 32);
        vb[u] = __ldcs(P.er_val + b.pos + int64_t(k + u) * 32);
      }
    }
    T xa[U], xb[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      xa[u] = (k + u < a.lw) ? __ldg(P.x + ca[u]) : T(0);
      xb[u] = (k + u < b.lw) ? __ldg(P.x + cb[u]) : T(0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (k + u < a.lw) acc_a = madd<STRICT>(acc_a, va[u], xa[u]);
      if (k + u < b.lw) acc_b = madd<STRICT>(acc_b, vb[u], xb[u]);
    }
  }
  if (a.rw >= 0 && (a.rw & kPadFlag)) acc_a = add_rn(acc_a, mul_rn(T(0), __ldg(P.x + P.er_pad_idx)));
  if (b.rw >= 0 && (b.rw & kPadFlag)) acc_b = add_rn(acc_b, mul_rn(T(0), __ldg(P.x + P.er_pad_idx)));
}

// ------------------------------------------------------------- long rows
// STRICT: the reference's serial order over entries [lo, hi) — acc from +0.0,
// each product rounded, then added. Entries are fetched 32*LB at a time (lane
// i holds entry base+i) two blocks ahead behind an L2 bulk prefetch, their x
// gathered one block ahead, and the rounded products staged in shared memory
// so the only exposed latency is the dependent add chain itself.
template <typename T>
__device__ __forceinline__ T long_chain_strict(const SpmvParams<T>& P, int64_t lo, int64_t hi,
                                               int lane, T* stage) {
  constexpr int LB = 2;
  constexpr int BLK = 32 * LB;
  T acc = T(0);
  if (hi <= lo) return acc;
  auto load = [&](int64_t base, T* v, uint32_t* c) {
#pragma unroll
    for (int b = 0; b < LB; ++b) {
      const int64_t i = base + 32 * b + lane;
      c[b] = 0;
      v[b] = T(0);
      if (i < hi) {
        c[b] = __ldcs(P.lr_col + i);
        v[b] = __ldcs(P.lr_val + i);
      }
    }
  };
  T v1[LB], v2[LB], x1[LB];
  uint32_t c1[LB], c2[LB];
  load(lo, v1, c1);
  load(lo + BLK, v2, c2);
#pragma unroll
  for (int b = 0; b < LB; ++b) x1[b] = (lo + 32 * b + lane < hi) ? __ldg(P.x + c1[b]) : T(0);
  for (int64_t base = lo; base < hi; base += BLK) {
    if (lane == 0) {  // keep the entry stream in L2 well ahead of the loads
      const int64_t a = (base + 16 * BLK) & ~int64_t(3);
      const int64_t n = (hi - a < 4 * BLK ? hi - a : 4 * BLK) & ~int64_t(3);
      if (n > 0) {
        bulk_prefetch_l2(P.lr_val + a, uint32_t(n * int64_t(sizeof(T))));
        bulk_prefetch_l2(P.lr_col + a, uint32_t(n * 4));
      }
    }
    __syncwarp();
#pragma unroll
    for (int b = 0; b < LB; ++b) stage[32 * b + lane] = mul_rn(v1[b], x1[b]);
    __syncwarp();
#pragma unroll
    for (int b = 0; b < LB; ++b) {
      v1[b] = v2[b];
      c1[b] = c2[b];
    }
    load(base + 2 * BLK, v2, c2);
#pragma unroll
    for (int b = 0; b < LB; ++b)
      x1[b] = (base + BLK + 32 * b + lane < hi) ? __ldg(P.x + c1[b]) : T(0);
    const int64_t rem = hi - base;
    if (rem >= BLK) {
#pragma unroll
      for (int i = 0; i < BLK; ++i) acc = add_rn(acc, stage[i]);
    } else {
      for (int i = 0; i < int(rem); ++i) acc = add_rn(acc, stage[i]);
    }
  }
  return acc;
}

// FMA mode: one segment [lo, hi) of a long row, lane-strided fused
// multiply-adds and a fixed shuffle tree (deterministic, reassociated).
template <typename T>
__device__ __forceinline__ T long_segment_fast(const SpmvParams<T>& P, int64_t lo, int64_t hi,
                                               int lane) {
  T acc = T(0);
  for (int64_t base = lo; base < hi; base += 32 * kUnroll) {
    T v[kUnroll];
    uint32_t c[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int64_t i = base + 32 * u + lane;
      c[u] = 0;
      v[u] = T(0);
      if (i < hi) {
        c[u] = __ldcs(P.lr_col + i);
        v[u] = __ldcs(P.lr_val + i);
      }
    }
    T xv[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) xv[u] = (base + 32 * u + lane < hi) ? __ldg(P.x + c[u]) : T(0);
#pragma unroll
    for (int u = 0; u < kUnroll; ++u)
      if (base + 32 * u + lane < hi) acc = fma(v[u], xv[u], acc);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  return acc;
}

// y of a long row from its ELL and ER accumulators (engine.py:140-154 order:
// y = acc_ell (+ padding products); y += acc_er (+ padding products)).
template <typename T>
__device__ __forceinline__ T long_finish(const SpmvParams<T>& P, int task, T ell, T er) {
  const int32_t rw = __ldg(P.lr_row + task);
  if (rw & kLrEllPad) ell = add_rn(ell, mul_rn(T(0), __ldg(P.x + __ldg(P.lr_padcol + task))));
  if (!(rw & kLrHasEr)) return ell;
  if (rw & kLrErPad) er = add_rn(er, mul_rn(T(0), __ldg(P.x + P.er_pad_idx)));
  return add_rn(ell, er);
}

// Long-row work of one warp, claimed from a grid-wide counter: whole rows in
// STRICT mode (serial chains, longest first), segments in FMA mode (the last
// segment of a row to finish sums the partials in segment order).
template <typename T, int MODE>
__device__ void long_rows_warp(const SpmvParams<T>& P, int lane, T* stage, uint32_t ep) {
  unsigned int* ctr = P.lr_ctr + (ep & 1u);
  // EHYB_MODE_STRICT: one serial chain per row; DEFAULT / FMA: segments
  constexpr bool serial = MODE == EHYB_MODE_STRICT;
  const int n_items = serial ? P.lr_tasks : P.lr_segs;
  for (;;) {
    unsigned int v = 0;
    if (lane == 0) v = atomicAdd(ctr, 1u);
    const int item = int(__shfl_sync(0xffffffffu, v, 0));
    if (item >= n_items) break;
    if constexpr (serial) {
      const int64_t lo = __ldg(P.lr_span + 3 * item), mid = __ldg(P.lr_span + 3 * item + 1),
                    hi = __ldg(P.lr_span + 3 * item + 2);
      const T ell = long_chain_strict(P, lo, mid, lane, stage);
      const T er = long_chain_strict(P, mid, hi, lane, stage);
      const T yv = long_finish(P, item, ell, er);
      if (lane == 0) P.y[__ldg(P.lr_row + item) & kLrRowMask] = yv;
    } else {
      const int task = int(__ldg(P.lr_seg + 3 * item));
      const T part = long_segment_fast(P, __ldg(P.lr_seg + 3 * item + 1),
                                       __ldg(P.lr_seg + 3 * item + 2), lane);
      if (lane == 0) {
        P.lr_part[item] = part;
        __threadfence();
        const int s0 = __ldg(P.lr_task_seg + task), s1 = __ldg(P.lr_task_seg + task + 1);
        if (atomicAdd(P.lr_cnt + task, 1u) == unsigned(s1 - s0 - 1)) {
          __threadfence();
          const int s_mid = s0 + __ldg(P.lr_task_nell + task);
          T ell = T(0), er = T(0);
          for (int s = s0; s < s_mid; ++s) ell += __ldcg(P.lr_part + s);
          for (int s = s_mid; s < s1; ++s) er += __ldcg(P.lr_part + s);
          P.y[__ldg(P.lr_row + task) & kLrRowMask] = long_finish(P, task, ell, er);
          P.lr_cnt[task] = 0u;  // ready for the next launch
        }
      }
    }
  }
}

// Pooled ER slices: claim from the grid-wide counter, compute, write the 32
// row sums to the scratch, then count the slice for its owning partition
// (release: the sums are visible before the count). At most `max_items`
// slices (<= 0: until the pool is exhausted); returns false once exhausted.
template <typename T, bool STRICT, bool SPLIT>
__device__ bool pool_drain(const SpmvParams<T>& P, int lane, int max_items, uint32_t ep) {
  if (P.pool_hi <= P.pool_lo) return false;
  unsigned int* ctr = P.pool_ctr + (ep & 1u);
  unsigned int* done = P.pool_done + (ep & 1u) * uint32_t(P.n_parts);
  auto pclaim = [&]() -> int64_t {
    unsigned int v = 0;
    if (lane == 0) v = atomicAdd(ctr, 1u);
    return P.pool_lo + int64_t(__shfl_sync(0xffffffffu, v, 0));
  };
  // counts are published in batches of up to 4 slices: one gpu-scope fence
  // per batch orders all their sums before the counter increments
  // fp64 keeps the batch small: its ER slices need more registers
  constexpr int kBatch = sizeof(T) == 4 ? 4 : EHYB_POOL_BATCH_F64;
  uint32_t pend0 = 0, pend1 = 0, pend2 = 0, pend3 = 0;  // owners of unpublished slices
  int n_pend = 0;
  auto flush = [&]() {
    if (n_pend == 0) return;
    __threadfence();
    __syncwarp();
    if (lane == 0) {
      atomicAdd(done + pend0, 1u);
      if (n_pend > 1) atomicAdd(done + pend1, 1u);
      if (n_pend > 2) atomicAdd(done + pend2, 1u);
      if (n_pend > 3) atomicAdd(done + pend3, 1u);
    }
    n_pend = 0;
  };
  auto finish = [&](int64_t s, const ErMeta& m) {
    const int64_t pp = __ldg(P.pool_pos + (s - P.pool_lo));  // in flight with the slice
    const T acc = er_slice_compute<T, STRICT>(P, m);
    P.pool_acc[pp * 32 + lane] = acc;
    const int32_t rw0 = __shfl_sync(0xffffffffu, m.rw, 0);  // lane 0 always holds a row
    const uint32_t owner = unit_of_row<SPLIT>(P, uint32_t(rw0 & kRowMask));
    if (n_pend == 0) pend0 = owner;
    else if (n_pend == 1) pend1 = owner;
    else if (n_pend == 2) pend2 = owner;
    else pend3 = owner;
    if (++n_pend == kBatch) flush();
  };
  if (max_items > 0) {
    for (int i = 0; i < max_items; ++i) {
      const int64_t s = pclaim();
      if (s >= P.pool_hi) {
        flush();
        return false;
      }
      finish(s, er_claimed_meta(P, s, P.pool_hi, lane));
    }
    flush();
    return true;
  }
  if constexpr (EHYB_ER_PAIRS && (sizeof(T) == 4 || EHYB_ER_PAIRS_F64)) {
  for (;;) {  // two slices per claim (fp32: the pair fits the register budget)
    unsigned int v = 0;
    if (lane == 0) v = atomicAdd(ctr, 2u);
    const int64_t s = P.pool_lo + int64_t(__shfl_sync(0xffffffffu, v, 0));
    if (s >= P.pool_hi) break;
    const bool two = s + 1 < P.pool_hi;
    const ErMeta ma = er_claimed_meta(P, s, P.pool_hi, lane);
    const ErMeta mb = er_claimed_meta(P, s + 1, P.pool_hi, lane);
    const int64_t pa = __ldg(P.pool_pos + (s - P.pool_lo));
    const int64_t pb = two ? __ldg(P.pool_pos + (s + 1 - P.pool_lo)) : 0;
    T acc_a, acc_b;
    er_pair_compute<T, STRICT>(P, ma, mb, acc_a, acc_b);
    P.pool_acc[pa * 32 + lane] = acc_a;
    if (two) P.pool_acc[pb * 32 + lane] = acc_b;
    __threadfence();
    __syncwarp();
    const int32_t ra = __shfl_sync(0xffffffffu, ma.rw, 0), rb = __shfl_sync(0xffffffffu, mb.rw, 0);
    if (lane == 0) {
      atomicAdd(done + unit_of_row<SPLIT>(P, uint32_t(ra & kRowMask)), 1u);
      if (two) atomicAdd(done + unit_of_row<SPLIT>(P, uint32_t(rb & kRowMask)), 1u);
    }
  }
  } else {
  int64_t s = pclaim();
  ErMeta m = er_claimed_meta(P, s, P.pool_hi, lane);
  while (s < P.pool_hi) {  // next slice's metadata one claim ahead
    const int64_t nxt = pclaim();
    const ErMeta mn = er_claimed_meta(P, nxt, P.pool_hi, lane);
    finish(s, m);
    s = nxt;
    m = mn;
  }
}
  flush();
  return false;
}

// Pooled ER slices of one iteration group when CTAs run several partitions:
// claimed from the group's counter, two per claim (fp32), each row finished
// in place as y[r] = y_final_of_owner[r] + sum once its owner partition is
// published (part_flag == epoch). Group g's owners run in iteration g, and a
// warp drains group g only after its own CTA has finished iteration g, so
// every wait is on an earlier-or-equal iteration of another CTA: no cycle.
template <typename T, bool STRICT, bool SPLIT>
__device__ void pool_drain_group(const SpmvParams<T>& P, int lane, uint32_t ep, int g) {
  if (g < 0 || g >= P.pool_groups) return;
  const int64_t lo = __ldg(P.pool_grp + g), hi = __ldg(P.pool_grp + g + 1);
  if (hi <= lo) return;
  unsigned int* ctr = P.pool_gctr + (ep & 1u) * uint32_t(P.pool_groups) + uint32_t(g);
  auto finish = [&](const ErMeta& m, T acc) {
    if (m.rw < 0) return;
    const uint32_t r = uint32_t(m.rw & kRowMask);
    const uint32_t owner = unit_of_row<SPLIT>(P, r);
    while (ld_acquire_gpu(P.part_flag + owner) != ep) __nanosleep(64);
    P.y[r] = add_rn(__ldcg(P.y + r), acc);
  };
  constexpr unsigned kStep = (EHYB_ER_PAIRS && (sizeof(T) == 4 || EHYB_ER_PAIRS_F64_GROUP)) ? 2u : 1u;
  for (;;) {
    unsigned int v = 0;
    if (lane == 0) v = atomicAdd(ctr, kStep);
    const int64_t s = lo + int64_t(__shfl_sync(0xffffffffu, v, 0));
    if (s >= hi) break;
    const ErMeta ma = er_claimed_meta(P, s, hi, lane);
    if constexpr (kStep == 2u) {
      const ErMeta mb = er_claimed_meta(P, s + 1, hi, lane);
      T acc_a, acc_b;
      er_pair_compute<T, STRICT>(P, ma, mb, acc_a, acc_b);
      finish(ma, acc_a);
      finish(mb, acc_b);
    } else {
      finish(ma, er_slice_compute<T, STRICT>(P, ma));
    }
  }
}

// The last iteration group when pool_last_scratch: its owners run in the
// final iteration, so finishing in place would leave the whole group to the
// end of the launch. Instead every slice is computed as soon as a warp claims
// it (ER-first warps of the last iteration, then anyone after the loop) into
// the scratch and counted for its owner; the owner CTA adds the sums once
// its count is complete. Computing never waits.
template <typename T, bool STRICT, bool SPLIT>
__device__ void pool_scratch_group(const SpmvParams<T>& P, int lane, uint32_t ep, int g) {
  if (g < 0 || g >= P.pool_groups) return;
  const int64_t lo = __ldg(P.pool_grp + g), hi = __ldg(P.pool_grp + g + 1);
  if (hi <= lo) return;
  unsigned int* ctr = P.pool_gctr + (ep & 1u) * uint32_t(P.pool_groups) + uint32_t(g);
  unsigned int* done = P.pool_done + (ep & 1u) * uint32_t(P.n_parts);
  for (;;) {
    unsigned int v = 0;
    if (lane == 0) v = atomicAdd(ctr, 1u);
    const int64_t s = lo + int64_t(__shfl_sync(0xffffffffu, v, 0));
    if (s >= hi) break;
    const ErMeta m = er_claimed_meta(P, s, hi, lane);
    const int64_t pp = __ldg(P.pool_pos + (s - P.pool_lo));
    P.pool_acc[pp * 32 + lane] = er_slice_compute<T, STRICT>(P, m);
    const int32_t rw0 = __shfl_sync(0xffffffffu, m.rw, 0);  // lane 0 always holds a row
    __threadfence();
    __syncwarp();
    if (lane == 0) atomicAdd(done + unit_of_row<SPLIT>(P, uint32_t(rw0 & kRowMask)), 1u);
  }
}

__device__ __forceinline__ unsigned long long ld_acquire_gpu_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_acquire_sys_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Cross-rank waits (P2P) depend on other processes launching their matching
// SpMV; if one never does, trap instead of hanging every rank.
__device__ __forceinline__ void spin_check(unsigned long long t0, unsigned long long limit) {
  if (globaltimer() - t0 > limit) __trap();
}

// P2P halo pull of one warp: halo slots [lo, hi) (grouped by source peer)
// read from the peers' x once each peer has published this SpMV's x; then
// the pulled values are counted for the peers (served: they may overwrite x)
// and for this rank (pulled: halo rows may start).
template <typename T>
__device__ void p2p_pull(const SpmvParams<T>& P, int lane, int64_t lo, int64_t hi) {
  T* x_ext = const_cast<T*>(P.x);
  int64_t i = lo;
  while (i < hi) {
    const int src = __ldg(P.pull_src + i);
    int64_t j = i;  // end of this peer's run
    while (j < hi && __ldg(P.pull_src + j) == src) ++j;
    if (lane == 0) {
      const unsigned long long t0 = globaltimer();
      while (ld_acquire_sys_u64(P.peer_flags[src]) < P.seq) {
        __nanosleep(100);
        spin_check(t0, P.spin_timeout_ns);
      }
    }
    __syncwarp();
    const T* px = P.peer_x[src];
    for (int64_t k = i + lane; k < j; k += 32) x_ext[P.local_rows + k] = px[__ldg(P.pull_off + k)];
    __threadfence_system();
    __syncwarp();
    if (lane == 0) atomicAdd_system(P.peer_flags[src] + 1, (unsigned long long)(j - i));
    i = j;
  }
  __threadfence();
  __syncwarp();
  if (lane == 0 && hi > lo) atomicAdd(P.my_flags + 2, (unsigned long long)(hi - lo));
}

__device__ __forceinline__ int lds_volatile(const uint32_t* p, uint32_t bit) {
  return (*reinterpret_cast<const volatile uint32_t*>(p) & bit) != 0;
}

constexpr int kMaxChunks = EHYB_MAX_LOCAL_INDEX / 32;  // 32-row chunks per partition
constexpr int kMaxErBuf = 2048;                        // buffered own ER slices per CTA

// Fused EHYB SpMV, one CTA per partition.
//   SMEM : the x window is staged in shared memory (else read from global)
//   C32  : slice height 32 (warp == slice); else generic height
// Warps claim ELL chunks from a shared counter; when the counter runs dry a
// warp moves straight on to the partition's ER slices (no CTA barrier). An
// ER row whose ELL chunk is still in flight waits on that chunk's done bit,
// so y[r] = y_ell[r] + er_acc keeps the reference's order of operations.
template <typename T, int MODE, bool C32, bool SMEM, bool RING, bool P2P = false, bool SPLIT = false>
__global__ void __launch_bounds__(max_threads_for(int(sizeof(T))), 1)
    spmv_fused_kernel(const SpmvParams<T> P) {
  // EHYB_MODE_*: STRICT and DEFAULT round every slice product and add
  // separately (reference order); they differ only in the long-row path
  constexpr bool STRICT = MODE != EHYB_MODE_FMA;
  static_assert(!RING || (C32 && SMEM), "the ELL ring needs 32-row slices and a staged window");
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ uint64_t bar;
  // RING: ELL stages (runs of consecutive chunks, one bulk copy each for
  // values and columns) streamed into shared memory by one producer warp
  // (full: bytes landed; empty: every chunk of the stage consumed)
  __shared__ uint64_t rfull[RING ? kRingFB : 1], rempty[RING ? kRingNS : 1];
  __shared__ int rcount[RING ? kRingNS : 1];   // consumed chunks of the stage in the slot
  __shared__ int rsize[RING ? kRingNS : 1];    // chunks of the stage in the slot
  __shared__ int next_chunk;
  __shared__ int next_er;
  __shared__ int next_comb;
  __shared__ int next_pcomb;
  __shared__ uint32_t chunk_done[kMaxChunks / 32];
  __shared__ uint32_t er_done[kMaxErBuf / 32];
  __shared__ __align__(16) T lr_stage[64];  // long-row products (warp 0)
  const int lane = threadIdx.x & 31;
  const int wid = threadIdx.x >> 5;
  const int cta = blockIdx.x;
  const int64_t part_chunks = (P.vec + 31) >> 5;
  T* xs = reinterpret_cast<T*>(smem_raw);

  __shared__ uint32_t s_ep;
  if (threadIdx.x == 0) {
    // launch epoch (parity selects this launch's counters; the other parity
    // is reset here for the next launch, which is stream-ordered after this)
    const uint32_t e0 = *reinterpret_cast<volatile unsigned int*>(P.epoch_dev);
    s_ep = e0;
    if (P.timing) P.timing[8 * cta] = globaltimer();
    if (cta == 0 && P.pool_ctr) P.pool_ctr[(e0 + 1u) & 1u] = 0u;
    if (cta == 0 && P.lr_ctr) P.lr_ctr[(e0 + 1u) & 1u] = 0u;
    if (cta == 0 && P.pool_gctr)
      for (int g = 0; g < P.pool_groups; ++g)
        P.pool_gctr[((e0 + 1u) & 1u) * uint32_t(P.pool_groups) + uint32_t(g)] = 0u;
    if constexpr (SMEM) {
      if (P.window_tma) {
        mbar_init(&bar, 1);
        if constexpr (RING) {
          for (int i = 0; i < kRingFB; ++i) mbar_init(&rfull[i], 1);
          for (int i = 0; i < kRingNS; ++i) mbar_init(&rempty[i], 1);
        }
        fence_mbar_init();
      }
    }
  }
  __syncthreads();
  const uint32_t ep = s_ep;
  const bool persistent = int(gridDim.x) < P.n_parts;
  auto claim = [&](int* ctr) -> int64_t {
    int v = 0;
    if (lane == 0) v = atom_add_shared(ctr, 1);
    return __shfl_sync(0xffffffffu, v, 0);
  };
  // ring producer state (lane 0 of the last warp), kept across partitions
  const int prod_warp = int(blockDim.x >> 5) - 1;
  int64_t r_sbase = 0;  // stages of this CTA's earlier partitions (ring stage numbering)

  // Persistent over partitions: CTA b runs partitions b, b + grid, ... (one
  // pass when the grid covers every partition). A CTA waiting for pooled
  // slices of its partition computes pooled slices itself, and computing a
  // pooled slice never waits, so the wait always ends.
  for (int it = 0, part = cta; part < P.n_parts; ++it, part += gridDim.x) {
  // unit `part` = chunks [c0, c0 + n_chunks) of partition q; row0 is the
  // unit's first row, the window is the whole partition's
  // (SPLIT: compiled only into the variant launched when split > 1)
  const int64_t q = SPLIT ? part / P.split : (P.unit_part ? int64_t(__ldg(P.unit_part + part)) : part);
  const int64_t c0 = SPLIT ? int64_t(part - q * P.split) * P.unit_chunks : 0;
  const int64_t n_chunks =
      SPLIT ? (part_chunks - c0 < P.unit_chunks ? part_chunks - c0 : P.unit_chunks) : part_chunks;
  const int64_t unit_rows =
      SPLIT ? (P.vec - c0 * 32 < n_chunks * 32 ? P.vec - c0 * 32 : n_chunks * 32) : P.vec;
  const int64_t row0 = q * P.vec + c0 * 32;
  const T* xwin = P.x + q * P.vec;
  T* const y_lane = P.y + row0 + lane;  // this lane's row of chunk 0 of the unit
  const int64_t s0 = P.er_sel == 2 ? __ldg(P.er_part_mid + part) : __ldg(P.er_part_ptr + part);
  const int64_t s1 = P.er_sel == 1 ? __ldg(P.er_part_mid + part) : __ldg(P.er_part_ptr + part + 1);
  const uint32_t phase = uint32_t(it) & 1u;

  if (it > 0) {
    if (P.part_flag) __threadfence();  // the previous partition's y, gpu-wide
    __syncthreads();                   // every warp is done with the previous partition
    if (P.part_flag && threadIdx.x == 0) st_release_gpu(P.part_flag + (part - gridDim.x), ep);
  }
  // the window copy first (every warp is done with the previous window)
  if (threadIdx.x == 0) {
    if constexpr (SMEM) {
      if (P.window_tma) {
        // the previous partition's window was read through the generic proxy
        if (it > 0) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        const uint32_t bytes = uint32_t(P.vec * int64_t(sizeof(T)));
        mbar_expect_tx(&bar, bytes);
        for (uint32_t off = 0; off < bytes; off += kTmaChunk) {
          const uint32_t len = bytes - off < uint32_t(kTmaChunk) ? bytes - off : uint32_t(kTmaChunk);
          tma_bulk_g2s(smem_raw + off, reinterpret_cast<const unsigned char*>(xwin) + off, len,
                       &bar);
        }
      }
    }
  }
  if (threadIdx.x == 0) {
    next_chunk = 0;
    next_er = 0;
    next_comb = 0;
    next_pcomb = 0;
    if (P.pool_done)  // the next launch's counter of this partition
      P.pool_done[((ep + 1u) & 1u) * uint32_t(P.n_parts) + uint32_t(part)] = 0u;
  }
  for (int i = threadIdx.x; i < int((n_chunks + 31) >> 5); i += blockDim.x)
    chunk_done[i] = P.do_ell ? 0u : 0xffffffffu;
  for (int i = threadIdx.x; i < kMaxErBuf / 32; i += blockDim.x) er_done[i] = 0u;
  if constexpr (C32) {
    // the unit's chunk metadata, once: claims then read shared memory instead
    // of an L2 round trip per chunk
    if (P.meta_off >= 0 && P.do_ell) {
      int2* sm = reinterpret_cast<int2*>(smem_raw + P.meta_off);
      const int64_t sf = row0 >> 5;
      for (int i = threadIdx.x; i < int(n_chunks); i += blockDim.x)
        sm[i] = make_int2(__ldg(P.pos_ell + sf + i), __ldg(P.width_ell + sf + i));
    }
  }
  __syncthreads();

  if constexpr (C32) {
    // warm L2 with the first slices of the partition's ELL stream
    if (P.do_ell && P.pf_ell > 0 && wid == 0) {
      for (int64_t c = lane; c < P.pf_ell && c < n_chunks; c += 32) {
        const int64_t s = (row0 >> 5) + c;
        prefetch_slice(P.val_ell, P.col_ell, int64_t(__ldg(P.pos_ell + s)),
                       int64_t(__ldg(P.pos_ell + s + 1)));
      }
    }
  }
  // C32: each warp waits for the window inside its first ELL chunk, after
  // that chunk's loads are in flight (ell_slice32)
  bool win_pending = false;
  if constexpr (SMEM) {
    if (P.window_tma) {
      if constexpr (C32) win_pending = true;
      else mbar_wait(&bar, phase);
    } else {
      for (int64_t i = threadIdx.x; i < P.vec; i += blockDim.x) xs[i] = xwin[i];
      __syncthreads();
    }
  }
  const T* win = SMEM ? xs : xwin;
  if (P.timing && threadIdx.x == 0 && !win_pending) P.timing[8 * cta + 1] = globaltimer();
  if constexpr (P2P) {
   if (it == 0) {
    if (cta == 0 && threadIdx.x == 0) {  // this rank's x is final: peers may pull
      __threadfence_system();
      st_release_sys_u64(P.my_flags, P.seq);
    }
    const int nw = int(blockDim.x >> 5);
    if (wid >= nw - 2) {  // two pull warps per CTA, the halo split over the grid
      const int64_t per = (P.n_halo + int64_t(gridDim.x) * 2 - 1) / (int64_t(gridDim.x) * 2);
      const int64_t lo = (int64_t(cta) * 2 + (wid - (nw - 2))) * per;
      const int64_t hi = lo + per < P.n_halo ? lo + per : P.n_halo;
      if (lo < hi) p2p_pull(P, lane, lo, hi);
    }
   }
  }
  auto wait_halo = [&]() {  // every halo value of this SpMV is in x_ext
    if constexpr (!P2P) return;
    if (lane == 0) {
      const unsigned long long t0 = globaltimer();
      while (ld_acquire_gpu_u64(P.my_flags + 2) < P.seq * (unsigned long long)P.n_halo) {
        __nanosleep(64);
        spin_check(t0, P.spin_timeout_ns);
      }
    }
    __syncwarp();
  };
  // long rows first (warp 0 of every CTA): their serial chains are the
  // longest dependent work of the launch
  if (it == 0 && P.do_er && P.lr_tasks > 0 && wid == 0) {
    wait_halo();
    long_rows_warp<T, MODE>(P, lane, lr_stage, ep);
  }

  // own ER slices [s0, s1): the first n_buf are computed into a buffer at
  // any time (ER-first warps overlap them with the ELL stream) and combined
  // with y_ell at the end; the rest finish directly against y_ell
  const int64_t n_own = s1 - s0;
  // own slices beyond the shared-memory buffer go to a global scratch
  // (own_acc) when the handle has one, up to the done-bitmap capacity
  const int64_t buf_cap = P.own_acc ? int64_t(kMaxErBuf) : int64_t(P.er_buf_slices);
  // P2P: slices [n_loc, n_own) read halo values (wait for the pulls)
  const int64_t n_loc = P2P ? int64_t(__ldg(P.er_part_mid + part)) - s0 : n_own;
  const int64_t n_bufable = P2P ? n_loc : n_own;
  const int64_t n_buf = (P.do_er && P.do_ell) ? (n_bufable < buf_cap ? n_bufable : buf_cap) : 0;
  bool halo_seen = !P2P;
  auto need_halo = [&](int64_t idx) {
    if (!halo_seen && idx >= n_loc) {
      wait_halo();
      halo_seen = true;
    }
  };
  T* er_buf = reinterpret_cast<T*>(smem_raw + P.er_buf_offset);
  auto buf_at = [&](int64_t idx) -> T* {
    return idx < P.er_buf_slices ? er_buf + idx * 32 + lane
                                 : P.own_acc + (s0 + idx) * 32 + lane;
  };

  auto wait_chunk = [&](int64_t r) {
    const int64_t ch = (r - row0) >> 5;
    const uint32_t bit = 1u << (ch & 31);
    while (!lds_volatile(&chunk_done[ch >> 5], bit)) {
    }
    __threadfence_block();
  };
  // per-chunk metadata, loaded one claim ahead so its latency overlaps the
  // previous chunk's stream (narrow slices would otherwise pay two extra
  // round trips per chunk)
  struct EllMeta {
    int32_t eff;  // width | kEff* flags
    int32_t pos;
  };
  auto ell_meta = [&](int64_t chunk) -> EllMeta {
    EllMeta m{0, 0};
    if (chunk < n_chunks) {
      if constexpr (C32) {
        if (P.meta_off >= 0) {
          const int2 v = reinterpret_cast<const int2*>(smem_raw + P.meta_off)[chunk];
          m.pos = v.x;
          m.eff = v.y;
        } else {
          const int64_t s = (row0 >> 5) + chunk;
          m.eff = __ldg(P.width_ell + s);
          m.pos = __ldg(P.pos_ell + s);
        }
        const int w = m.eff & kEffWidth;
        if (lane == 0 && P.pf_ell > 0 && w > 0)  // precise L2 prefetch of the claimed chunk
          prefetch_slice(P.val_ell, P.col_ell, int64_t(m.pos), int64_t(m.pos) + 32 * int64_t(w));
      }
    }
    return m;
  };
  // Chunk completion is published one chunk late: the CTA-scope fence that
  // orders y[chunk] before its done bit runs after the warp has computed the
  // NEXT chunk, when the earlier y store has long completed — a fence right
  // after the store would stall the warp for a full store round trip.
  int64_t unpublished = -1;
  auto publish = [&]() {
    if (unpublished < 0) return;
#ifndef EHYB_NO_PUBLISH_FENCE
    __threadfence_block();
#endif
    __syncwarp();
    if (lane == 0) {
      atomicOr(&chunk_done[unpublished >> 5], 1u << (unpublished & 31));
      if (P.timing) atomicMax(P.timing + 8 * cta + 7, globaltimer());  // dev: last publication
    }
    unpublished = -1;
  };
  auto run_chunk = [&](int64_t chunk, const EllMeta& m) {
    if constexpr (C32) {
      const int w = m.eff & kEffWidth;
      const bool vec = P.ell_vec && !(m.eff & kEffHasLong);
      T acc;
      if (SMEM && win_pending) {
        if (vec)
          acc = ell_slice32_vec<T, STRICT, true>(P.val_ell, P.col_ell, int64_t(m.pos), w, lane,
                                                 win, &bar, phase);
        else
          acc = ell_slice32<T, STRICT, true>(P.val_ell, P.col_ell, int64_t(m.pos) + lane, w, win,
                                             &bar, phase);
        if (w == 0) mbar_wait(&bar, phase);
        win_pending = false;
        if (P.timing && threadIdx.x == 0) P.timing[8 * cta + 1] = globaltimer();
      } else if (vec) {
        acc = ell_slice32_vec<T, STRICT, false>(P.val_ell, P.col_ell, int64_t(m.pos), w, lane,
                                                win, nullptr, 0u);
      } else {
        acc = ell_slice32<T, STRICT, false>(P.val_ell, P.col_ell, int64_t(m.pos) + lane, w, win,
                                            nullptr, 0u);
      }
      bool store = true;
      if (m.eff & (kEffPadTail | kEffHasLong)) {
        // a slice narrowed by a long row: the reference's remaining padding
        // products 0*win[0] (idempotent, so one stands for all of them); the
        // long row's own lane is written by the long-row path
        if (m.eff & kEffPadTail) acc = add_rn(acc, mul_rn(T(0), win[0]));
        store = !((__ldg(P.long_bits + (row0 >> 5) + chunk) >> lane) & 1u);
      }
      publish();
      if (store) y_lane[int(chunk) * 32] = acc;
      // only slices with an ER row are waited on (wait_chunk / own_pre)
      unpublished = (m.eff & kEffHasEr) ? chunk : -1;
    } else {
      const int64_t lr = chunk * 32 + lane;
      T acc = T(0);
      bool skip = lr >= unit_rows;
      if (!skip) {
        const int64_t r = row0 + lr;
        const int64_t C = P.warp;
        const int64_t s = r / C;
        const int32_t eff = __ldg(P.width_ell + s);
        const int64_t pos = int64_t(__ldg(P.pos_ell + s)) + (r - s * C);
        acc = ell_row_generic<T, STRICT>(P.val_ell, P.col_ell, pos, eff & kEffWidth, C, win);
        if (eff & kEffPadTail) acc = add_rn(acc, mul_rn(T(0), win[0]));
        if (eff & kEffHasLong) skip = (__ldg(P.long_bits + (r >> 5)) >> (r & 31)) & 1u;
      }
      publish();
      if (!skip) P.y[row0 + lr] = acc;
      unpublished = chunk;
    }
  };
  auto er_meta = [&](int64_t s, int64_t s_end) { return er_claimed_meta(P, s, s_end, lane); };
  // a row whose ELL value is already final has y read before the slice's
  // loads, so that round trip overlaps them
  auto own_pre = [&](int64_t idx, const ErMeta& m, T& yv) -> bool {
    need_halo(idx);
    const bool direct = idx >= n_buf && m.rw >= 0;
    bool have_y = false;
    if (direct) {
      const int64_t r = m.rw & kRowMask;
      if (!P.do_ell) {
        have_y = true;
      } else {
        const int64_t ch = (r - row0) >> 5;
        if (lds_volatile(&chunk_done[ch >> 5], 1u << (ch & 31))) {
          __threadfence_block();
          have_y = true;
        }
      }
      if (have_y) yv = __ldcg(P.y + r);
    }
    return have_y;
  };
  auto own_post = [&](int64_t idx, const ErMeta& m, T acc, T yv, bool have_y) {
    if (idx < n_buf) {
      *buf_at(idx) = acc;
      __threadfence_block();
      __syncwarp();
      if (lane == 0) atomicOr(&er_done[idx >> 5], 1u << (idx & 31));
    } else if (m.rw >= 0) {
      const int64_t r = m.rw & kRowMask;
      if (!have_y) {
        wait_chunk(r);
        yv = __ldcg(P.y + r);
      }
      P.y[r] = add_rn(yv, acc);
    }
  };
  auto finish_own_er = [&](int64_t idx, const ErMeta& m) {
    need_halo(idx);
    const bool direct = idx >= n_buf && m.rw >= 0;
    const int64_t r = m.rw & kRowMask;
    T yv = T(0);
    const bool have_y = own_pre(idx, m, yv);
    const T acc = er_slice_compute<T, STRICT>(P, m);
    if (idx < n_buf) {
      *buf_at(idx) = acc;
      __threadfence_block();
      __syncwarp();
      if (lane == 0) atomicOr(&er_done[idx >> 5], 1u << (idx & 31));
    } else if (direct) {
      if (!have_y) {
        wait_chunk(r);
        yv = __ldcg(P.y + r);
      }
      P.y[r] = add_rn(yv, acc);
    }
  };

  int64_t pending = -1;
  if (P.do_er && P.do_ell && wid < P.er_warps && !(RING && wid == prod_warp)) {  // ER-first warps
    if (n_buf > 0) {
      for (;;) {
        const int64_t idx = claim(&next_er);
        if (idx >= n_buf) {
          pending = idx;
          break;
        }
        finish_own_er(idx, er_meta(s0 + idx, s1));
      }
    }
    // pooled slices of every partition, hidden behind the other warps' ELL
    // stream; with several partitions per CTA, the group whose owners ran in
    // the previous iteration
    if (!persistent) pool_drain<T, STRICT, SPLIT>(P, lane, 0, ep);
    else if (P.part_flag) {
      pool_drain_group<T, STRICT, SPLIT>(P, lane, ep, it - 1);
      if (P.pool_last_scratch && it == P.pool_groups - 1) pool_scratch_group<T, STRICT, SPLIT>(P, lane, ep, it);
    }
  }
  const int64_t st_lo = RING ? int64_t(__ldg(P.part_stage_ptr + part)) : 0;
  const int64_t n_st = RING ? int64_t(__ldg(P.part_stage_ptr + part + 1)) - st_lo : 0;
  if (RING && P.do_ell && wid == prod_warp) {
    // producer: stage sg = r_sbase + t into data slot sg % ring_stages once
    // the slot's previous stage is consumed; one bulk copy per region
    unsigned char* rbase = smem_raw + P.ring_offset;
    const int64_t ns = P.ring_stages;
    int32_t m_pos = 0, m_slots = 0, m_nch = 0;
    for (int64_t t = 0; t < n_st; ++t) {
      if ((t & 31) == 0) {  // the next 32 stages' plan, one load per lane
        const bool ok = t + lane < n_st;
        m_pos = ok ? __ldg(P.st_pos + st_lo + t + lane) : 0;
        m_slots = ok ? __ldg(P.st_slots + st_lo + t + lane) : 0;
        m_nch = ok ? __ldg(P.st_chunks + st_lo + t + lane) : 0;
      }
      const int32_t pos = __shfl_sync(0xffffffffu, m_pos, int(t & 31));
      const int32_t slots = __shfl_sync(0xffffffffu, m_slots, int(t & 31));
      const int32_t nch = __shfl_sync(0xffffffffu, m_nch, int(t & 31));
      if (lane == 0) {
        const int64_t sg = r_sbase + t;
        const int sl = int(sg % ns);
        if (sg >= ns) {
          const unsigned long long tw = P.timing ? globaltimer() : 0ull;
          mbar_wait(&rempty[sl], uint32_t(sg / ns - 1) & 1u);
          if (P.timing) {  // dev profile: producer time blocked on a full ring, waits
            atomicAdd(P.timing + 8 * cta + 5, globaltimer() - tw);
            atomicAdd(P.timing + 8 * cta + 6, 1ull);
          }
        }
        unsigned char* dst = rbase + int64_t(sl) * P.stage_bytes;
        rcount[sl] = 0;
        rsize[sl] = nch;
        uint64_t* fb = &rfull[sg % kRingFB];
        if (slots > 0) {
          const uint32_t vb = uint32_t(slots) * uint32_t(sizeof(T)), cb = uint32_t(slots) * 2u;
          mbar_expect_tx(fb, vb + cb);
          tma_bulk_g2s(dst, P.val_ell + pos, vb, fb);
          tma_bulk_g2s(dst + P.stage_vbytes, P.col_ell + pos, cb, fb);
        } else {
          mbar_arrive(fb);
        }
      }
    }
    if (P.timing && lane == 0) P.timing[8 * cta + 2] = globaltimer();
    __syncwarp();
  } else if (RING && P.do_ell) {
    // consumers: chunks in claim order, read from their stage in the ring
    // (chunk metadata one claim ahead)
    const unsigned char* rbase = smem_raw + P.ring_offset;
    const int64_t ns = P.ring_stages;
    auto rmeta = [&](int64_t c, int32_t& eff, uint2& cs) {
      if (c < n_chunks) {
        eff = __ldg(P.width_ell + (row0 >> 5) + c);
        cs = __ldg(P.ch_stage + (row0 >> 5) + c);
      }
    };
    int64_t chunk = claim(&next_chunk);
    int32_t eff = 0;
    uint2 cs = make_uint2(0u, 0u);
    rmeta(chunk, eff, cs);
    while (chunk < n_chunks) {
      const int64_t nxt = claim(&next_chunk);
      int32_t eff_n = 0;
      uint2 cs_n = make_uint2(0u, 0u);
      rmeta(nxt, eff_n, cs_n);
      const int64_t sg = r_sbase + int64_t(cs.x);
      mbar_wait(&rfull[sg % kRingFB], uint32_t(sg / kRingFB) & 1u);
      const int sl = int(sg % ns);
      const int w = eff & kEffWidth;
      const unsigned char* base = rbase + int64_t(sl) * P.stage_bytes;
      const T* sv = reinterpret_cast<const T*>(base) + cs.y;
      const uint16_t* sc = reinterpret_cast<const uint16_t*>(base + P.stage_vbytes) + cs.y;
      if (win_pending) {
        mbar_wait(&bar, phase);
        win_pending = false;
        if (P.timing && threadIdx.x == 0) P.timing[8 * cta + 1] = globaltimer();
      }
      T acc = ell_slice32_smem<T, STRICT>(sv + lane, sc + lane, w, win);
      __syncwarp();
      if (lane == 0 && atomicAdd(&rcount[sl], 1) == rsize[sl] - 1)
        mbar_arrive(&rempty[sl]);  // the whole stage is consumed
      bool store = true;
      if (eff & (kEffPadTail | kEffHasLong)) {
        if (eff & kEffPadTail) acc = add_rn(acc, mul_rn(T(0), win[0]));
        store = !((__ldg(P.long_bits + (row0 >> 5) + chunk) >> lane) & 1u);
      }
      publish();
      if (store) P.y[row0 + chunk * 32 + lane] = acc;
      unpublished = chunk;
      chunk = nxt;
      eff = eff_n;
      cs = cs_n;
    }
    publish();
  } else if (P.do_ell) {
    int64_t chunk = claim(&next_chunk);
    if (P.ell_ahead) {
      EllMeta m = ell_meta(chunk);
      while (chunk < n_chunks) {
        const int64_t nxt = claim(&next_chunk);
        const EllMeta mn = ell_meta(nxt);
        run_chunk(chunk, m);
        chunk = nxt;
        m = mn;
      }
    } else {
      for (; chunk < n_chunks; chunk = claim(&next_chunk)) run_chunk(chunk, ell_meta(chunk));
    }
    publish();  // this warp's last chunk
    // the warp whose claim first ran past the end stamps the end of ELL issue
    if (P.timing && lane == 0 && chunk == n_chunks) P.timing[8 * cta + 2] = globaltimer();
  }

  if (P.do_er) {
    if (pending >= 0 && pending < n_own) finish_own_er(pending, er_meta(s0 + pending, s1));
    if constexpr (EHYB_ER_PAIRS && (sizeof(T) == 4 || EHYB_ER_PAIRS_F64)) {
    for (;;) {  // two own slices per claim (fp32: the pair fits the register budget)
      int v = 0;
      if (lane == 0) v = atom_add_shared(&next_er, 2);
      const int64_t idx = __shfl_sync(0xffffffffu, v, 0);
      if (idx >= n_own) break;
      const ErMeta ma = er_meta(s0 + idx, s1), mb = er_meta(s0 + idx + 1, s1);
      T ya = T(0), yb = T(0);
      const bool ha = own_pre(idx, ma, ya);
      const bool hb = idx + 1 < n_own ? own_pre(idx + 1, mb, yb) : false;
      T acc_a, acc_b;
      er_pair_compute<T, STRICT>(P, ma, mb, acc_a, acc_b);
      own_post(idx, ma, acc_a, ya, ha);
      if (idx + 1 < n_own) own_post(idx + 1, mb, acc_b, yb, hb);
    }
    } else if (P.er_ahead) {
      int64_t idx = claim(&next_er);
      ErMeta m = er_meta(s0 + idx, s1);
      while (idx < n_own) {
        const int64_t nxt = claim(&next_er);
        const ErMeta mn = er_meta(s0 + nxt, s1);
        finish_own_er(idx, m);
        idx = nxt;
        m = mn;
      }
    } else {
      for (int64_t idx = claim(&next_er); idx < n_own; idx = claim(&next_er))
        finish_own_er(idx, er_meta(s0 + idx, s1));
    }

    auto stamp = [&](int i) {
      if (P.timing && lane == 0 && !(RING && (i == 5 || i == 6)))
        atomicMax(P.timing + 8 * cta + i, globaltimer());
    };
    stamp(4);
    if (!persistent) pool_drain<T, STRICT, SPLIT>(P, lane, 0, ep);  // whatever the ER-first warps left
    // combine the buffered own ER rows: y[r] = y_ell[r] + er_acc, two
    // slices per claim so their row and y reads overlap
    constexpr int kCs = sizeof(T) == 8 ? 2 : 1;  // fp32: one per claim (register budget)
    for (;;) {
      int v = 0;
      if (lane == 0) v = atom_add_shared(&next_comb, kCs);
      const int64_t idx = __shfl_sync(0xffffffffu, v, 0);
      if (idx >= n_buf) break;
      const bool two = kCs == 2 && idx + 1 < n_buf;
      const int32_t rw = __ldg(P.er_rows + (s0 + idx) * 32 + lane);
      const int32_t rw2 = two ? __ldg(P.er_rows + (s0 + idx + 1) * 32 + lane) : -1;
      while (!lds_volatile(&er_done[idx >> 5], 1u << (idx & 31))) {
      }
      if (two)
        while (!lds_volatile(&er_done[(idx + 1) >> 5], 1u << ((idx + 1) & 31))) {
        }
      __threadfence_block();
      T y1 = T(0), y2 = T(0);
      if (rw >= 0) {
        wait_chunk(rw & kRowMask);
        y1 = __ldcg(P.y + (rw & kRowMask));
      }
      if (rw2 >= 0) {
        wait_chunk(rw2 & kRowMask);
        y2 = __ldcg(P.y + (rw2 & kRowMask));
      }
      if (rw >= 0)
        P.y[rw & kRowMask] = add_rn(y1, idx < P.er_buf_slices ? er_buf[idx * 32 + lane]
                                                              : __ldcg(buf_at(idx)));
      if (rw2 >= 0)
        P.y[rw2 & kRowMask] = add_rn(y2, idx + 1 < P.er_buf_slices ? er_buf[(idx + 1) * 32 + lane]
                                                                   : __ldcg(buf_at(idx + 1)));
    }
    stamp(5);
    // pooled slices of this partition: once all are in, y[r] = y_ell[r] + sum
    // (a CTA that runs several partitions does this once, after all of them)
    const int32_t q0 = (P.pool_own_ptr && !persistent) ? __ldg(P.pool_own_ptr + part) : 0;
    const int32_t q1 = (P.pool_own_ptr && !persistent) ? __ldg(P.pool_own_ptr + part + 1) : 0;
    if (q1 > q0) {
      const unsigned int* done =
          P.pool_done + (ep & 1u) * uint32_t(P.n_parts) + uint32_t(part);
      // every pooled slice is claimed by now (this warp drained the pool
      // above), so only slices still in flight elsewhere remain
      while (ld_acquire_gpu(done) != unsigned(q1 - q0)) __nanosleep(128);
      // owner-major scratch: the row and its sum in one round trip, two
      // pooled slices per claim so their reads overlap
      // (fp32 keeps one slice per claim: measured 111.9 vs 120.3 us on cfg3)
      constexpr int kPs = sizeof(T) == 8 ? 2 : 1;
      for (;;) {
        int v = 0;
        if (lane == 0) v = atom_add_shared(&next_pcomb, kPs);
        const int64_t idx = __shfl_sync(0xffffffffu, v, 0);
        if (idx >= q1 - q0) break;
        const bool two = kPs == 2 && idx + 1 < q1 - q0;
        const int64_t o = (q0 + idx) * 32 + lane;
        const int32_t rw = __ldg(P.pool_rows + o);
        const T acc = __ldcg(P.pool_acc + o);
        const int32_t rw2 = two ? __ldg(P.pool_rows + o + 32) : -1;
        const T acc2 = two ? __ldcg(P.pool_acc + o + 32) : T(0);
        T y1 = T(0), y2 = T(0);
        if (rw >= 0) {
          wait_chunk(rw & kRowMask);
          y1 = __ldcg(P.y + (rw & kRowMask));
        }
        if (rw2 >= 0) {
          wait_chunk(rw2 & kRowMask);
          y2 = __ldcg(P.y + (rw2 & kRowMask));
        }
        if (rw >= 0) P.y[rw & kRowMask] = add_rn(y1, acc);
        if (rw2 >= 0) P.y[rw2 & kRowMask] = add_rn(y2, acc2);
      }
    }
    stamp(6);
  }
  r_sbase += n_st;
  }  // partitions of this CTA

  if (persistent && P.do_er && P.part_flag) {
    // publish the last partition, then every group left (the last two at
    // least) — rows finished in place as their owners are published
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
      int last = cta;
      while (last + int(gridDim.x) < P.n_parts) last += gridDim.x;
      st_release_gpu(P.part_flag + last, ep);
    }
    const int g_end = P.pool_last_scratch ? P.pool_groups - 1 : P.pool_groups;
    for (int g = 0; g < g_end; ++g) pool_drain_group<T, STRICT, SPLIT>(P, lane, ep, g);
    if (P.pool_last_scratch) {
      const int gl = P.pool_groups - 1;
      pool_scratch_group<T, STRICT, SPLIT>(P, lane, ep, gl);
      const int pl = cta + gl * int(gridDim.x);  // this CTA's partition in the last group
      if (pl < P.n_parts) {
        const int32_t q0 = __ldg(P.pool_own_ptr + pl), q1 = __ldg(P.pool_own_ptr + pl + 1);
        if (q1 > q0) {
          const unsigned int* done = P.pool_done + (ep & 1u) * uint32_t(P.n_parts) + uint32_t(pl);
          if (lane == 0)
            while (ld_acquire_gpu(done) != unsigned(q1 - q0)) __nanosleep(64);
          __syncwarp();
          for (int64_t t = wid; t < q1 - q0; t += int64_t(blockDim.x >> 5)) {
            const int64_t o = (q0 + t) * 32 + lane;
            const int32_t rw = __ldg(P.pool_rows + o);
            const T acc = __ldcg(P.pool_acc + o);
            if (rw >= 0) {
              const int64_t r = rw & kRowMask;
              P.y[r] = add_rn(__ldcg(P.y + r), acc);
            }
          }
        }
      }
    }
  } else if (persistent && P.do_er && P.pool_own_ptr) {
    pool_drain<T, STRICT, SPLIT>(P, lane, 0, ep);
    __syncthreads();
    for (int64_t t = claim(&next_pcomb);; t = claim(&next_pcomb)) {
      int64_t base = 0;
      int pt = -1;
      int32_t q0 = 0, cnt = 0;
      for (int p = cta; p < P.n_parts; p += gridDim.x) {
        q0 = __ldg(P.pool_own_ptr + p);
        cnt = __ldg(P.pool_own_ptr + p + 1) - q0;
        if (t < base + cnt) {
          pt = p;
          break;
        }
        base += cnt;
      }
      if (pt < 0) break;
      const unsigned int* done = P.pool_done + (ep & 1u) * uint32_t(P.n_parts) + uint32_t(pt);
      while (ld_acquire_gpu(done) != unsigned(cnt)) __nanosleep(128);
      const int64_t o = (q0 + (t - base)) * 32 + lane;
      const int32_t rw = __ldg(P.pool_rows + o);
      const T acc = __ldcg(P.pool_acc + o);
      if (rw >= 0) {
        const int64_t r = rw & kRowMask;
        P.y[r] = add_rn(__ldcg(P.y + r), acc);
      }
    }
  }

  __syncthreads();
  if (P2P && cta == 0 && threadIdx.x == 0) {
    // this rank's x may be overwritten by the next stream operation only
    // once every peer has pulled its halo values from it
    const unsigned long long t0 = globaltimer();
    while (ld_acquire_sys_u64(P.my_flags + 1) < P.seq * P.served_per_spmv) {
      __nanosleep(100);
      spin_check(t0, P.spin_timeout_ns);
    }
  }
  if (threadIdx.x == 0) {
    if (P.timing) P.timing[8 * cta + 3] = globaltimer();
    // the last CTA to finish advances the launch epoch
    __threadfence();
    if (atomicAdd(P.epoch_dev + 1, 1u) == gridDim.x - 1) {
      P.epoch_dev[1] = 0u;
      P.epoch_dev[0] = ep + 1u;
    }
  }
}

// Shards whose x does not hold the ER padding column (global column 0 lives
// on another rank): their ER rows skip the reference's padding products
// 0*x[0] in the launch, and this pass applies them once the halo (which then
// carries that column) is in. z = 0*x[pad] is -0.0, +0.0 or NaN; adding it
// to the row's ER sum before y = y_ell + er_sum changes y only if z is NaN
// (y becomes NaN) or z is +0.0 and y came out -0.0 (both terms -0.0: the
// reference gets +0.0). Exact for every x, one read of z per thread.
template <typename T>
__global__ void pad_fixup_kernel(T* __restrict__ y, const int32_t* __restrict__ rows, int64_t n,
                                 const T* __restrict__ xpad) {
  const T z = mul_rn(T(0), __ldg(xpad));
  const bool is_nan = z != z;
  if (!is_nan && signbit(z)) return;  // -0.0 is the identity of the add
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int32_t r = __ldg(rows + i);
    const T v = y[r];
    if (is_nan) y[r] = add_rn(v, z);
    else if (v == T(0) && signbit(v)) y[r] = T(0);
  }
}

// ------------------------------------------- CSR product, reference order
// The reference oracle spmv_csr (engine.py:56-69): fp64 products
// v[j] * x[c[j]], then np.add.reduceat over each non-empty row. numpy's
// reduce loop seeds the row sum with its first product and adds the pairwise
// sum of the rest (numpy's pairwise_sum: < 8 terms sequential from -0.0,
// <= 128 terms in 8 strided accumulators combined as a fixed tree plus a
// sequential tail, longer runs split at n/2 rounded down to a multiple of 8).
// Reproduced term for term, so y is bitwise the reference's.
__device__ __forceinline__ double csr_term(const double* __restrict__ v,
                                           const int32_t* __restrict__ c,
                                           const double* __restrict__ x, int64_t j) {
  return __dmul_rn(__ldg(v + j), __ldg(x + __ldg(c + j)));
}

__device__ double csr_pairwise(const double* __restrict__ v, const int32_t* __restrict__ c,
                               const double* __restrict__ x, int64_t a, int64_t n) {
  // iterative form of the recursion: an explicit stack of pending right
  // halves and of finished left sums (depth <= 2 log2(n / 128) + 2)
  struct Frame {
    int64_t a, n;
    int state;  // 0: not started, 1: left done (sum in `left`)
    double left;
  };
  Frame st[64];
  int sp = 0;
  st[0] = {a, n, 0, 0.0};
  double ret = 0.0;
  for (;;) {
    Frame& f = st[sp];
    if (f.n > 128 && f.state == 0) {
      int64_t n2 = f.n / 2;
      n2 -= n2 % 8;
      f.state = 1;
      st[sp + 1] = {f.a, n2, 0, 0.0};
      ++sp;
      continue;
    }
    if (f.n > 128 && f.state == 1) {  // left half finished in `ret`
      int64_t n2 = f.n / 2;
      n2 -= n2 % 8;
      f.left = ret;
      f.state = 2;
      st[sp + 1] = {f.a + n2, f.n - n2, 0, 0.0};
      ++sp;
      continue;
    }
    if (f.n > 128) {  // state 2: right half finished in `ret`
      ret = __dadd_rn(f.left, ret);
    } else if (f.n < 8) {
      double res = -0.0;
      for (int64_t i = 0; i < f.n; ++i) res = __dadd_rn(res, csr_term(v, c, x, f.a + i));
      ret = res;
    } else {
      double r[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) r[u] = csr_term(v, c, x, f.a + u);
      int64_t i = 8;
      for (; i < f.n - (f.n % 8); i += 8) {
#pragma unroll
        for (int u = 0; u < 8; ++u) r[u] = __dadd_rn(r[u], csr_term(v, c, x, f.a + i + u));
      }
      double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                             __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
      for (; i < f.n; ++i) res = __dadd_rn(res, csr_term(v, c, x, f.a + i));
      ret = res;
    }
    if (sp == 0) return ret;
    --sp;
  }
}

// one thread per row; empty rows are 0.0 (the reference's np.zeros)
__global__ void csr_ref_kernel(const int32_t* __restrict__ row_ptr, const int32_t* __restrict__ col,
                               const double* __restrict__ val, const double* __restrict__ x,
                               int64_t n_rows, double* __restrict__ y) {
  for (int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; r < n_rows;
       r += int64_t(gridDim.x) * blockDim.x) {
    const int64_t a = __ldg(row_ptr + r), b = __ldg(row_ptr + r + 1);
    double s = 0.0;
    if (b > a) {
      s = csr_term(val, col, x, a);
      if (b - a > 1) s = __dadd_rn(s, csr_pairwise(val, col, x, a + 1, b - a - 1));
    }
    y[r] = s;
  }
}

// ---------------------------------------------------------- vector kernels
template <typename T>
__global__ void permute_kernel(const T* __restrict__ x_user, const int32_t* __restrict__ inverse,
                               int64_t n, int64_t padded, T* __restrict__ x_r) {
  #pragma unroll 4  // independent iterations: loads of 4 elements in flight per thread
  for (int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; j < padded;
       j += int64_t(gridDim.x) * blockDim.x) {
    const int64_t src = __ldg(inverse + j);
    x_r[j] = src < n ? __ldg(x_user + src) : T(0);
  }
}

template <typename T>
__global__ void unpermute_kernel(const T* __restrict__ y_r, const int32_t* __restrict__ reorder,
                                 int64_t n, T* __restrict__ y_user) {
  #pragma unroll 4  // independent iterations: loads of 4 elements in flight per thread
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    y_user[i] = __ldg(y_r + __ldg(reorder + i));
}

template <typename T>
__global__ void gather_kernel(const T* __restrict__ src, const int64_t* __restrict__ idx,
                              int64_t count, T* __restrict__ dst) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < count;
       i += int64_t(gridDim.x) * blockDim.x)
    dst[i] = __ldg(src + __ldg(idx + i));
}

// deterministic two-level dot: fixed grid, per-block tree, then one block
template <typename T>
__global__ void dot_partial_kernel(const T* __restrict__ a, const T* __restrict__ b, int64_t n,
                                   double* __restrict__ partial) {
  __shared__ double red[32];
  double s = 0.0;
  #pragma unroll 4  // independent iterations: loads of 4 elements in flight per thread
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    s += double(a[i]) * double(b[i]);
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    s = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (threadIdx.x == 0) partial[blockIdx.x] = s;
  }
}

__global__ void dot_final_kernel(const double* __restrict__ partial, int n,
                                 double* __restrict__ out) {
  __shared__ double red[32];
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += partial[i];
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    s = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (threadIdx.x == 0) out[0] = s;
  }
}

// CG vector updates with the scalars kept on the device (no host round trip
// per iteration). scal = {rr, pq}: alpha = rr / pq; x += alpha p; r -= alpha q;
// the block partials of r.r go to `partial` (reduced by dot_final_kernel).
template <typename T>
__global__ void cg_xr_kernel(T* __restrict__ x, T* __restrict__ r, const T* __restrict__ p,
                             const T* __restrict__ q, const double* __restrict__ rr,
                             const double* __restrict__ pq, int64_t n,
                             double* __restrict__ partial) {
  __shared__ double red[32];
  const double alpha = rr[0] / pq[0];
  const T a = T(alpha);
  double s = 0.0;
  #pragma unroll 4  // independent iterations: loads of 4 elements in flight per thread
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    x[i] = x[i] + a * p[i];
    const T ri = r[i] - a * q[i];
    r[i] = ri;
    s += double(ri) * double(ri);
  }
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    s = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (threadIdx.x == 0) partial[blockIdx.x] = s;
  }
}

// p = r + (rr_new / rr_old) p
template <typename T>
__global__ void cg_p_kernel(T* __restrict__ p, const T* __restrict__ r,
                            const double* __restrict__ rr_new, const double* __restrict__ rr_old,
                            int64_t n) {
  const T beta = T(rr_new[0] / rr_old[0]);
  #pragma unroll 4  // independent iterations: loads of 4 elements in flight per thread
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    p[i] = r[i] + beta * p[i];
}

// Two dot products in one pass (Chronopoulos-Gear CG needs (r,r) and (w,r)
// together): block partials, reduced by dot2_final_kernel.
template <typename T>
__global__ void dot2_partial_kernel(const T* __restrict__ a, const T* __restrict__ b,
                                    const T* __restrict__ c, const T* __restrict__ d, int64_t n,
                                    double* __restrict__ partial) {
  __shared__ double red[2][32];
  double s0 = 0.0, s1 = 0.0;
  #pragma unroll 4  // independent iterations: loads of 4 elements in flight per thread
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    s0 += double(a[i]) * double(b[i]);
    s1 += double(c[i]) * double(d[i]);
  }
  for (int o = 16; o; o >>= 1) {
    s0 += __shfl_xor_sync(0xffffffffu, s0, o);
    s1 += __shfl_xor_sync(0xffffffffu, s1, o);
  }
  if ((threadIdx.x & 31) == 0) {
    red[0][threadIdx.x >> 5] = s0;
    red[1][threadIdx.x >> 5] = s1;
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    const bool ok = threadIdx.x < (blockDim.x >> 5);
    s0 = ok ? red[0][threadIdx.x] : 0.0;
    s1 = ok ? red[1][threadIdx.x] : 0.0;
    for (int o = 16; o; o >>= 1) {
      s0 += __shfl_xor_sync(0xffffffffu, s0, o);
      s1 += __shfl_xor_sync(0xffffffffu, s1, o);
    }
    if (threadIdx.x == 0) {
      partial[2 * blockIdx.x] = s0;
      partial[2 * blockIdx.x + 1] = s1;
    }
  }
}

__global__ void dot2_final_kernel(const double* __restrict__ partial, int n,
                                  double* __restrict__ out) {
  __shared__ double red[2][32];
  double s0 = 0.0, s1 = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    s0 += partial[2 * i];
    s1 += partial[2 * i + 1];
  }
  for (int o = 16; o; o >>= 1) {
    s0 += __shfl_xor_sync(0xffffffffu, s0, o);
    s1 += __shfl_xor_sync(0xffffffffu, s1, o);
  }
  if ((threadIdx.x & 31) == 0) {
    red[0][threadIdx.x >> 5] = s0;
    red[1][threadIdx.x >> 5] = s1;
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    const bool ok = threadIdx.x < (blockDim.x >> 5);
    s0 = ok ? red[0][threadIdx.x] : 0.0;
    s1 = ok ? red[1][threadIdx.x] : 0.0;
    for (int o = 16; o; o >>= 1) {
      s0 += __shfl_xor_sync(0xffffffffu, s0, o);
      s1 += __shfl_xor_sync(0xffffffffu, s1, o);
    }
    if (threadIdx.x == 0) {
      out[0] = s0;
      out[1] = s1;
    }
  }
}

// Chronopoulos-Gear CG scalars, kept on the device. sc = {gamma = (r,r),
// delta = (w,r) (both all-reduced), gamma_old, alpha, beta}:
// first iteration beta = 0, alpha = gamma/delta; then beta = gamma/gamma_old,
// alpha = gamma / (delta - beta*gamma/alpha_old).
__global__ void cgcg_scalars_kernel(double* __restrict__ sc, int first) {
  const double g = sc[0], d = sc[1];
  double beta = 0.0, alpha;
  if (first) {
    alpha = g / d;
  } else {
    beta = g / sc[2];
    alpha = g / (d - beta * g / sc[3]);
  }
  sc[2] = g;
  sc[3] = alpha;
  sc[4] = beta;
}

// p = r + beta p; s = w + beta s; x += alpha p; r -= alpha s
template <typename T>
__global__ void cgcg_update_kernel(T* __restrict__ x, T* __restrict__ r, T* __restrict__ p,
                                   T* __restrict__ s, const T* __restrict__ w,
                                   const double* __restrict__ sc, int64_t n) {
  const T alpha = T(sc[3]), beta = T(sc[4]);
  #pragma unroll 4  // independent iterations: loads of 4 elements in flight per thread
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const T pi = r[i] + beta * p[i];
    const T si = w[i] + beta * s[i];
    p[i] = pi;
    s[i] = si;
    x[i] = x[i] + alpha * pi;
    r[i] = r[i] - alpha * si;
  }
}

template <typename T>
__global__ void axpy_kernel(const double* __restrict__ a, double sign, const T* __restrict__ x,
                            T* __restrict__ y, int64_t n) {
  const T alpha = T(sign * a[0]);
  #pragma unroll 4  // independent iterations: loads of 4 elements in flight per thread
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    y[i] = y[i] + alpha * x[i];
}

}  // namespace ehyb
