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
  const int64_t* __restrict__ er_pos;       // [n_slices] slot offset of each slice
  const int32_t* __restrict__ er_swidth;    // [n_slices] slice width
  const int32_t* __restrict__ er_rows;      // [n_slices*32] row | kPadFlag, -1 = empty lane
  const int32_t* __restrict__ er_lwidth;    // [n_slices*32] lane width
  const T* __restrict__ er_val;
  const uint32_t* __restrict__ er_col;
  const T* __restrict__ x;  // reordered (or [owned | halo]) input
  T* __restrict__ y;        // reordered (or owned) output
  int64_t vec;
  int32_t warp;             // slice height C of the ELL body
  int32_t window_in_smem;
  int32_t window_tma;
  int32_t do_ell;
  int32_t do_er;
  int32_t pf_ell;            // ELL slices kept in flight ahead of the warps by L2 bulk prefetch (0 = off)
  int32_t pf_er;             // 1 = L2 bulk prefetch of the next ER slice per warp
  unsigned long long* timing;  // optional per-CTA %globaltimer stamps [start, window, ell, end]
  // ER work pool shared by all CTAs (load balance across partitions)
  int64_t pool_lo, pool_hi;         // global slice range of the pool
  unsigned int* pool_ctr;           // [2] claim counters, alternating by epoch
  unsigned int* part_flag;          // [n_parts] epoch whose ELL phase the partition published
  unsigned int epoch;               // launch sequence number (>= 1)
  // own-ER shared-memory buffer (overlap of ER gathers with the ELL stream)
  int32_t er_buf_slices;            // buffered own ER slices (<= kMaxErBuf)
  int32_t er_buf_offset;            // byte offset of the buffer in dynamic smem
  int32_t er_warps;                 // warps that start on ER before ELL
  int32_t ell_ahead;                // 1 = claim the next ELL chunk (and its metadata) one ahead
  int32_t er_ahead;                 // 1 = same for ER slices
  int32_t er_mix;                   // 1 = own buffered ER slices interleaved with ELL chunks
};

constexpr int32_t kPadFlag = 0x40000000;  // row had reference ER padding slots
constexpr int32_t kRowMask = 0x3fffffff;

// ------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
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
template <typename T>
struct EllUnroll {
  static constexpr int value = sizeof(T) == 4 ? 16 : 8;
};

template <typename T, bool STRICT>
__device__ __forceinline__ T ell_slice32(const T* __restrict__ val,
                                         const uint16_t* __restrict__ col, int64_t pos, int w,
                                         const T* win, uint64_t* win_bar) {
  constexpr int U = EllUnroll<T>::value;
  T acc = T(0);
  int k = 0;
  for (; k + U <= w; k += U) {
    uint32_t c[U];
    T v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) c[u] = __ldcs(col + pos + int64_t(k + u) * 32);
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldcs(val + pos + int64_t(k + u) * 32);
    // a warp's first chunk issues its stream loads before the window has
    // landed: the TMA copy and the first HBM round trip overlap
    if (win_bar) {
      mbar_wait(win_bar, 0);
      win_bar = nullptr;
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
        c[u] = __ldcs(col + pos + int64_t(k + u) * 32);
        v[u] = __ldcs(val + pos + int64_t(k + u) * 32);
      }
    }
    if (win_bar) mbar_wait(win_bar, 0);
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (k + u < w) acc = madd<STRICT>(acc, v[u], win[c[u]]);
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
  if (m.rw >= 0 && (m.rw & kPadFlag)) acc = add_rn(acc, mul_rn(T(0), __ldg(P.x)));
  return acc;
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
template <typename T, bool STRICT, bool C32, bool SMEM>
__global__ void __launch_bounds__(1024, 1) spmv_fused_kernel(const SpmvParams<T> P) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ uint64_t bar;
  __shared__ int next_chunk;
  __shared__ int next_er;
  __shared__ int next_comb;
  __shared__ int ell_finished;
  __shared__ uint32_t chunk_done[kMaxChunks / 32];
  __shared__ uint32_t er_done[kMaxErBuf / 32];

  const int part = blockIdx.x;
  const int64_t row0 = int64_t(part) * P.vec;
  const int lane = threadIdx.x & 31;
  const int wid = threadIdx.x >> 5;
  const int64_t n_chunks = (P.vec + 31) >> 5;
  T* xs = reinterpret_cast<T*>(smem_raw);
  const T* xwin = P.x + row0;
  const int64_t s0 = __ldg(P.er_part_ptr + part);
  const int64_t s1 = __ldg(P.er_part_ptr + part + 1);

  if (threadIdx.x == 0) {
    next_chunk = 0;
    next_er = (P.er_mix && P.do_er && P.do_ell)
                  ? int(min(int64_t(P.er_buf_slices),
                            int64_t(__ldg(P.er_part_ptr + part + 1) - __ldg(P.er_part_ptr + part))))
                  : 0;
    next_comb = 0;
    ell_finished = 0;
    if (P.timing) P.timing[4 * part] = globaltimer();
    if (part == 0 && P.pool_ctr) P.pool_ctr[(P.epoch + 1u) & 1u] = 0u;  // next launch's counter
  }
  for (int i = threadIdx.x; i < int((n_chunks + 31) >> 5); i += blockDim.x)
    chunk_done[i] = P.do_ell ? 0u : 0xffffffffu;
  for (int i = threadIdx.x; i < kMaxErBuf / 32; i += blockDim.x) er_done[i] = 0u;
  if constexpr (SMEM) {
    if (P.window_tma) {
      if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
      }
    }
  }
  __syncthreads();

  if (threadIdx.x == 0) {
    if constexpr (SMEM) {
      if (P.window_tma) {
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
      else mbar_wait(&bar, 0);
    } else {
      for (int64_t i = threadIdx.x; i < P.vec; i += blockDim.x) xs[i] = xwin[i];
      __syncthreads();
    }
  }
  const T* win = SMEM ? xs : xwin;
  if (P.timing && threadIdx.x == 0 && !win_pending) P.timing[4 * part + 1] = globaltimer();

  // own ER slices [s0, s1): the first n_buf are computed into a shared-memory
  // buffer at any time (ER-first warps overlap them with the ELL stream) and
  // combined with y_ell at the end; the rest finish directly against y_ell
  const int64_t n_own = s1 - s0;
  const int64_t n_buf = (P.do_er && P.do_ell) ? (n_own < P.er_buf_slices ? n_own : P.er_buf_slices) : 0;
  T* er_buf = reinterpret_cast<T*>(smem_raw + P.er_buf_offset);

  auto claim = [&](int* ctr) -> int64_t {
    int v = 0;
    if (lane == 0) v = atomicAdd(ctr, 1);
    return __shfl_sync(0xffffffffu, v, 0);
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
    int w;
    int64_t pos;
  };
  auto ell_meta = [&](int64_t chunk) -> EllMeta {
    EllMeta m{0, 0};
    if (chunk < n_chunks) {
      if constexpr (C32) {
        const int64_t s = (row0 >> 5) + chunk;
        m.w = __ldg(P.width_ell + s);
        m.pos = int64_t(__ldg(P.pos_ell + s));
        if (lane == 0 && P.pf_ell > 0 && m.w > 0)  // precise L2 prefetch of the claimed chunk
          prefetch_slice(P.val_ell, P.col_ell, m.pos, m.pos + 32 * int64_t(m.w));
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
    __threadfence_block();
    __syncwarp();
    if (lane == 0) {
      atomicOr(&chunk_done[unpublished >> 5], 1u << (unpublished & 31));
      // the warp publishing the partition's last chunk publishes the whole
      // ELL phase to other CTAs (pooled ER rows): one gpu-scope fence per
      // CTA instead of one per chunk
      if (P.part_flag && atomicAdd(&ell_finished, 1) == int(n_chunks) - 1) {
        __threadfence();
        st_release_gpu(P.part_flag + part, P.epoch);
      }
    }
    unpublished = -1;
  };
  auto run_chunk = [&](int64_t chunk, const EllMeta& m) {
    if constexpr (C32) {
      const T acc = ell_slice32<T, STRICT>(P.val_ell, P.col_ell, m.pos + lane, m.w, win,
                                           (SMEM && win_pending) ? &bar : nullptr);
      if (SMEM && win_pending) {
        win_pending = false;
        if (P.timing && threadIdx.x == 0) P.timing[4 * part + 1] = globaltimer();
      }
      publish();
      P.y[row0 + chunk * 32 + lane] = acc;
    } else {
      const int64_t lr = chunk * 32 + lane;
      T acc = T(0);
      if (lr < P.vec) {
        const int64_t r = row0 + lr;
        const int64_t C = P.warp;
        const int64_t s = r / C;
        const int w = __ldg(P.width_ell + s);
        const int64_t pos = int64_t(__ldg(P.pos_ell + s)) + (r - s * C);
        acc = ell_row_generic<T, STRICT>(P.val_ell, P.col_ell, pos, w, C, win);
      }
      publish();
      if (lr < P.vec) P.y[row0 + lr] = acc;
    }
    unpublished = chunk;
  };
  auto er_meta = [&](int64_t s, int64_t s_end) -> ErMeta {
    ErMeta m{-1, 0, 0, 0};
    if (s < s_end) {
      m = er_slice_meta(P, s, lane);
      if (lane == 0 && P.pf_er && m.sw > 0) {  // precise L2 prefetch of the claimed slice
        bulk_prefetch_l2(P.er_val + m.pos - lane, uint32_t(32 * int64_t(m.sw) * int64_t(sizeof(T))));
        bulk_prefetch_l2(P.er_col + m.pos - lane, uint32_t(32 * int64_t(m.sw) * 4));
      }
    }
    return m;
  };
  auto finish_own_er = [&](int64_t idx, const ErMeta& m) {
    const T acc = er_slice_compute<T, STRICT>(P, m);
    if (idx < n_buf) {
      er_buf[idx * 32 + lane] = acc;
      __threadfence_block();
      __syncwarp();
      if (lane == 0) atomicOr(&er_done[idx >> 5], 1u << (idx & 31));
    } else if (m.rw >= 0) {
      const int64_t r = m.rw & kRowMask;
      if (P.do_ell) wait_chunk(r);
      P.y[r] = add_rn(__ldcg(P.y + r), acc);
    }
  };

  int64_t pending = -1;
  const bool mix = P.er_mix && n_buf > 0;
  if (mix) {
    // one shared item sequence: the n_buf buffered own ER slices spread evenly
    // among the n_chunks ELL chunks, so their gather latency hides behind the
    // ELL stream of the other warps; item t is ER slice floor(t*n_buf/total)
    // when that floor steps at t, else ELL chunk t - floor(t*n_buf/total)
    const int64_t total = n_chunks + n_buf;
    for (int64_t t = claim(&next_chunk); t < total; t = claim(&next_chunk)) {
      const int64_t e0 = (t * n_buf) / total;
      if (((t + 1) * n_buf) / total > e0) {
        finish_own_er(e0, er_meta(s0 + e0, s1));
        publish();
      } else {
        run_chunk(t - e0, ell_meta(t - e0));
      }
      if (P.timing && lane == 0 && t + 1 == total) P.timing[4 * part + 2] = globaltimer();
    }
    publish();
  } else if (n_buf > 0 && wid < P.er_warps) {  // ER-first warps
    for (;;) {
      const int64_t idx = claim(&next_er);
      if (idx >= n_buf) {
        pending = idx;
        break;
      }
      finish_own_er(idx, er_meta(s0 + idx, s1));
    }
  }
  if (P.do_ell && !mix) {
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
    if (P.timing && lane == 0 && chunk == n_chunks) P.timing[4 * part + 2] = globaltimer();
  }

  if (P.do_er) {
    if (pending >= 0 && pending < n_own) finish_own_er(pending, er_meta(s0 + pending, s1));
    if (P.er_ahead) {
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
    // combine the buffered own ER rows: y[r] = y_ell[r] + er_acc
    for (int64_t idx = claim(&next_comb); idx < n_buf; idx = claim(&next_comb)) {
      while (!lds_volatile(&er_done[idx >> 5], 1u << (idx & 31))) {
      }
      __threadfence_block();
      const int32_t rw = __ldg(P.er_rows + (s0 + idx) * 32 + lane);
      if (rw >= 0) {
        const int64_t r = rw & kRowMask;
        wait_chunk(r);
        P.y[r] = add_rn(__ldcg(P.y + r), er_buf[idx * 32 + lane]);
      }
    }
    // shared pool: excess ER slices of heavy partitions, claimed by any CTA;
    // rows of other CTAs are finished once their ELL chunk is published
    if (P.pool_hi > P.pool_lo) {
      unsigned int* ctr = P.pool_ctr + (P.epoch & 1u);
      auto pclaim = [&]() -> int64_t {
        unsigned int v = 0;
        if (lane == 0) v = atomicAdd(ctr, 1u);
        return P.pool_lo + int64_t(__shfl_sync(0xffffffffu, v, 0));
      };
      int64_t s = pclaim();
      ErMeta m = er_meta(s, P.pool_hi);
      while (s < P.pool_hi) {
        const int64_t nxt = pclaim();
        const ErMeta mn = er_meta(nxt, P.pool_hi);
        const T acc = er_slice_compute<T, STRICT>(P, m);
        if (m.rw >= 0) {
          const int64_t r = m.rw & kRowMask;
          if (P.do_ell) {  // the owning CTA's ELL phase must be published
            const uint32_t rp = uint32_t(r) / uint32_t(P.vec);
            while (ld_acquire_gpu(P.part_flag + rp) != P.epoch) __nanosleep(64);
          }
          P.y[r] = add_rn(__ldcg(P.y + r), acc);
        }
        s = nxt;
        m = mn;
      }
    }
  }
  if (P.timing) {
    __syncthreads();
    if (threadIdx.x == 0) P.timing[4 * part + 3] = globaltimer();
  }
}

// ---------------------------------------------------------- vector kernels
template <typename T>
__global__ void permute_kernel(const T* __restrict__ x_user, const int32_t* __restrict__ inverse,
                               int64_t n, int64_t padded, T* __restrict__ x_r) {
  for (int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; j < padded;
       j += int64_t(gridDim.x) * blockDim.x) {
    const int64_t src = __ldg(inverse + j);
    x_r[j] = src < n ? __ldg(x_user + src) : T(0);
  }
}

template <typename T>
__global__ void unpermute_kernel(const T* __restrict__ y_r, const int32_t* __restrict__ reorder,
                                 int64_t n, T* __restrict__ y_user) {
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
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    p[i] = r[i] + beta * p[i];
}

template <typename T>
__global__ void axpy_kernel(const double* __restrict__ a, double sign, const T* __restrict__ x,
                            T* __restrict__ y, int64_t n) {
  const T alpha = T(sign * a[0]);
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    y[i] = y[i] + alpha * x[i];
}

}  // namespace ehyb
