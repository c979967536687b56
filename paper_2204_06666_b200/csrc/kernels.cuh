// EHYB SpMV kernels for B200 (sm_100a).
//
// One CTA per partition (Alg.3; reference simulation
// engine.py:134-154):
//   1. the partition's x window x[p*vec, (p+1)*vec) is staged into shared
//      memory by TMA bulk copies (cp.async.bulk ... mbarrier::complete_tx);
//   2. warps claim 32-row chunks (= SELL slices for warp_size 32) from a
//      shared-memory counter (the paper's in-block slice stealing) and stream
//      val/col with coalesced, evict-first loads, U slots in flight per lane,
//      gathering x from the staged window through the u16 local columns;
//   3. after a CTA barrier the same CTA runs the partition's ER rows (derived
//      per-partition SELL layout, x through the read-only path) and finishes
//      y[r] = y_ell[r] + er_acc — the reference's phase-2 "y[y_idx] += acc"
//      without a grid-wide barrier or atomics (each ER row belongs to exactly
//      one partition, so only its own CTA touches it).
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

// One SELL row: lane slots pos, pos+C, ..., pos+(w-1)C; x gathered from `win`
// (shared-memory window or global). U independent loads per lane in flight.
template <typename T, bool STRICT>
__device__ __forceinline__ T ell_row(const T* __restrict__ val, const uint16_t* __restrict__ col,
                                     int64_t pos, int w, int64_t C, const T* win) {
  T acc = T(0);
  for (int k = 0; k < w; k += kUnroll) {
    T v[kUnroll];
    uint32_t c[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
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

template <typename T, bool STRICT, bool C32>
__global__ void __launch_bounds__(1024, 1) spmv_fused_kernel(const SpmvParams<T> P) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ uint64_t bar;
  __shared__ int next_chunk;
  __shared__ int next_er;

  const int part = blockIdx.x;
  const int64_t row0 = int64_t(part) * P.vec;
  const int lane = threadIdx.x & 31;
  const int wid = threadIdx.x >> 5;
  const int nwarps = blockDim.x >> 5;
  T* xs = reinterpret_cast<T*>(smem_raw);
  const T* xwin = P.x + row0;

  if (threadIdx.x == 0) {
    next_chunk = nwarps;
    next_er = nwarps;
  }
  if (P.do_ell && P.window_in_smem && P.window_tma) {
    if (threadIdx.x == 0) {
      mbar_init(&bar, 1);
      fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      const uint32_t bytes = uint32_t(P.vec * int64_t(sizeof(T)));
      mbar_expect_tx(&bar, bytes);
      for (uint32_t off = 0; off < bytes; off += kTmaChunk) {
        const uint32_t len = bytes - off < uint32_t(kTmaChunk) ? bytes - off : uint32_t(kTmaChunk);
        tma_bulk_g2s(smem_raw + off, reinterpret_cast<const unsigned char*>(xwin) + off, len, &bar);
      }
    }
    mbar_wait(&bar, 0);
  } else if (P.do_ell && P.window_in_smem) {
    for (int64_t i = threadIdx.x; i < P.vec; i += blockDim.x) xs[i] = xwin[i];
    __syncthreads();
  } else {
    __syncthreads();
  }
  const T* win = P.window_in_smem ? xs : xwin;

  if (P.do_ell) {
    const int64_t n_chunks = (P.vec + 31) >> 5;
    int64_t chunk = wid;
    while (chunk < n_chunks) {
      if constexpr (C32) {
        // warp == one SELL slice: warp-uniform width, 256 B (fp64) coalesced rows
        const int64_t s = (row0 >> 5) + chunk;
        const int w = __ldg(P.width_ell + s);
        const int64_t pos = int64_t(__ldg(P.pos_ell + s)) + lane;
        const T acc = ell_row<T, STRICT>(P.val_ell, P.col_ell, pos, w, 32, win);
        P.y[row0 + chunk * 32 + lane] = acc;
      } else {
        const int64_t lr = chunk * 32 + lane;
        if (lr < P.vec) {
          const int64_t r = row0 + lr;
          const int64_t C = P.warp;
          const int64_t s = r / C;
          const int w = __ldg(P.width_ell + s);
          const int64_t pos = int64_t(__ldg(P.pos_ell + s)) + (r - s * C);
          P.y[r] = ell_row<T, STRICT>(P.val_ell, P.col_ell, pos, w, C, win);
        }
      }
      int nxt = 0;
      if (lane == 0) nxt = atomicAdd(&next_chunk, 1);
      chunk = __shfl_sync(0xffffffffu, nxt, 0);
    }
  }

  if (P.do_er) {
    if (P.do_ell) __syncthreads();  // this CTA's y_ell writes precede the ER combine
    const int64_t s0 = __ldg(P.er_part_ptr + part);
    const int64_t s1 = __ldg(P.er_part_ptr + part + 1);
    int64_t s = s0 + wid;
    while (s < s1) {
      const int32_t rw = __ldg(P.er_rows + s * 32 + lane);
      const int lw = __ldg(P.er_lwidth + s * 32 + lane);
      const int sw = __ldg(P.er_swidth + s);
      const int64_t pos = __ldg(P.er_pos + s) + lane;
      T acc = T(0);
      for (int k = 0; k < sw; k += kUnroll) {
        T v[kUnroll];
        uint32_t c[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
          if (k + u < lw) {
            v[u] = __ldcs(P.er_val + pos + int64_t(k + u) * 32);
            c[u] = __ldcs(P.er_col + pos + int64_t(k + u) * 32);
          }
        }
#pragma unroll
        for (int u = 0; u < kUnroll; ++u)
          if (k + u < lw) acc = madd<STRICT>(acc, v[u], __ldg(P.x + c[u]));
      }
      if (rw >= 0) {
        // reference ER padding products 0*x[0] (engine.py:148-151): inert for
        // finite x, NaN-propagating otherwise — reproduced with one product
        if (rw & kPadFlag) acc = add_rn(acc, mul_rn(T(0), __ldg(P.x)));
        const int64_t r = rw & kRowMask;
        P.y[r] = add_rn(P.y[r], acc);
      }
      int nxt = 0;
      if (lane == 0) nxt = atomicAdd(&next_er, 1);
      s = s0 + __shfl_sync(0xffffffffu, nxt, 0);
    }
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

template <typename T>
__global__ void axpy_kernel(const double* __restrict__ a, double sign, const T* __restrict__ x,
                            T* __restrict__ y, int64_t n) {
  const T alpha = T(sign * a[0]);
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    y[i] = y[i] + alpha * x[i];
}

}  // namespace ehyb
