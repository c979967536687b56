// Dev probe: the HBM rate a SELL-slice stream reaches on this B200 as a
// function of slice width W, loads in flight per lane (U), CTA size and the
// load form — the ELL stream of the fused kernel without its gathers, ER or
// metadata. Each CTA owns a contiguous run of 32-row slices (one partition),
// warps claim slices from a shared counter, lane = row, slots pos + 32 k.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        scripts/stream_probe.cu -o scripts/tmp/stream_probe
//   scripts/tmp/stream_probe > profiles/stream_probe_<tag>.txt
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e_ = (x);                                                       \
    if (e_ != cudaSuccess) {                                                    \
      std::fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
      std::exit(1);                                                             \
    }                                                                           \
  } while (0)

// MODE 0: scalar SELL loads, batches of U slots (cols then values)
// MODE 1: two slices per claim, their batches interleaved (2U loads in flight)
template <typename T, int U, int MODE>
__global__ void __launch_bounds__(1024, 1)
probe(const T* __restrict__ val, const uint16_t* __restrict__ col, int64_t slices_per_cta, int w,
      T* __restrict__ y) {
  __shared__ int ctr;
  if (threadIdx.x == 0) ctr = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t s0 = int64_t(blockIdx.x) * slices_per_cta;
  const int step = MODE == 1 ? 2 : 1;
  for (;;) {
    int c = 0;
    if (lane == 0) c = atomicAdd(&ctr, step);
    c = __shfl_sync(0xffffffffu, c, 0);
    if (c >= slices_per_cta) break;
    if (MODE == 0) {
      const int64_t pos = (s0 + c) * 32 * int64_t(w) + lane;
      T acc = T(0);
      for (int k = 0; k < w; k += U) {
        uint32_t cc[U];
        T v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) cc[u] = (k + u < w) ? __ldcs(col + pos + 32 * int64_t(k + u)) : 0u;
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = (k + u < w) ? __ldcs(val + pos + 32 * int64_t(k + u)) : T(0);
#pragma unroll
        for (int u = 0; u < U; ++u) acc += v[u] * T(cc[u]);
      }
      y[(s0 + c) * 32 + lane] = acc;
    } else {
      const bool two = c + 1 < slices_per_cta;
      const int64_t pa = (s0 + c) * 32 * int64_t(w) + lane;
      const int64_t pb = pa + 32 * int64_t(w);
      T a = T(0), b = T(0);
      for (int k = 0; k < w; k += U) {
        uint32_t ca[U], cb[U];
        T va[U], vb[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          ca[u] = (k + u < w) ? __ldcs(col + pa + 32 * int64_t(k + u)) : 0u;
          cb[u] = (two && k + u < w) ? __ldcs(col + pb + 32 * int64_t(k + u)) : 0u;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          va[u] = (k + u < w) ? __ldcs(val + pa + 32 * int64_t(k + u)) : T(0);
          vb[u] = (two && k + u < w) ? __ldcs(val + pb + 32 * int64_t(k + u)) : T(0);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          a += va[u] * T(ca[u]);
          b += vb[u] * T(cb[u]);
        }
      }
      y[(s0 + c) * 32 + lane] = a;
      if (two) y[(s0 + c + 1) * 32 + lane] = b;
    }
  }
}

// MODE 2: the 128-bit interleaved layout: per block of 4 k, each lane loads
// its 4 values (float4 / 2 x double2) and 4 columns (uint2) contiguously;
// UB blocks per batch (w is a multiple of 4 here)
template <typename T>
__device__ __forceinline__ void ld4(const T* p, T* v);
template <>
__device__ __forceinline__ void ld4<float>(const float* p, float* v) {
  const float4 q = __ldcs(reinterpret_cast<const float4*>(p));
  v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
}
template <>
__device__ __forceinline__ void ld4<double>(const double* p, double* v) {
  const double2 q0 = __ldcs(reinterpret_cast<const double2*>(p));
  const double2 q1 = __ldcs(reinterpret_cast<const double2*>(p) + 1);
  v[0] = q0.x; v[1] = q0.y; v[2] = q1.x; v[3] = q1.y;
}
template <typename T, int UB>
__global__ void __launch_bounds__(1024, 1)
probe_vec(const T* __restrict__ val, const uint16_t* __restrict__ col, int64_t slices_per_cta,
          int w, T* __restrict__ y) {
  __shared__ int ctr;
  if (threadIdx.x == 0) ctr = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t s0 = int64_t(blockIdx.x) * slices_per_cta;
  const int nb = w / 4;
  for (;;) {
    int c = 0;
    if (lane == 0) c = atomicAdd(&ctr, 1);
    c = __shfl_sync(0xffffffffu, c, 0);
    if (c >= slices_per_cta) break;
    const int64_t pos = (s0 + c) * 32 * int64_t(w) + 4 * lane;
    T acc = T(0);
    for (int b = 0; b < nb; b += UB) {
      uint2 cc[UB];
      T v[4 * UB];
#pragma unroll
      for (int u = 0; u < UB; ++u)
        cc[u] = (b + u < nb) ? __ldcs(reinterpret_cast<const uint2*>(col + pos + 128 * int64_t(b + u)))
                             : make_uint2(0u, 0u);
#pragma unroll
      for (int u = 0; u < UB; ++u) {
        if (b + u < nb) ld4<T>(val + pos + 128 * int64_t(b + u), v + 4 * u);
        else for (int j = 0; j < 4; ++j) v[4 * u + j] = T(0);
      }
#pragma unroll
      for (int u = 0; u < UB; ++u)
        acc += v[4 * u] * T(cc[u].x & 0xffff) + v[4 * u + 1] * T(cc[u].x >> 16) +
               v[4 * u + 2] * T(cc[u].y & 0xffff) + v[4 * u + 3] * T(cc[u].y >> 16);
    }
    y[(s0 + c) * 32 + lane] = acc;
  }
}

// MODE 3: the real ELL chunk loop piece by piece (FEAT bits): 1 = x gathers
// from a shared-memory window through the stored columns, 2 = per-slice
// metadata (width, position) loaded from global memory after the claim,
// 4 = chunk publication (block fence + shared atomics), 8 = metadata claimed
// one slice ahead. Vec layout, UB blocks per batch.
template <typename T, int UB, int FEAT>
__global__ void __launch_bounds__(1024, 1)
probe_real(const T* __restrict__ val, const uint16_t* __restrict__ col, int64_t slices_per_cta,
           int w, T* __restrict__ y, const int32_t* __restrict__ wid_g,
           const int32_t* __restrict__ pos_g, int win_elems) {
  extern __shared__ __align__(16) unsigned char smem[];
  T* win = reinterpret_cast<T*>(smem);
  __shared__ int ctr;
  __shared__ uint32_t done[64];
  __shared__ int fin;
  for (int i = threadIdx.x; i < win_elems; i += blockDim.x) win[i] = T(i & 7);
  if (threadIdx.x == 0) { ctr = 0; fin = 0; }
  if (threadIdx.x < 64) done[threadIdx.x] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t s0 = int64_t(blockIdx.x) * slices_per_cta;
  auto claim = [&]() {
    int c = 0;
    if (lane == 0) c = atomicAdd(&ctr, 1);
    return __shfl_sync(0xffffffffu, c, 0);
  };
  auto meta = [&](int c, int& ww, int64_t& pp) {
    if (FEAT & 2) {
      if (c < slices_per_cta) { ww = __ldg(wid_g + s0 + c); pp = __ldg(pos_g + s0 + c); }
    } else {
      ww = w;
      pp = (s0 + c) * 32 * int64_t(w);
    }
  };
  int c = claim();
  int ww = 0;
  int64_t pp = 0;
  int prev = -1;
  meta(c, ww, pp);
  while (c < slices_per_cta) {
    int cn = 0, wn = 0;
    int64_t pn = 0;
    if (FEAT & 8) { cn = claim(); meta(cn, wn, pn); }
    const int nb = ww / 4;
    const int64_t pos = ((FEAT & 2) ? int64_t(pp) : pp) + 4 * lane;
    T acc = T(0);
    for (int b = 0; b < nb; b += UB) {
      uint2 cc[UB];
      T v[4 * UB];
#pragma unroll
      for (int u = 0; u < UB; ++u)
        cc[u] = (b + u < nb) ? __ldcs(reinterpret_cast<const uint2*>(col + pos + 128 * int64_t(b + u)))
                             : make_uint2(0u, 0u);
#pragma unroll
      for (int u = 0; u < UB; ++u) {
        if (b + u < nb) ld4<T>(val + pos + 128 * int64_t(b + u), v + 4 * u);
        else for (int j = 0; j < 4; ++j) v[4 * u + j] = T(0);
      }
      if (FEAT & 1) {
#pragma unroll
        for (int u = 0; u < UB; ++u)
          acc += v[4 * u] * win[cc[u].x & 0xffff] + v[4 * u + 1] * win[cc[u].x >> 16] +
                 v[4 * u + 2] * win[cc[u].y & 0xffff] + v[4 * u + 3] * win[cc[u].y >> 16];
      } else {
#pragma unroll
        for (int u = 0; u < UB; ++u)
          acc += v[4 * u] * T(cc[u].x & 0xffff) + v[4 * u + 1] * T(cc[u].x >> 16) +
                 v[4 * u + 2] * T(cc[u].y & 0xffff) + v[4 * u + 3] * T(cc[u].y >> 16);
      }
    }
    // 4: publish (16: the previous chunk, after this one's compute; 32: no
    // fence; 64: no atomics; 128: one release reduction instead of fence + atomics)
    const int pc = (FEAT & 16) ? prev : c;
    if ((FEAT & 4) && pc >= 0) {
      if (FEAT & 128) {
        __syncwarp();
        if (lane == 0) {
          const uint32_t addr = static_cast<uint32_t>(__cvta_generic_to_shared(&done[(pc >> 5) & 63]));
          asm volatile("red.release.cta.shared::cta.or.b32 [%0], %1;" ::"r"(addr), "r"(1u << (pc & 31)) : "memory");
        }
      } else {
        if (!(FEAT & 32)) __threadfence_block();
        __syncwarp();
        if (lane == 0 && !(FEAT & 64)) { atomicOr(&done[(pc >> 5) & 63], 1u << (pc & 31)); atomicAdd(&fin, 1); }
      }
    }
    y[(s0 + c) * 32 + lane] = acc;
    prev = c;
    if (FEAT & 8) { c = cn; ww = wn; pp = pn; }
    else { c = claim(); meta(c, ww, pp); }
  }
}

template <typename T, int UB, int FEAT>
void run_real(int w, int sms, size_t budget_bytes, int win_bytes) {
  const int64_t slot_bytes = sizeof(T) + 2;
  int64_t slices = int64_t(budget_bytes / (32 * w * slot_bytes));
  const int64_t per_cta = slices / sms;
  slices = per_cta * sms;
  const int64_t slots = slices * 32 * w;
  const int win_elems = win_bytes / int(sizeof(T));
  T* val;
  uint16_t* col;
  T* y;
  int32_t *wid, *pos;
  CK(cudaMalloc(&val, slots * sizeof(T)));
  CK(cudaMalloc(&col, slots * 2));
  CK(cudaMalloc(&y, slices * 32 * sizeof(T)));
  CK(cudaMalloc(&wid, slices * 4));
  CK(cudaMalloc(&pos, slices * 4));
  CK(cudaMemset(val, 0, slots * sizeof(T)));
  std::vector<uint16_t> hc(static_cast<size_t>(slots));
  uint32_t st = 12345u;
  for (auto& x : hc) { st = st * 1664525u + 1013904223u; x = uint16_t((st >> 8) % uint32_t(win_elems)); }
  CK(cudaMemcpy(col, hc.data(), slots * 2, cudaMemcpyHostToDevice));
  std::vector<int32_t> hw(static_cast<size_t>(slices), w), hp(static_cast<size_t>(slices));
  for (int64_t i = 0; i < slices; ++i) hp[size_t(i)] = int32_t(i * 32 * w);
  CK(cudaMemcpy(wid, hw.data(), slices * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(pos, hp.data(), slices * 4, cudaMemcpyHostToDevice));
  CK(cudaFuncSetAttribute(probe_real<T, UB, FEAT>, cudaFuncAttributeMaxDynamicSharedMemorySize, win_bytes));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  auto launch = [&]() {
    probe_real<T, UB, FEAT><<<sms, 1024, win_bytes>>>(val, col, per_cta, w, y, wid, pos, win_elems);
  };
  for (int i = 0; i < 3; ++i) launch();
  CK(cudaDeviceSynchronize());
  const int reps = 20;
  CK(cudaEventRecord(a));
  for (int i = 0; i < reps; ++i) launch();
  CK(cudaEventRecord(b));
  CK(cudaEventSynchronize(b));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, a, b));
  const double t = ms / 1e3 / reps;
  const double bytes = double(slots) * slot_bytes + double(slices) * 32 * sizeof(T);
  std::printf("real feat=%2d tau=%zu w=%2d UB=%d win=%6d  %.1f us  %.0f GB/s\n", FEAT, sizeof(T), w,
              UB, win_bytes, t * 1e6, bytes / t / 1e9);
  std::fflush(stdout);
  CK(cudaFree(val));
  CK(cudaFree(col));
  CK(cudaFree(y));
  CK(cudaFree(wid));
  CK(cudaFree(pos));
}

template <typename T, int U, int MODE>
void run(const char* name, int w, int threads, int sms, size_t budget_bytes) {
  const int64_t slot_bytes = sizeof(T) + 2;
  int64_t slices = int64_t(budget_bytes / (32 * w * slot_bytes));
  const int64_t per_cta = slices / sms;
  slices = per_cta * sms;
  const int64_t slots = slices * 32 * w;
  T* val;
  uint16_t* col;
  T* y;
  CK(cudaMalloc(&val, slots * sizeof(T)));
  CK(cudaMalloc(&col, slots * 2));
  CK(cudaMalloc(&y, slices * 32 * sizeof(T)));
  CK(cudaMemset(val, 0, slots * sizeof(T)));
  CK(cudaMemset(col, 0, slots * 2));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  auto launch = [&]() {
    if constexpr (MODE == 2) probe_vec<T, U><<<sms, threads>>>(val, col, per_cta, w, y);
    else probe<T, U, MODE><<<sms, threads>>>(val, col, per_cta, w, y);
  };
  for (int i = 0; i < 3; ++i) launch();
  CK(cudaDeviceSynchronize());
  const int reps = 20;
  CK(cudaEventRecord(a));
  for (int i = 0; i < reps; ++i) launch();
  CK(cudaEventRecord(b));
  CK(cudaEventSynchronize(b));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, a, b));
  const double t = ms / 1e3 / reps;
  const double bytes = double(slots) * slot_bytes + double(slices) * 32 * sizeof(T);
  std::printf("%-10s tau=%zu w=%2d U=%2d threads=%4d  %.1f us  %.0f GB/s\n", name, sizeof(T), w, U,
              threads, t * 1e6, bytes / t / 1e9);
  std::fflush(stdout);
  CK(cudaFree(val));
  CK(cudaFree(col));
  CK(cudaFree(y));
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const size_t budget = size_t(480) << 20;  // ~ the cfg2 / cfg3 ELL slab
  // fp32, w = 16, window 132 KB (cfg3 fp32); fp64, w = 28, window 113 KB (cfg2)
  run_real<float, 4, 3>(16, sms, budget, 135168);
  run_real<float, 4, 7>(16, sms, budget, 135168);
  run_real<float, 4, 7 + 16>(16, sms, budget, 135168);
  run_real<float, 4, 7 + 32>(16, sms, budget, 135168);
  run_real<float, 4, 7 + 64>(16, sms, budget, 135168);
  run_real<float, 4, 7 + 128>(16, sms, budget, 135168);
  run_real<float, 4, 7 + 16 + 128>(16, sms, budget, 135168);
  run_real<float, 4, 15 + 16>(16, sms, budget, 135168);
  run_real<float, 4, 15 + 16 + 128>(16, sms, budget, 135168);
  run_real<double, 2, 3>(28, sms, budget, 113408);
  run_real<double, 2, 15 + 16>(28, sms, budget, 113408);
  run_real<double, 2, 15 + 16 + 128>(28, sms, budget, 113408);
  return 0;
}
