// GPU preprocessing: build_graph (partition.py:77-98) and classify_rows +
// build_reorder_plan + assemble_ehyb (format.py:123-409) on the B200, bit-exact
// with the host C++ path in prep.cpp (and so with the reference). The BFS
// partitioner between the two (partition.py:101-204) is sequential by the
// reference's semantics and stays on the host.
//
// Pipeline (one context per matrix, the COO uploaded once):
//   ehyb_gprep_create     COO -> device, entries grouped by (row, column,
//                         entry index) with a stable radix sort = the order of
//                         np.lexsort((cols, rows)) the reference assembles in
//   ehyb_gprep_build_graph symmetrised off-diagonal keys u<<32|v, radix sort,
//                         unique -> adjacency CSR (np.unique order)
//   ehyb_gprep_assemble   inner/outer counts, row_order = lexsort((rows,
//                         -inner, part)) and er_row_order (stable radix sorts),
//                         the reorder plan, slice widths / int32 positions,
//                         ELL / ER placement — results copied back into the
//                         caller's (numpy) arrays
#include <cuda_runtime.h>
#include <cub/cub.cuh>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <climits>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "ehyb_common.h"

namespace {

using ehyb::fail;

#define GP_TRY(expr)                                                                   \
  do {                                                                                 \
    cudaError_t e_ = (expr);                                                           \
    if (e_ != cudaSuccess)                                                             \
      return fail(std::string("CUDA error in GPU preprocessing: ") + cudaGetErrorString(e_), \
                  EHYB_ECUDA);                                                         \
  } while (0)

constexpr int kT = 256;

inline int blocks_for(int64_t n) {
  return int(std::max<int64_t>(1, std::min<int64_t>((n + kT - 1) / kT, int64_t(1) << 20)));
}

int bits_for(uint64_t v) {  // bits needed to represent v (>= 1)
  int b = 1;
  while (b < 64 && (uint64_t(1) << b) <= v) ++b;
  return b;
}

// EHYB_GPREP_TIMING=1: per-stage wall times on stderr (dev measurement)
struct StageTimer {
  bool on = std::getenv("EHYB_GPREP_TIMING") != nullptr;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void mark(const char* what) {
    if (!on) return;
    cudaDeviceSynchronize();
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "gprep %-28s %8.2f ms\n", what,
                 std::chrono::duration<double, std::milli>(now - t).count());
    t = now;
  }
};

struct DevBuf {
  void* p = nullptr;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  template <typename T>
  T* as() const { return static_cast<T*>(p); }
  cudaError_t alloc(size_t bytes) {
    if (p) cudaFree(p);
    p = nullptr;
    return cudaMalloc(&p, std::max<size_t>(bytes, 16));
  }
};

// Host <-> device copies of pageable (numpy / malloc) memory through a
// double-buffered pinned staging area: the host side of every chunk is
// copied by all OpenMP threads (which also spreads the first-touch page
// faults of fresh output arrays), overlapped with the DMA of the other half.
// the pinned area is process-wide (page-locking 64 MB costs 100+ ms); one
// preprocessing context uses it at a time
std::mutex g_pinned_mu;
unsigned char* g_pinned = nullptr;

struct Staging {
  static constexpr size_t kHalf = size_t(32) << 20;
  unsigned char* buf = nullptr;
  cudaStream_t st = nullptr;
  cudaEvent_t ev[2] = {nullptr, nullptr};
  std::unique_lock<std::mutex> hold;
  ~Staging() {
    for (auto e : ev)
      if (e) cudaEventDestroy(e);
    if (st) cudaStreamDestroy(st);
  }
  cudaError_t init() {
    if (buf) return cudaSuccess;
    hold = std::unique_lock<std::mutex>(g_pinned_mu);
    cudaError_t e = cudaSuccess;
    if (!g_pinned) e = cudaMallocHost(reinterpret_cast<void**>(&g_pinned), 2 * kHalf);
    buf = g_pinned;
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    for (int i = 0; i < 2 && e == cudaSuccess; ++i) e = cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming);
    return e;
  }
  static void par_copy(void* dst, const void* src, size_t bytes) {
    const int64_t nb = int64_t((bytes + (1 << 20) - 1) >> 20);
#pragma omp parallel for schedule(static) if (nb > 1)
    for (int64_t b = 0; b < nb; ++b) {
      const size_t off = size_t(b) << 20;
      std::memcpy(static_cast<unsigned char*>(dst) + off, static_cast<const unsigned char*>(src) + off,
                  std::min<size_t>(size_t(1) << 20, bytes - off));
    }
  }
  cudaError_t h2d(void* dev, const void* host, size_t bytes) {
    if (bytes <= kHalf) return cudaMemcpy(dev, host, bytes, cudaMemcpyHostToDevice);
    cudaError_t e = init();
    if (e == cudaSuccess) e = cudaDeviceSynchronize();  // earlier default-stream work is done
    for (size_t off = 0, i = 0; e == cudaSuccess && off < bytes; off += kHalf, ++i) {
      const size_t len = std::min(kHalf, bytes - off);
      unsigned char* half = buf + (i & 1) * kHalf;
      if (i >= 2) e = cudaEventSynchronize(ev[i & 1]);  // the DMA out of this half is done
      if (e != cudaSuccess) break;
      par_copy(half, static_cast<const unsigned char*>(host) + off, len);
      e = cudaMemcpyAsync(static_cast<unsigned char*>(dev) + off, half, len, cudaMemcpyHostToDevice, st);
      if (e == cudaSuccess) e = cudaEventRecord(ev[i & 1], st);
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    return e;
  }
  cudaError_t d2h(void* host, const void* dev, size_t bytes) {
    if (bytes <= kHalf) return bytes ? cudaMemcpy(host, dev, bytes, cudaMemcpyDeviceToHost) : cudaSuccess;
    cudaError_t e = init();
    if (e != cudaSuccess || bytes == 0) return e;
    e = cudaDeviceSynchronize();  // results of the default-stream kernels
    const size_t n = (bytes + kHalf - 1) / kHalf;
    for (size_t i = 0; e == cudaSuccess && i < n; ++i) {
      const size_t off = i * kHalf, len = std::min(kHalf, bytes - off);
      if (i == 0) {
        e = cudaMemcpyAsync(buf, static_cast<const unsigned char*>(dev), len, cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaEventRecord(ev[0], st);
      }
      if (e == cudaSuccess && i + 1 < n) {  // next chunk into the other half
        const size_t o2 = off + kHalf, l2 = std::min(kHalf, bytes - o2);
        e = cudaMemcpyAsync(buf + ((i + 1) & 1) * kHalf, static_cast<const unsigned char*>(dev) + o2, l2,
                            cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaEventRecord(ev[(i + 1) & 1], st);
      }
      if (e == cudaSuccess) e = cudaEventSynchronize(ev[i & 1]);
      if (e == cudaSuccess) par_copy(static_cast<unsigned char*>(host) + off, buf + (i & 1) * kHalf, len);
      // the half just drained is reused two chunks later: the stream waits
      // for nothing else, the host copy above finished before the next issue
    }
    return e;
  }
};

// ------------------------------------------------------------------ kernels
__global__ void k_pack_rc(const int64_t* __restrict__ rows, const int64_t* __restrict__ cols,
                          int64_t nnz, uint64_t* __restrict__ key) {
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < nnz;
       e += int64_t(gridDim.x) * blockDim.x)
    key[e] = (uint64_t(rows[e]) << 32) | uint64_t(uint32_t(cols[e]));
}

__global__ void k_row_count(const uint64_t* __restrict__ key, int64_t nnz, int64_t* __restrict__ cnt) {
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < nnz;
       e += int64_t(gridDim.x) * blockDim.x)
    atomicAdd(reinterpret_cast<unsigned long long*>(cnt + (key[e] >> 32)), 1ull);
}

__global__ void k_split_cols(const uint64_t* __restrict__ key, int64_t nnz, int32_t* __restrict__ col) {
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < nnz;
       e += int64_t(gridDim.x) * blockDim.x)
    col[e] = int32_t(uint32_t(key[e]));
}

// off-diagonal entries: flag, then both orientations of each
__global__ void k_offdiag_flag(const uint64_t* __restrict__ key, int64_t nnz, int64_t* __restrict__ flag) {
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < nnz;
       e += int64_t(gridDim.x) * blockDim.x)
    flag[e] = (key[e] >> 32) != (key[e] & 0xffffffffull) ? 1 : 0;
}

__global__ void k_sym_keys(const uint64_t* __restrict__ key, const int64_t* __restrict__ at, int64_t nnz,
                           int64_t m, uint64_t* __restrict__ out) {
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < nnz;
       e += int64_t(gridDim.x) * blockDim.x) {
    const uint64_t k = key[e];
    const uint64_t u = k >> 32, v = k & 0xffffffffull;
    if (u != v) {
      const int64_t d = at[e];
      out[d] = k;
      out[m + d] = (v << 32) | u;
    }
  }
}

__global__ void k_adj_out(const uint64_t* __restrict__ key, int64_t m, int32_t* __restrict__ adj,
                          int64_t* __restrict__ cnt) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < m;
       i += int64_t(gridDim.x) * blockDim.x) {
    adj[i] = int32_t(uint32_t(key[i]));
    atomicAdd(reinterpret_cast<unsigned long long*>(cnt + (key[i] >> 32)), 1ull);
  }
}

__global__ void k_i64_to_i32(const int64_t* __restrict__ a, int64_t n, int32_t* __restrict__ b) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    b[i] = int32_t(a[i]);
}

// inner / outer counts per row over its grouped entries
__global__ void k_classify(const int64_t* __restrict__ rptr, const int32_t* __restrict__ col,
                           const int32_t* __restrict__ part, int64_t n, int64_t* __restrict__ inner,
                           int64_t* __restrict__ outer) {
  for (int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; r < n;
       r += int64_t(gridDim.x) * blockDim.x) {
    const int32_t pr = part[r];
    int64_t ni = 0;
    const int64_t a = rptr[r], b = rptr[r + 1];
    for (int64_t j = a; j < b; ++j) ni += part[col[j]] == pr;
    inner[r] = ni;
    outer[r] = (b - a) - ni;
  }
}

// row_order key: (part, inner descending); rows enter in ascending order and
// the radix sort is stable, so ties keep the original row order
__global__ void k_order_keys(const int32_t* __restrict__ part, const int64_t* __restrict__ inner,
                             int64_t n, uint64_t* __restrict__ key, int64_t* __restrict__ val) {
  for (int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; r < n;
       r += int64_t(gridDim.x) * blockDim.x) {
    key[r] = (uint64_t(uint32_t(part[r])) << 32) | uint64_t(0xffffffffu - uint32_t(inner[r]));
    val[r] = r;
  }
}

__global__ void k_iota(int64_t* __restrict__ a, int64_t n) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    a[i] = i;
}

__global__ void k_er_keys(const int64_t* __restrict__ rows, const int64_t* __restrict__ outer,
                          int64_t m, uint32_t* __restrict__ key) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < m;
       i += int64_t(gridDim.x) * blockDim.x)
    key[i] = 0xffffffffu - uint32_t(outer[rows[i]]);
}

struct HasOuter {
  const int64_t* outer;
  __device__ bool operator()(const int64_t& r) const { return outer[r] > 0; }
};

__global__ void k_part_hist(const int32_t* __restrict__ part, int64_t n, int64_t* __restrict__ occ) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    atomicAdd(reinterpret_cast<unsigned long long*>(occ + part[i]), 1ull);
}

// reorder[row_order[i]] = p * vec + (i - start[p])
__global__ void k_reorder(const int64_t* __restrict__ row_order, const int32_t* __restrict__ part,
                          const int64_t* __restrict__ start, int64_t n, int64_t vec,
                          int64_t* __restrict__ reorder) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = row_order[i];
    const int64_t p = part[r];
    reorder[r] = p * vec + (i - start[p]);
  }
}

// padding rows n.. take the free ids of every part in ascending order:
// free id t of part p (t < vec - occ_p) goes to row n + free_start[p] + t
__global__ void k_pad_ids(const int64_t* __restrict__ occ, const int64_t* __restrict__ free_start,
                          int64_t n_parts, int64_t vec, int64_t n, int64_t* __restrict__ reorder) {
  const int64_t p = blockIdx.x;
  if (p >= n_parts) return;
  const int64_t o = occ[p];
  for (int64_t t = threadIdx.x; t < vec - o; t += blockDim.x)
    reorder[n + free_start[p] + t] = p * vec + o + t;
}

__global__ void k_inverse(const int64_t* __restrict__ reorder, int64_t padded, int64_t* __restrict__ inv) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < padded;
       i += int64_t(gridDim.x) * blockDim.x)
    inv[reorder[i]] = i;
}

__global__ void k_fill_i64(int64_t* __restrict__ a, int64_t n, int64_t v) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    a[i] = v;
}

__global__ void k_arrange(const int64_t* __restrict__ er_order, const int64_t* __restrict__ reorder,
                          int64_t n_er, int64_t* __restrict__ arrange, int64_t* __restrict__ y_idx) {
  for (int64_t s = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; s < n_er;
       s += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = er_order[s];
    arrange[r] = s;
    y_idx[s] = reorder[r];
  }
}

__global__ void k_row_widths(const int64_t* __restrict__ inner, const int64_t* __restrict__ outer,
                             const int64_t* __restrict__ reorder, const int64_t* __restrict__ arrange,
                             int64_t n, int32_t* __restrict__ ellw, int32_t* __restrict__ erw) {
  for (int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; r < n;
       r += int64_t(gridDim.x) * blockDim.x) {
    ellw[reorder[r]] = int32_t(inner[r]);
    if (arrange[r] >= 0) erw[arrange[r]] = int32_t(outer[r]);
  }
}

// slice width = max over its rows; slot count per slice = warp * width (int64)
__global__ void k_slice_width(const int32_t* __restrict__ rw, int64_t n_rows, int64_t warp,
                              int64_t n_sl, int32_t* __restrict__ width, int64_t* __restrict__ slots) {
  for (int64_t s = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; s < n_sl;
       s += int64_t(gridDim.x) * blockDim.x) {
    int32_t w = 0;
    const int64_t e = n_rows < (s + 1) * warp ? n_rows : (s + 1) * warp;
    for (int64_t l = s * warp; l < e; ++l) w = max(w, rw[l]);
    width[s] = w;
    slots[s] = warp * int64_t(w);
  }
}

__global__ void k_positions32(const int64_t* __restrict__ excl, int64_t n_sl, int64_t total,
                              int32_t* __restrict__ pos) {
  for (int64_t s = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; s <= n_sl;
       s += int64_t(gridDim.x) * blockDim.x)
    pos[s] = int32_t(s < n_sl ? excl[s] : total);
}

template <typename V>
__global__ void k_place(const int64_t* __restrict__ rptr, const int32_t* __restrict__ col,
                        const double* __restrict__ val, const int32_t* __restrict__ part,
                        const int64_t* __restrict__ reorder, const int64_t* __restrict__ arrange,
                        const int32_t* __restrict__ pos_ell, const int32_t* __restrict__ pos_er,
                        int64_t n, int64_t warp, int64_t vec, int64_t lim,
                        V* __restrict__ val_ell, uint16_t* __restrict__ col_ell,
                        V* __restrict__ val_er, uint32_t* __restrict__ col_er, int* __restrict__ bad) {
  for (int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; r < n;
       r += int64_t(gridDim.x) * blockDim.x) {
    const int64_t nr = reorder[r];
    const int64_t base = (nr / vec) * vec;
    const int64_t slot = arrange[r];
    const int32_t pr = part[r];
    int64_t ki = 0, ko = 0;
    for (int64_t j = rptr[r]; j < rptr[r + 1]; ++j) {
      const int64_t c = col[j];
      const double x = val[j];
      if (part[c] == pr) {
        const int64_t loc = reorder[c] - base;
        if (loc < 0 || loc >= lim) {
          atomicExch(bad, 1);
          continue;
        }
        const int64_t d = int64_t(pos_ell[nr / warp]) + nr % warp + ki * warp;
        ++ki;
        col_ell[d] = uint16_t(loc);
        val_ell[d] = V(x);  // float(x): round to nearest even, as numpy astype
      } else {
        if (slot < 0) {
          atomicExch(bad, 2);
          continue;
        }
        const int64_t d = int64_t(pos_er[slot / warp]) + slot % warp + ko * warp;
        ++ko;
        col_er[d] = uint32_t(reorder[c]);
        val_er[d] = V(x);
      }
    }
  }
}

}  // namespace

namespace ehyb {
// pageable host -> device copy of a large array through the process-wide
// pinned double buffer (device.cu: the device-matrix upload); small copies
// go straight through cudaMemcpy
cudaError_t staged_h2d(void* dev, const void* host, size_t bytes) {
  Staging st;
  return st.h2d(dev, host, bytes);
}
}  // namespace ehyb

struct ehyb_gprep {
  int device = 0;
  Staging stage;
  int64_t n = 0, nnz = 0;
  DevBuf rptr;  // int64 [n+1]
  DevBuf key;   // uint64 [nnz] grouped (row << 32 | col)
  DevBuf col;   // int32 [nnz] grouped columns
  DevBuf val;   // double [nnz] grouped values
};

namespace {

struct Guard {
  int prev = -1;
  explicit Guard(int d) {
    cudaGetDevice(&prev);
    cudaSetDevice(d);
  }
  ~Guard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

// exclusive scan of int64 counts into out (n + 1 entries)
cudaError_t scan_excl(const int64_t* in, int64_t n, int64_t* out) {
  size_t tmp = 0;
  cudaError_t e = cub::DeviceScan::ExclusiveSum(nullptr, tmp, in, out, int(n + 1));
  if (e != cudaSuccess) return e;
  DevBuf t;
  if ((e = t.alloc(tmp)) != cudaSuccess) return e;
  return cub::DeviceScan::ExclusiveSum(t.p, tmp, in, out, int(n + 1));
}

template <typename K, typename V>
cudaError_t sort_pairs(const K* ki, K* ko, const V* vi, V* vo, int64_t n, int end_bit) {
  size_t tmp = 0;
  cudaError_t e = cub::DeviceRadixSort::SortPairs(nullptr, tmp, ki, ko, vi, vo, n, 0, end_bit);
  if (e != cudaSuccess) return e;
  DevBuf t;
  if ((e = t.alloc(tmp)) != cudaSuccess) return e;
  return cub::DeviceRadixSort::SortPairs(t.p, tmp, ki, ko, vi, vo, n, 0, end_bit);
}

template <typename K>
cudaError_t sort_keys(const K* ki, K* ko, int64_t n, int end_bit) {
  size_t tmp = 0;
  cudaError_t e = cub::DeviceRadixSort::SortKeys(nullptr, tmp, ki, ko, n, 0, end_bit);
  if (e != cudaSuccess) return e;
  DevBuf t;
  if ((e = t.alloc(tmp)) != cudaSuccess) return e;
  return cub::DeviceRadixSort::SortKeys(t.p, tmp, ki, ko, n, 0, end_bit);
}

}  // namespace

extern "C" {

EHYB_API int ehyb_gprep_create(int64_t n, int64_t nnz, const int64_t* rows, const int64_t* cols,
                               const double* values, int device, ehyb_gprep** out) {
  EHYB_TRY {
    if (!out) return fail("null argument");
    if (n < 0 || n > INT32_MAX || nnz < 0) return fail("graph dimension outside int32 range");
    int ndev = 0;
    GP_TRY(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) return fail("invalid CUDA device ordinal", EHYB_ECUDA);
    Guard g(device);
    StageTimer st;
    auto c = std::make_unique<ehyb_gprep>();
    c->device = device;
    c->n = n;
    c->nnz = nnz;
    DevBuf rd, cd, vd, kin, vout;
    GP_TRY(rd.alloc(size_t(nnz) * 8));
    GP_TRY(cd.alloc(size_t(nnz) * 8));
    GP_TRY(vd.alloc(size_t(nnz) * 8));
    st.mark("create: device alloc");
    if (nnz) {
      GP_TRY(c->stage.h2d(rd.p, rows, size_t(nnz) * 8));
      GP_TRY(c->stage.h2d(cd.p, cols, size_t(nnz) * 8));
      GP_TRY(c->stage.h2d(vd.p, values, size_t(nnz) * 8));
    }
    st.mark("create: H2D rows/cols/vals");
    GP_TRY(kin.alloc(size_t(nnz) * 8));
    k_pack_rc<<<blocks_for(nnz), kT>>>(rd.as<int64_t>(), cd.as<int64_t>(), nnz, kin.as<uint64_t>());
    GP_TRY(cudaGetLastError());
    rd.alloc(0);
    cd.alloc(0);
    st.mark("create: pack keys");
    // (row, col) stable: duplicates keep entry order, as np.lexsort((cols, rows))
    GP_TRY(c->key.alloc(size_t(nnz) * 8));
    GP_TRY(c->val.alloc(size_t(nnz) * 8));
    st.mark("create: alloc key/val");
    if (nnz)
      GP_TRY(sort_pairs(kin.as<uint64_t>(), c->key.as<uint64_t>(), vd.as<double>(),
                        c->val.as<double>(), nnz, 32 + bits_for(uint64_t(std::max<int64_t>(n, 1)))));
    st.mark("create: sort (row, col)");
    kin.alloc(0);
    vd.alloc(0);
    DevBuf cnt;
    GP_TRY(cnt.alloc(size_t(n + 1) * 8));
    GP_TRY(cudaMemset(cnt.p, 0, size_t(n + 1) * 8));
    k_row_count<<<blocks_for(nnz), kT>>>(c->key.as<uint64_t>(), nnz, cnt.as<int64_t>());
    GP_TRY(c->rptr.alloc(size_t(n + 1) * 8));
    GP_TRY(scan_excl(cnt.as<int64_t>(), n, c->rptr.as<int64_t>()));
    GP_TRY(c->col.alloc(size_t(nnz) * 4));
    k_split_cols<<<blocks_for(nnz), kT>>>(c->key.as<uint64_t>(), nnz, c->col.as<int32_t>());
    GP_TRY(cudaDeviceSynchronize());
    st.mark("create: row pointers");
    *out = c.release();
    return 0;
  }
  EHYB_CATCH
}

EHYB_API int ehyb_gprep_destroy(ehyb_gprep* c) {
  if (!c) return 0;
  Guard g(c->device);
  delete c;
  return 0;
}

// partition.py:77-98: adj_ptr (caller, n+1 int64) and the adjacency (library
// allocated int32, released with ehyb_free), np.unique order
EHYB_API int ehyb_gprep_build_graph(ehyb_gprep* c, int64_t* adj_ptr, int32_t** out_adj,
                                    int64_t* out_n_adj) {
  EHYB_TRY {
    if (!c || !adj_ptr || !out_adj || !out_n_adj) return fail("null argument");
    Guard g(c->device);
    const int64_t n = c->n, nnz = c->nnz;
    DevBuf flag, at;
    GP_TRY(flag.alloc(size_t(nnz + 1) * 8));
    GP_TRY(at.alloc(size_t(nnz + 1) * 8));
    GP_TRY(cudaMemset(flag.p, 0, size_t(nnz + 1) * 8));
    k_offdiag_flag<<<blocks_for(nnz), kT>>>(c->key.as<uint64_t>(), nnz, flag.as<int64_t>());
    GP_TRY(scan_excl(flag.as<int64_t>(), nnz, at.as<int64_t>()));
    int64_t m = 0;
    GP_TRY(cudaMemcpy(&m, at.as<int64_t>() + nnz, 8, cudaMemcpyDeviceToHost));
    flag.alloc(0);
    DevBuf keys, sorted;
    GP_TRY(keys.alloc(size_t(2 * m) * 8));
    k_sym_keys<<<blocks_for(nnz), kT>>>(c->key.as<uint64_t>(), at.as<int64_t>(), nnz, m,
                                        keys.as<uint64_t>());
    GP_TRY(cudaGetLastError());
    at.alloc(0);
    GP_TRY(sorted.alloc(size_t(2 * m) * 8));
    if (m) GP_TRY(sort_keys(keys.as<uint64_t>(), sorted.as<uint64_t>(), 2 * m,
                            32 + bits_for(uint64_t(std::max<int64_t>(n, 1)))));
    // unique
    DevBuf nsel;
    GP_TRY(nsel.alloc(8));
    size_t tmp = 0;
    GP_TRY(cub::DeviceSelect::Unique(nullptr, tmp, sorted.as<uint64_t>(), keys.as<uint64_t>(),
                                     nsel.as<int64_t>(), 2 * m));
    {
      DevBuf t;
      GP_TRY(t.alloc(tmp));
      GP_TRY(cub::DeviceSelect::Unique(t.p, tmp, sorted.as<uint64_t>(), keys.as<uint64_t>(),
                                       nsel.as<int64_t>(), 2 * m));
    }
    int64_t nu = 0;
    GP_TRY(cudaMemcpy(&nu, nsel.p, 8, cudaMemcpyDeviceToHost));
    sorted.alloc(0);
    DevBuf adj, cnt, ptr;
    GP_TRY(adj.alloc(size_t(nu) * 4));
    GP_TRY(cnt.alloc(size_t(n + 1) * 8));
    GP_TRY(cudaMemset(cnt.p, 0, size_t(n + 1) * 8));
    k_adj_out<<<blocks_for(nu), kT>>>(keys.as<uint64_t>(), nu, adj.as<int32_t>(), cnt.as<int64_t>());
    GP_TRY(ptr.alloc(size_t(n + 1) * 8));
    GP_TRY(scan_excl(cnt.as<int64_t>(), n, ptr.as<int64_t>()));
    int32_t* h = static_cast<int32_t*>(std::malloc(size_t(std::max<int64_t>(nu, 1)) * 4));
    if (!h) return ehyb::fail_oom();
    cudaError_t e1 = c->stage.d2h(h, adj.p, size_t(nu) * 4);
    cudaError_t e2 = c->stage.d2h(adj_ptr, ptr.p, size_t(n + 1) * 8);
    if (e1 != cudaSuccess || e2 != cudaSuccess) {
      std::free(h);
      GP_TRY(e1 != cudaSuccess ? e1 : e2);
    }
    *out_adj = h;
    *out_n_adj = nu;
    return 0;
  }
  EHYB_CATCH
}

// format.py:123-409 in one pass on the device. Fixed-size outputs go to the
// caller's arrays (the shapes of ehyb_classify_rows / ehyb_build_reorder_plan
// / ehyb_assemble); er_row_order, y_idx_er and the four slab arrays are
// library-allocated (ehyb_free), their lengths returned.
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
                                 void** out_val_er, uint32_t** out_col_er, int64_t* out_slots_er) {
  EHYB_TRY {
    if (!c || !assignment) return fail("null argument");
    if (tau != 4 && tau != 8) return fail("tau must be 4 or 8");
    if (warp < 1 || vec < 1 || n_parts < 1) return fail("invalid EHYB parameters");
    Guard g(c->device);
    StageTimer st;
    const int64_t n = c->n;
    const int64_t padded = n_parts * vec;
    for (int64_t i = 0; i < n; ++i)
      if (assignment[i] < 0 || assignment[i] >= n_parts) return fail("partition id out of range");
    // assignment -> int32 on the device
    DevBuf a64, part;
    GP_TRY(a64.alloc(size_t(n) * 8));
    GP_TRY(part.alloc(size_t(n) * 4));
    if (n) GP_TRY(c->stage.h2d(a64.p, assignment, size_t(n) * 8));
    k_i64_to_i32<<<blocks_for(n), kT>>>(a64.as<int64_t>(), n, part.as<int32_t>());
    a64.alloc(0);
    // classify_rows
    DevBuf din, dout;
    GP_TRY(din.alloc(size_t(n) * 8));
    GP_TRY(dout.alloc(size_t(n) * 8));
    k_classify<<<blocks_for(n), kT>>>(c->rptr.as<int64_t>(), c->col.as<int32_t>(), part.as<int32_t>(),
                                      n, din.as<int64_t>(), dout.as<int64_t>());
    GP_TRY(cudaGetLastError());
    st.mark("assemble: H2D part + classify");
    // row_order: stable sort of (part, -inner) over rows in ascending order
    DevBuf k1, k2, v1, rord;
    GP_TRY(k1.alloc(size_t(n) * 8));
    GP_TRY(k2.alloc(size_t(n) * 8));
    GP_TRY(v1.alloc(size_t(n) * 8));
    GP_TRY(rord.alloc(size_t(n) * 8));
    k_order_keys<<<blocks_for(n), kT>>>(part.as<int32_t>(), din.as<int64_t>(), n, k1.as<uint64_t>(),
                                        v1.as<int64_t>());
    if (n) GP_TRY(sort_pairs(k1.as<uint64_t>(), k2.as<uint64_t>(), v1.as<int64_t>(), rord.as<int64_t>(),
                             n, 32 + bits_for(uint64_t(n_parts))));
    k1.alloc(0);
    k2.alloc(0);
    // er_row_order: rows with outer > 0, outer descending, row ascending
    DevBuf ids, sel, nsel;
    GP_TRY(ids.alloc(size_t(n) * 8));
    GP_TRY(sel.alloc(size_t(n) * 8));
    GP_TRY(nsel.alloc(8));
    k_iota<<<blocks_for(n), kT>>>(ids.as<int64_t>(), n);
    size_t tmp = 0;
    HasOuter pred{dout.as<int64_t>()};
    GP_TRY(cub::DeviceSelect::If(nullptr, tmp, ids.as<int64_t>(), sel.as<int64_t>(),
                                 nsel.as<int64_t>(), n, pred));
    {
      DevBuf t;
      GP_TRY(t.alloc(tmp));
      GP_TRY(cub::DeviceSelect::If(t.p, tmp, ids.as<int64_t>(), sel.as<int64_t>(),
                                   nsel.as<int64_t>(), n, pred));
    }
    int64_t n_er = 0;
    GP_TRY(cudaMemcpy(&n_er, nsel.p, 8, cudaMemcpyDeviceToHost));
    DevBuf ek, ek2, eord;
    GP_TRY(ek.alloc(size_t(n_er) * 4));
    GP_TRY(ek2.alloc(size_t(n_er) * 4));
    GP_TRY(eord.alloc(size_t(n_er) * 8));
    k_er_keys<<<blocks_for(n_er), kT>>>(sel.as<int64_t>(), dout.as<int64_t>(), n_er, ek.as<uint32_t>());
    if (n_er) GP_TRY(sort_pairs(ek.as<uint32_t>(), ek2.as<uint32_t>(), sel.as<int64_t>(),
                                eord.as<int64_t>(), n_er, 32));
    ek.alloc(0);
    ek2.alloc(0);
    st.mark("assemble: row / ER orders");
    // build_reorder_plan (format.py:161-199)
    DevBuf occ, start;
    GP_TRY(occ.alloc(size_t(n_parts + 1) * 8));
    GP_TRY(start.alloc(size_t(n_parts + 1) * 8));
    GP_TRY(cudaMemset(occ.p, 0, size_t(n_parts + 1) * 8));
    k_part_hist<<<blocks_for(n), kT>>>(part.as<int32_t>(), n, occ.as<int64_t>());
    std::vector<int64_t> hocc(size_t(n_parts) + 1, 0);
    GP_TRY(cudaMemcpy(hocc.data(), occ.p, size_t(n_parts) * 8, cudaMemcpyDeviceToHost));
    for (int64_t p = 0; p < n_parts; ++p)
      if (hocc[size_t(p)] > vec) return fail("a partition exceeds the vector cache capacity");
    std::vector<int64_t> hstart(size_t(n_parts) + 1, 0), hfree(size_t(n_parts) + 1, 0);
    for (int64_t p = 0; p < n_parts; ++p) {
      hstart[size_t(p) + 1] = hstart[size_t(p)] + hocc[size_t(p)];
      hfree[size_t(p) + 1] = hfree[size_t(p)] + (vec - hocc[size_t(p)]);
    }
    DevBuf fstart, dreo, dinv, darr, dyidx;
    GP_TRY(cudaMemcpy(start.p, hstart.data(), size_t(n_parts + 1) * 8, cudaMemcpyHostToDevice));
    GP_TRY(fstart.alloc(size_t(n_parts + 1) * 8));
    GP_TRY(cudaMemcpy(fstart.p, hfree.data(), size_t(n_parts + 1) * 8, cudaMemcpyHostToDevice));
    GP_TRY(dreo.alloc(size_t(padded) * 8));
    GP_TRY(dinv.alloc(size_t(padded) * 8));
    GP_TRY(darr.alloc(size_t(n) * 8));
    GP_TRY(dyidx.alloc(size_t(n_er) * 8));
    k_reorder<<<blocks_for(n), kT>>>(rord.as<int64_t>(), part.as<int32_t>(), start.as<int64_t>(), n,
                                     vec, dreo.as<int64_t>());
    k_pad_ids<<<unsigned(n_parts), kT>>>(occ.as<int64_t>(), fstart.as<int64_t>(), n_parts, vec, n,
                                         dreo.as<int64_t>());
    k_inverse<<<blocks_for(padded), kT>>>(dreo.as<int64_t>(), padded, dinv.as<int64_t>());
    k_fill_i64<<<blocks_for(n), kT>>>(darr.as<int64_t>(), n, -1);
    k_arrange<<<blocks_for(n_er), kT>>>(eord.as<int64_t>(), dreo.as<int64_t>(), n_er,
                                        darr.as<int64_t>(), dyidx.as<int64_t>());
    GP_TRY(cudaGetLastError());
    st.mark("assemble: reorder plan");
    // assemble_ehyb (format.py:302-409): row widths, slice widths, positions
    const int64_t n_sl = padded / warp;
    const int64_t n_er_sl = n_er ? (n_er + warp - 1) / warp : 0;
    DevBuf ellw, erw, wid_ell, wid_er, sl_ell, sl_er, ex_ell, ex_er, pos_ell, pos_er;
    GP_TRY(ellw.alloc(size_t(padded) * 4));
    GP_TRY(erw.alloc(size_t(n_er) * 4));
    GP_TRY(cudaMemset(ellw.p, 0, size_t(padded) * 4));
    k_row_widths<<<blocks_for(n), kT>>>(din.as<int64_t>(), dout.as<int64_t>(), dreo.as<int64_t>(),
                                        darr.as<int64_t>(), n, ellw.as<int32_t>(), erw.as<int32_t>());
    GP_TRY(wid_ell.alloc(size_t(n_sl) * 4));
    GP_TRY(sl_ell.alloc(size_t(n_sl + 1) * 8));
    GP_TRY(ex_ell.alloc(size_t(n_sl + 1) * 8));
    GP_TRY(wid_er.alloc(size_t(n_er_sl) * 4));
    GP_TRY(sl_er.alloc(size_t(n_er_sl + 1) * 8));
    GP_TRY(ex_er.alloc(size_t(n_er_sl + 1) * 8));
    GP_TRY(cudaMemset(sl_ell.p, 0, size_t(n_sl + 1) * 8));
    GP_TRY(cudaMemset(sl_er.p, 0, size_t(n_er_sl + 1) * 8));
    k_slice_width<<<blocks_for(n_sl), kT>>>(ellw.as<int32_t>(), padded, warp, n_sl,
                                            wid_ell.as<int32_t>(), sl_ell.as<int64_t>());
    k_slice_width<<<blocks_for(n_er_sl), kT>>>(erw.as<int32_t>(), n_er, warp, n_er_sl,
                                               wid_er.as<int32_t>(), sl_er.as<int64_t>());
    GP_TRY(scan_excl(sl_ell.as<int64_t>(), n_sl, ex_ell.as<int64_t>()));
    GP_TRY(scan_excl(sl_er.as<int64_t>(), n_er_sl, ex_er.as<int64_t>()));
    int64_t slots_ell = 0, slots_er = 0;
    GP_TRY(cudaMemcpy(&slots_ell, ex_ell.as<int64_t>() + n_sl, 8, cudaMemcpyDeviceToHost));
    GP_TRY(cudaMemcpy(&slots_er, ex_er.as<int64_t>() + n_er_sl, 8, cudaMemcpyDeviceToHost));
    if (slots_ell > INT32_MAX) return fail("ELL slot count exceeds the int32 position range");
    if (slots_er > INT32_MAX) return fail("ER slot count exceeds the int32 position range");
    GP_TRY(pos_ell.alloc(size_t(n_sl + 1) * 4));
    GP_TRY(pos_er.alloc(size_t(n_er_sl + 1) * 4));
    k_positions32<<<blocks_for(n_sl + 1), kT>>>(ex_ell.as<int64_t>(), n_sl, slots_ell, pos_ell.as<int32_t>());
    k_positions32<<<blocks_for(n_er_sl + 1), kT>>>(ex_er.as<int64_t>(), n_er_sl, slots_er, pos_er.as<int32_t>());
    st.mark("assemble: widths / positions");
    // placement; padding slots stay 0.0 / column 0 (format.py:350-351, 379-380)
    const size_t vb = size_t(tau);
    DevBuf dve, dce, dvr, dcr, dbad;
    GP_TRY(dve.alloc(size_t(slots_ell) * vb));
    GP_TRY(dce.alloc(size_t(slots_ell) * 2));
    GP_TRY(dvr.alloc(size_t(slots_er) * vb));
    GP_TRY(dcr.alloc(size_t(slots_er) * 4));
    GP_TRY(dbad.alloc(4));
    GP_TRY(cudaMemset(dve.p, 0, size_t(slots_ell) * vb));
    GP_TRY(cudaMemset(dce.p, 0, size_t(slots_ell) * 2));
    GP_TRY(cudaMemset(dvr.p, 0, size_t(slots_er) * vb));
    GP_TRY(cudaMemset(dcr.p, 0, size_t(slots_er) * 4));
    GP_TRY(cudaMemset(dbad.p, 0, 4));
    const int64_t lim = std::min<int64_t>(vec, EHYB_MAX_LOCAL_INDEX);
    if (tau == 4)
      k_place<float><<<blocks_for(n), kT>>>(c->rptr.as<int64_t>(), c->col.as<int32_t>(), c->val.as<double>(),
                                            part.as<int32_t>(), dreo.as<int64_t>(), darr.as<int64_t>(),
                                            pos_ell.as<int32_t>(), pos_er.as<int32_t>(), n, warp, vec, lim,
                                            dve.as<float>(), dce.as<uint16_t>(), dvr.as<float>(),
                                            dcr.as<uint32_t>(), dbad.as<int>());
    else
      k_place<double><<<blocks_for(n), kT>>>(c->rptr.as<int64_t>(), c->col.as<int32_t>(), c->val.as<double>(),
                                             part.as<int32_t>(), dreo.as<int64_t>(), darr.as<int64_t>(),
                                             pos_ell.as<int32_t>(), pos_er.as<int32_t>(), n, warp, vec, lim,
                                             dve.as<double>(), dce.as<uint16_t>(), dvr.as<double>(),
                                             dcr.as<uint32_t>(), dbad.as<int>());
    GP_TRY(cudaGetLastError());
    int bad = 0;
    GP_TRY(cudaMemcpy(&bad, dbad.p, 4, cudaMemcpyDeviceToHost));
    if (bad)
      return fail(bad == 1 ? "inner entry maps outside its partition cache window"
                           : "outer entry in a row missing from the ER arrangement");
    st.mark("assemble: placement");
    // results back to the host
    auto d2h = [&](void* dst, const DevBuf& src, size_t bytes) {
      return bytes ? c->stage.d2h(dst, src.p, bytes) : cudaSuccess;
    };
    GP_TRY(d2h(inner, din, size_t(n) * 8));
    GP_TRY(d2h(outer, dout, size_t(n) * 8));
    GP_TRY(d2h(row_order, rord, size_t(n) * 8));
    GP_TRY(d2h(reorder, dreo, size_t(padded) * 8));
    GP_TRY(d2h(inverse, dinv, size_t(padded) * 8));
    GP_TRY(d2h(arrange, darr, size_t(n) * 8));
    GP_TRY(d2h(position_ell, pos_ell, size_t(n_sl + 1) * 4));
    GP_TRY(d2h(width_ell, wid_ell, size_t(n_sl) * 4));
    GP_TRY(d2h(ell_row_widths, ellw, size_t(padded) * 4));
    for (int64_t p = 0; p <= n_parts; ++p) part_boundary[p] = int32_t(p * vec);
    st.mark("assemble: D2H caller arrays");
    // library-allocated outputs
    std::vector<void*> owned;
    auto lib_alloc = [&](size_t bytes) {
      void* p = std::malloc(std::max<size_t>(bytes, 8));
      owned.push_back(p);
      return p;
    };
    auto release = [&]() {
      for (void* p : owned) std::free(p);
    };
    int64_t* h_eord = static_cast<int64_t*>(lib_alloc(size_t(n_er) * 8));
    int64_t* h_yidx = static_cast<int64_t*>(lib_alloc(size_t(n_er) * 8));
    int32_t* h_pos_er = static_cast<int32_t*>(lib_alloc(size_t(n_er_sl + 1) * 4));
    int32_t* h_wid_er = static_cast<int32_t*>(lib_alloc(size_t(n_er_sl) * 4));
    int32_t* h_erw = static_cast<int32_t*>(lib_alloc(size_t(n_er) * 4));
    void* h_ve = lib_alloc(size_t(slots_ell) * vb);
    uint16_t* h_ce = static_cast<uint16_t*>(lib_alloc(size_t(slots_ell) * 2));
    void* h_vr = lib_alloc(size_t(slots_er) * vb);
    uint32_t* h_cr = static_cast<uint32_t*>(lib_alloc(size_t(slots_er) * 4));
    for (void* p : owned)
      if (!p) {
        release();
        return ehyb::fail_oom();
      }
    cudaError_t e = cudaSuccess;
    for (auto cp : {std::make_pair(std::make_pair(static_cast<void*>(h_eord), &eord), size_t(n_er) * 8),
                    std::make_pair(std::make_pair(static_cast<void*>(h_yidx), &dyidx), size_t(n_er) * 8),
                    std::make_pair(std::make_pair(static_cast<void*>(h_pos_er), &pos_er), size_t(n_er_sl + 1) * 4),
                    std::make_pair(std::make_pair(static_cast<void*>(h_wid_er), &wid_er), size_t(n_er_sl) * 4),
                    std::make_pair(std::make_pair(static_cast<void*>(h_erw), &erw), size_t(n_er) * 4),
                    std::make_pair(std::make_pair(h_ve, &dve), size_t(slots_ell) * vb),
                    std::make_pair(std::make_pair(static_cast<void*>(h_ce), &dce), size_t(slots_ell) * 2),
                    std::make_pair(std::make_pair(h_vr, &dvr), size_t(slots_er) * vb),
                    std::make_pair(std::make_pair(static_cast<void*>(h_cr), &dcr), size_t(slots_er) * 4)}) {
      if (e == cudaSuccess) e = d2h(cp.first.first, *cp.first.second, cp.second);
    }
    if (e != cudaSuccess) {
      release();
      GP_TRY(e);
    }
    st.mark("assemble: D2H library arrays");
    *out_er_row_order = h_eord;
    *out_n_er = n_er;
    *out_y_idx_er = h_yidx;
    *out_position_er = h_pos_er;
    *out_width_er = h_wid_er;
    *out_er_row_widths = h_erw;
    *out_val_ell = h_ve;
    *out_col_ell = h_ce;
    *out_slots_ell = slots_ell;
    *out_val_er = h_vr;
    *out_col_er = h_cr;
    *out_slots_er = slots_er;
    return 0;
  }
  EHYB_CATCH
}

}  // extern "C"
