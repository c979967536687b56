#include <memory>
// EHYB host preprocessing — bit-exact C++17 restatement of the reference
// pipeline (arXiv 2204.06666 reference package `ehyb`):
//   compute_params      format.py:83-107   (Eq.1-2)
//   build_graph         partition.py:77-98
//   partition_graph     partition.py:101-204 (BFS region growing + refinement)
//   rebalance_partition partition.py:224-262
//   classify_rows       format.py:123-137  (Alg.1 row classification)
//   build_reorder_plan  format.py:161-199  (Alg.1 reorder / arrange tables)
//   assemble_ehyb       format.py:302-409  (Alg.2 SELL placement)
//   EhybMatrix.check    format.py:250-299
// Every output array is byte-identical to the reference's on the same input
// (pinned by tests/test_prep.py against golden digests of the reference).
// Work that does not feed an order-dependent decision runs in parallel
// (OpenMP); the partitioner is inherently sequential and runs on one core
// with O(log n) seed selection instead of the reference's O(n) rescans.

#include "ehyb_common.h"

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <vector>

#include <omp.h>

namespace {

// ------------------------------------------------------------------ MT19937
// CPython's random.Random: init_by_array over the 32-bit words of |seed|,
// randrange(m) = rejection sampling of getrandbits(bit_length(m)).
struct MT19937 {
  static constexpr int N = 624, M = 397;
  uint32_t mt[N];
  int mti = N + 1;

  void init_genrand(uint32_t s) {
    mt[0] = s;
    for (int i = 1; i < N; ++i)
      mt[i] = 1812433253u * (mt[i - 1] ^ (mt[i - 1] >> 30)) + uint32_t(i);
    mti = N;
  }
  void init_by_array(const uint32_t* key, int len) {
    init_genrand(19650218u);
    int i = 1, j = 0;
    for (int k = std::max(N, len); k; --k) {
      mt[i] = (mt[i] ^ ((mt[i - 1] ^ (mt[i - 1] >> 30)) * 1664525u)) + key[j] + uint32_t(j);
      ++i; ++j;
      if (i >= N) { mt[0] = mt[N - 1]; i = 1; }
      if (j >= len) j = 0;
    }
    for (int k = N - 1; k; --k) {
      mt[i] = (mt[i] ^ ((mt[i - 1] ^ (mt[i - 1] >> 30)) * 1566083941u)) - uint32_t(i);
      ++i;
      if (i >= N) { mt[0] = mt[N - 1]; i = 1; }
    }
    mt[0] = 0x80000000u;
  }
  explicit MT19937(int64_t seed) {
    uint64_t s = seed < 0 ? uint64_t(-(seed + 1)) + 1u : uint64_t(seed);
    uint32_t key[2] = {uint32_t(s & 0xffffffffu), uint32_t(s >> 32)};
    init_by_array(key, key[1] ? 2 : 1);
  }
  uint32_t next() {
    static const uint32_t mag01[2] = {0u, 0x9908b0dfu};
    if (mti >= N) {
      int kk = 0;
      uint32_t y;
      for (; kk < N - M; ++kk) {
        y = (mt[kk] & 0x80000000u) | (mt[kk + 1] & 0x7fffffffu);
        mt[kk] = mt[kk + M] ^ (y >> 1) ^ mag01[y & 1u];
      }
      for (; kk < N - 1; ++kk) {
        y = (mt[kk] & 0x80000000u) | (mt[kk + 1] & 0x7fffffffu);
        mt[kk] = mt[kk + (M - N)] ^ (y >> 1) ^ mag01[y & 1u];
      }
      y = (mt[N - 1] & 0x80000000u) | (mt[0] & 0x7fffffffu);
      mt[N - 1] = mt[M - 1] ^ (y >> 1) ^ mag01[y & 1u];
      mti = 0;
    }
    uint32_t y = mt[mti++];
    y ^= (y >> 11);
    y ^= (y << 7) & 0x9d2c5680u;
    y ^= (y << 15) & 0xefc60000u;
    y ^= (y >> 18);
    return y;
  }
  // random.Random.randrange(m) for 2 <= m < 2^32
  uint32_t randbelow(uint32_t m) {
    int k = 32 - __builtin_clz(m);
    uint32_t r = next() >> (32 - k);
    while (r >= m) r = next() >> (32 - k);
    return r;
  }
};

// Rank/select set over positions of the degree order: 1 = still unassigned.
// A bitset with per-512-bit block counts and per-64-block super counts: an
// assignment clears one bit and decrements two counters (one random cache
// line instead of a Fenwick tree's ~log2(n) scattered nodes); the rare seed
// queries scan counters.
struct RankSet {
  static constexpr int kBlk = 9, kSup = 15;  // 512 bits per block, 32768 per super block
  std::vector<uint64_t> bits;
  std::vector<int32_t> blk, sup;
  int64_t n = 0;
  void init_ones(int64_t n_) {
    n = n_;
    bits.assign(size_t((n + 63) >> 6), ~0ull);
    if (n & 63) bits.back() = (1ull << (n & 63)) - 1;
    blk.assign(size_t((n >> kBlk) + 1), 0);
    sup.assign(size_t((n >> kSup) + 1), 0);
    for (int64_t i = 0; i < n; i += 64) {
      const int c = __builtin_popcountll(bits[size_t(i >> 6)]);
      blk[size_t(i >> kBlk)] += c;
      sup[size_t(i >> kSup)] += c;
    }
  }
  void dec(int64_t pos) {  // 0-based, the bit must be set
    bits[size_t(pos >> 6)] &= ~(1ull << (pos & 63));
    blk[size_t(pos >> kBlk)] -= 1;
    sup[size_t(pos >> kSup)] -= 1;
  }
  int64_t prefix(int64_t cnt) const {  // set bits in [0, cnt)
    int64_t s = 0;
    const int64_t S = cnt >> kSup;
    for (int64_t i = 0; i < S; ++i) s += sup[size_t(i)];
    for (int64_t i = S << (kSup - kBlk); i < (cnt >> kBlk); ++i) s += blk[size_t(i)];
    for (int64_t w = (cnt >> kBlk) << (kBlk - 6); w < (cnt >> 6); ++w)
      s += __builtin_popcountll(bits[size_t(w)]);
    if (cnt & 63) s += __builtin_popcountll(bits[size_t(cnt >> 6)] & ((1ull << (cnt & 63)) - 1));
    return s;
  }
  // smallest 0-based position p with prefix(p + 1) >= target (target >= 1)
  int64_t find(int64_t target) const {
    int64_t i = 0;
    while (sup[size_t(i)] < target) target -= sup[size_t(i++)];
    int64_t b = i << (kSup - kBlk);
    while (blk[size_t(b)] < target) target -= blk[size_t(b++)];
    int64_t w = b << (kBlk - 6);
    for (;; ++w) {
      const int c = __builtin_popcountll(bits[size_t(w)]);
      if (c >= target) break;
      target -= c;
    }
    uint64_t x = bits[size_t(w)];
    for (int64_t k = 1; k < target; ++k) x &= x - 1;  // drop the lowest target-1 set bits
    return (w << 6) + __builtin_ctzll(x);
  }
};

inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

// below this trip count a loop runs serially (OpenMP fork/join would dominate)
constexpr int64_t kParallelMin = 1 << 15;

// Entries grouped by row and ordered by (column, entry index) — the order of
// np.lexsort((cols, rows)) including duplicate coordinates — as a row pointer
// plus the sorted columns and values. Per-chunk histograms scatter the
// entries into buckets of 2^shift consecutive rows (chunks in entry order, so
// the scatter is stable), then each L2-sized bucket is LSD-radix sorted by
// column and by row (stable passes: duplicates keep entry order).
void group_rows(int64_t n, int64_t nnz, const int64_t* rows, const int64_t* cols,
                const double* values, std::vector<int64_t>& rptr,
                std::unique_ptr<int32_t[]>& scol, std::unique_ptr<double[]>& sval) {
  int shift = 0;
  while ((n >> shift) > 4096) ++shift;
  const int64_t n_b = (n >> shift) + 1;
  const int64_t nt = nnz > kParallelMin ? std::max(1, omp_get_max_threads()) : 1;
  const int64_t chunk = cdiv(std::max<int64_t>(nnz, 1), nt);
  std::vector<int64_t> hist(size_t(nt) * size_t(n_b), 0);
#pragma omp parallel for schedule(static, 1) if (nt > 1)
  for (int64_t t = 0; t < nt; ++t) {
    int64_t* h = hist.data() + size_t(t) * size_t(n_b);
    const int64_t e0 = std::min(nnz, t * chunk), e1 = std::min(nnz, e0 + chunk);
    for (int64_t e = e0; e < e1; ++e) h[rows[e] >> shift]++;
  }
  std::vector<int64_t> bstart(size_t(n_b) + 1, 0);
  int64_t acc = 0;
  for (int64_t i = 0; i < n_b; ++i) {
    bstart[size_t(i)] = acc;
    for (int64_t t = 0; t < nt; ++t) {
      int64_t& h = hist[size_t(t) * size_t(n_b) + size_t(i)];
      const int64_t c = h;
      h = acc;
      acc += c;
    }
  }
  bstart[size_t(n_b)] = acc;
  std::unique_ptr<uint64_t[]> keys(new uint64_t[size_t(std::max<int64_t>(nnz, 1))]);
  std::unique_ptr<double[]> kval(new double[size_t(std::max<int64_t>(nnz, 1))]);
#pragma omp parallel for schedule(static, 1) if (nt > 1)
  for (int64_t t = 0; t < nt; ++t) {
    int64_t* h = hist.data() + size_t(t) * size_t(n_b);
    const int64_t e0 = std::min(nnz, t * chunk), e1 = std::min(nnz, e0 + chunk);
    for (int64_t e = e0; e < e1; ++e) {
      const int64_t d = h[rows[e] >> shift]++;
      keys[size_t(d)] = (uint64_t(rows[e]) << 32) | uint64_t(cols[e]);
      kval[size_t(d)] = values[e];
    }
  }
  scol.reset(new int32_t[size_t(std::max<int64_t>(nnz, 1))]);
  sval.reset(new double[size_t(std::max<int64_t>(nnz, 1))]);
  rptr.assign(size_t(n) + 1, 0);
  int cbits = 0;
  while (cbits < 32 && (int64_t(1) << cbits) < n) ++cbits;
  constexpr int kRB = 11;
#pragma omp parallel if (nt > 1)
  {
    std::vector<uint64_t> ka, kb;
    std::vector<double> va, vb;
    std::vector<int64_t> cnt(size_t(1) << std::max(kRB, shift));  // the vertex pass uses shift bits
#pragma omp for schedule(dynamic, 1)
    for (int64_t bi = 0; bi < n_b; ++bi) {
      const int64_t r0 = bi << shift;
      const int64_t k0 = bstart[size_t(bi)], k1 = bstart[size_t(bi) + 1], nk = k1 - k0;
      if (nk == 0) continue;
      ka.assign(keys.get() + k0, keys.get() + k1);
      va.assign(kval.get() + k0, kval.get() + k1);
      kb.resize(size_t(nk));
      vb.resize(size_t(nk));
      auto pass = [&](int lo, int bits, uint64_t base) {
        const uint64_t mask = (uint64_t(1) << bits) - 1;
        std::fill(cnt.begin(), cnt.begin() + (int64_t(1) << bits), 0);
        for (int64_t k = 0; k < nk; ++k) cnt[size_t(((ka[size_t(k)] - base) >> lo) & mask)]++;
        int64_t a = 0;
        for (int64_t i = 0; i < (int64_t(1) << bits); ++i) {
          const int64_t c = cnt[size_t(i)];
          cnt[size_t(i)] = a;
          a += c;
        }
        for (int64_t k = 0; k < nk; ++k) {
          const int64_t d = cnt[size_t(((ka[size_t(k)] - base) >> lo) & mask)]++;
          kb[size_t(d)] = ka[size_t(k)];
          vb[size_t(d)] = va[size_t(k)];
        }
        ka.swap(kb);
        va.swap(vb);
      };
      for (int lo = 0; lo < cbits; lo += kRB) pass(lo, std::min(kRB, cbits - lo), 0);
      if (shift > 0) pass(32, shift, uint64_t(r0) << 32);
      for (int64_t k = 0; k < nk; ++k) {
        scol[size_t(k0 + k)] = int32_t(uint32_t(ka[size_t(k)]));
        sval[size_t(k0 + k)] = va[size_t(k)];
        rptr[size_t(ka[size_t(k)] >> 32) + 1]++;
      }
    }
  }
  for (int64_t i = 0; i < n; ++i) rptr[size_t(i) + 1] += rptr[size_t(i)];
}

}  // namespace

// ===================================================================== API
extern "C" {

EHYB_API int ehyb_compute_params(int64_t dimension, int32_t tau, int64_t procs, int64_t warp,
                                 int64_t shm, int64_t* out_k, int64_t* out_n_parts,
                                 int64_t* out_vec) {
  EHYB_TRY {
    if (dimension < 1) return ehyb::fail("dimension must be >= 1");
    if (tau != 4 && tau != 8) return ehyb::fail("tau must be 4 or 8");
    if (procs < 1 || warp < 1 || shm <= 0) return ehyb::fail("invalid device profile");
    if (warp * tau > shm || warp > EHYB_MAX_LOCAL_INDEX)
      return ehyb::fail(
          "infeasible device profile: a single warp-aligned cache window cannot fit");
    for (int64_t k = 1;; ++k) {
      int64_t n_parts = k * procs;
      int64_t vec = cdiv(cdiv(dimension, n_parts), warp) * warp;
      if (vec * tau <= shm && vec <= EHYB_MAX_LOCAL_INDEX) {
        *out_k = k;
        *out_n_parts = n_parts;
        *out_vec = vec;
        return 0;
      }
    }
  }
  EHYB_CATCH
}

EHYB_API int ehyb_build_graph(int64_t n, int64_t nnz, const int64_t* rows, const int64_t* cols,
                              int64_t* adj_ptr, int32_t** out_adj, int64_t* out_n_adj) {
  EHYB_TRY {
    if (n < 0 || n > INT32_MAX) return ehyb::fail("graph dimension outside int32 range");
    // Every off-diagonal (u,v) contributes the keys u<<32|v and v<<32|u; the
    // sorted distinct keys are np.unique over src*n+dst. Cache-friendly
    // two-level radix order: keys are scattered into buckets of 2^shift
    // consecutive vertices by per-thread histograms (no atomics), then each
    // bucket (L2-sized) is counting-sorted by vertex and every neighbour list
    // sorted and deduplicated locally.
    int shift = 0;
    while ((n >> shift) > 4096) ++shift;
    const int64_t n_b = (n >> shift) + 1;
    // fixed work split (independent of how many threads OpenMP grants)
    const int64_t nt = nnz > kParallelMin ? std::max(1, omp_get_max_threads()) : 1;
    const int64_t chunk = cdiv(std::max<int64_t>(nnz, 1), nt);
    std::vector<int64_t> hist(size_t(nt) * size_t(n_b), 0);
#pragma omp parallel for schedule(static, 1) if (nt > 1)
    for (int64_t t = 0; t < nt; ++t) {
      int64_t* h = hist.data() + size_t(t) * size_t(n_b);
      const int64_t e0 = std::min(nnz, t * chunk), e1 = std::min(nnz, e0 + chunk);
      // row-grouped inputs repeat a bucket many times in a row: count runs in
      // a register instead of a load-increment-store chain on one counter
      int64_t run_b = 0, run_c = 0;
      for (int64_t e = e0; e < e1; ++e) {
        const int64_t u = rows[e], v = cols[e];
        if (u == v) continue;
        const int64_t bu = u >> shift;
        if (bu != run_b) {
          h[run_b] += run_c;
          run_b = bu;
          run_c = 0;
        }
        ++run_c;
        h[v >> shift]++;
      }
      h[run_b] += run_c;
    }
    std::vector<int64_t> bstart(size_t(n_b) + 1, 0);
    {
      int64_t acc = 0;
      for (int64_t i = 0; i < n_b; ++i) {
        bstart[size_t(i)] = acc;
        for (int64_t t = 0; t < nt; ++t) {
          int64_t& h = hist[size_t(t) * size_t(n_b) + size_t(i)];
          const int64_t c = h;
          h = acc;  // chunk t's write cursor in bucket i
          acc += c;
        }
      }
      bstart[size_t(n_b)] = acc;
    }
    const int64_t n_keys = bstart[size_t(n_b)];
    // uninitialised (no serial zero-fill): first touched by the parallel scatter
    std::unique_ptr<uint64_t[]> keys(new uint64_t[size_t(std::max<int64_t>(n_keys, 1))]);
#pragma omp parallel for schedule(static, 1) if (nt > 1)
    for (int64_t t = 0; t < nt; ++t) {
      int64_t* h = hist.data() + size_t(t) * size_t(n_b);
      const int64_t e0 = std::min(nnz, t * chunk), e1 = std::min(nnz, e0 + chunk);
      for (int64_t e = e0; e < e1; ++e) {
        const uint64_t u = uint64_t(rows[e]), v = uint64_t(cols[e]);
        if (u != v) {
          keys[size_t(h[u >> shift]++)] = (u << 32) | v;
          keys[size_t(h[v >> shift]++)] = (v << 32) | u;
        }
      }
    }
    const bool serial = nt == 1;
    // per bucket (L2-sized): LSD radix sort of the keys by neighbour id, then
    // a stable counting pass by vertex, then deduplication — each neighbour
    // list ends up ascending and distinct, compacted at the bucket's start
    std::unique_ptr<int32_t[]> vals(new int32_t[size_t(std::max<int64_t>(n_keys, 1))]);
    std::vector<int64_t> uniq(size_t(n), 0);
    int vbits = 0;
    while (vbits < 32 && (int64_t(1) << vbits) < n) ++vbits;
    constexpr int kRB = 11;
#pragma omp parallel if (!serial)
    {
      std::vector<uint64_t> bufa, bufb;
      std::vector<int64_t> cnt(size_t(1) << std::max(kRB, shift));  // the vertex pass uses shift bits
#pragma omp for schedule(dynamic, 1)
      for (int64_t bi = 0; bi < n_b; ++bi) {
        const int64_t v0 = bi << shift, v1 = std::min<int64_t>(n, (bi + 1) << shift);
        if (v0 >= v1) continue;
        const int64_t k0 = bstart[size_t(bi)], k1 = bstart[size_t(bi) + 1], nk = k1 - k0;
        bufa.assign(keys.get() + k0, keys.get() + k1);
        bufb.resize(size_t(nk));
        auto pass = [&](int lo, int bits, uint64_t base) {  // stable counting pass on key bits [lo, lo+bits)
          const uint64_t mask = (uint64_t(1) << bits) - 1;
          std::fill(cnt.begin(), cnt.begin() + (int64_t(1) << bits), 0);
          for (int64_t k = 0; k < nk; ++k) cnt[size_t(((bufa[size_t(k)] - base) >> lo) & mask)]++;
          int64_t acc = 0;
          for (int64_t i = 0; i < (int64_t(1) << bits); ++i) {
            const int64_t c = cnt[size_t(i)];
            cnt[size_t(i)] = acc;
            acc += c;
          }
          for (int64_t k = 0; k < nk; ++k) {
            const uint64_t key = bufa[size_t(k)];
            bufb[size_t(cnt[size_t(((key - base) >> lo) & mask)]++)] = key;
          }
          bufa.swap(bufb);
        };
        for (int lo = 0; lo < vbits; lo += kRB) pass(lo, std::min(kRB, vbits - lo), 0);
        if (shift > 0) pass(32, shift, uint64_t(v0) << 32);  // by vertex within the bucket
        int32_t* out = vals.get() + k0;
        int64_t w = 0;
        uint64_t prev = ~uint64_t(0);
        for (int64_t k = 0; k < nk; ++k) {
          const uint64_t key = bufa[size_t(k)];
          if (key == prev) continue;
          prev = key;
          out[w++] = int32_t(uint32_t(key));
          uniq[size_t(key >> 32)]++;
        }
      }
    }
    adj_ptr[0] = 0;
    for (int64_t i = 0; i < n; ++i) adj_ptr[i + 1] = adj_ptr[i] + uniq[size_t(i)];
    const int64_t total = adj_ptr[n];
    int32_t* adj = static_cast<int32_t*>(std::malloc(size_t(std::max<int64_t>(total, 1)) * 4));
    if (!adj) return ehyb::fail_oom();
#pragma omp parallel for schedule(dynamic, 16) if (!serial)
    for (int64_t bi = 0; bi < n_b; ++bi) {
      const int64_t v0 = bi << shift, v1 = std::min<int64_t>(n, (bi + 1) << shift);
      if (v0 >= v1) continue;
      std::memcpy(adj + adj_ptr[v0], vals.get() + bstart[size_t(bi)],
                  size_t(adj_ptr[v1] - adj_ptr[v0]) * 4);
    }
    *out_adj = adj;
    *out_n_adj = total;
    return 0;
  }
  EHYB_CATCH
}

EHYB_API int ehyb_partition_graph(int64_t n, const int64_t* adj_ptr, const int32_t* adj,
                                  int64_t n_parts, int64_t capacity, int64_t seed,
                                  int64_t* assignment, int64_t* sizes) {
  EHYB_TRY {
    if (n_parts < 1) return ehyb::fail("n_parts must be >= 1");
    if (capacity < 1 || n_parts * capacity < n)
      return ehyb::fail("infeasible: " + std::to_string(n_parts) + " parts of capacity " +
                        std::to_string(capacity) + " cannot hold " + std::to_string(n) +
                        " vertices");
    MT19937 rng(seed);
    // part ids in a compact int32 copy (half the cache footprint of the
    // caller's int64 array), written back at the end
    std::vector<int32_t> part(size_t(n), -1);
    for (int64_t p = 0; p < n_parts; ++p) sizes[p] = 0;

    // stable degree order of connected vertices (counting sort = stable argsort)
    int64_t max_deg = 0;
    for (int64_t v = 0; v < n; ++v) max_deg = std::max(max_deg, adj_ptr[v + 1] - adj_ptr[v]);
    std::vector<int64_t> deg_start(size_t(max_deg) + 2, 0);
    for (int64_t v = 0; v < n; ++v) {
      int64_t d = adj_ptr[v + 1] - adj_ptr[v];
      if (d > 0) deg_start[size_t(d) + 1]++;
    }
    for (int64_t d = 0; d <= max_deg; ++d) deg_start[size_t(d) + 1] += deg_start[size_t(d)];
    const int64_t n_conn = deg_start[size_t(max_deg) + 1];
    std::vector<int32_t> by_degree(static_cast<size_t>(n_conn));
    std::vector<int64_t> pos_of(size_t(n), -1);
    {
      std::vector<int64_t> fill(deg_start.begin(), deg_start.end());
      for (int64_t v = 0; v < n; ++v) {
        int64_t d = adj_ptr[v + 1] - adj_ptr[v];
        if (d > 0) {
          int64_t p = fill[size_t(d)]++;
          by_degree[size_t(p)] = int32_t(v);
          pos_of[size_t(v)] = p;
        }
      }
    }
    RankSet fw;
    fw.init_ones(n_conn);
    int64_t cursor = 0;

    // assigned flags as a bitset (n/8 bytes: L2-resident where the int32
    // part array is not) for the BFS membership tests
    std::vector<uint64_t> taken(size_t((n + 63) >> 6), 0);
    auto is_taken = [&](int64_t v) { return (taken[size_t(v >> 6)] >> (v & 63)) & 1u; };
    auto assign = [&](int64_t v, int64_t pid) {
      taken[size_t(v >> 6)] |= 1ull << (v & 63);
      part[v] = int32_t(pid);
      sizes[pid] += 1;
      if (pos_of[size_t(v)] >= 0) fw.dec(pos_of[size_t(v)]);
    };
    // partition.py:131-144: first unassigned vertex of minimum degree; when the
    // unassigned part of its equal-degree run holds >1 vertex, draw its index
    auto next_seed = [&]() -> int64_t {
      while (cursor < n_conn && is_taken(by_degree[size_t(cursor)])) ++cursor;
      if (cursor >= n_conn) return -1;
      int64_t d = adj_ptr[by_degree[size_t(cursor)] + 1] - adj_ptr[by_degree[size_t(cursor)]];
      int64_t run_end = deg_start[size_t(d) + 1];
      int64_t before = fw.prefix(cursor);
      int64_t run = fw.prefix(run_end) - before;
      if (run <= 1) return by_degree[size_t(cursor)];
      if (run > int64_t(UINT32_MAX)) throw std::runtime_error("seed run exceeds 2^32");
      int64_t r = rng.randbelow(uint32_t(run));
      return by_degree[size_t(fw.find(before + r + 1))];
    };
    std::vector<int32_t> queue(size_t(std::max<int64_t>(n, 1)));
    // partition.py:146-165: BFS, assigning on enqueue, neighbours ascending
    auto grow = [&](int64_t pid) -> int64_t {
      int64_t start = next_seed();
      if (start < 0) return 0;
      int64_t grown = 1;
      assign(start, pid);
      size_t qh = 0, qt = 0;
      queue[qt++] = int32_t(start);
      while (qh < qt && sizes[pid] < capacity) {
        // software pipeline over the queue (the permuted graphs have no
        // locality): adjacency offsets 16 ahead, lists 8 ahead, the
        // neighbours' assignment words 4 ahead
        if (qh + 16 < qt) __builtin_prefetch(adj_ptr + queue[qh + 16]);
        if (qh + 8 < qt) __builtin_prefetch(adj + adj_ptr[queue[qh + 8]]);
        if (qh + 4 < qt) {
          const int64_t f = queue[qh + 4];
          for (int64_t j = adj_ptr[f]; j < adj_ptr[f + 1]; ++j) __builtin_prefetch(pos_of.data() + adj[j]);
        }
        int64_t u = queue[qh++];
        bool full = false;
        for (int64_t j = adj_ptr[u]; j < adj_ptr[u + 1]; ++j) {
          int64_t w = adj[j];
          if (!is_taken(w)) {
            assign(w, pid);
            ++grown;
            queue[qt++] = int32_t(w);
            if (sizes[pid] == capacity) { full = true; break; }
          }
        }
        if (full) break;
      }
      return grown;
    };

    int64_t left = n_conn;
    for (int64_t pid = 0; pid < n_parts && left > 0; ++pid) left -= grow(pid);
    while (left > 0) {  // partition.py:172-175: first least-full non-full part
      int64_t best = -1;
      for (int64_t p = 0; p < n_parts; ++p)
        if (sizes[p] < capacity && (best < 0 || sizes[p] < sizes[best])) best = p;
      left -= grow(best);
    }
    {  // partition.py:177-183: isolated vertices round-robin over non-full parts
      int64_t pid = 0;
      for (int64_t v = 0; v < n; ++v) {
        if (adj_ptr[v + 1] != adj_ptr[v]) continue;
        while (sizes[pid] >= capacity) pid = (pid + 1) % n_parts;
        part[v] = pid;
        sizes[pid] += 1;
        pid = (pid + 1) % n_parts;
      }
    }
    // partition.py:185-202: one sequential refinement pass. Only parts that
    // neighbour v can score above internal (>= 0), so the argmax over all
    // parts reduces to the adjacent movable parts (first id on ties).
    int64_t nonfull = 0;
    for (int64_t p = 0; p < n_parts; ++p) nonfull += sizes[p] < capacity;
    // A vertex whose neighbours all share its part has touched = {a} and
    // cannot move; that stays true until a neighbour moves. So only boundary
    // vertices (found in parallel) and later neighbours of moved vertices
    // are visited — the same decisions in the same order as the full pass.
    std::vector<uint8_t> active(size_t(n), 0);
#pragma omp parallel for schedule(dynamic, 4096) if (n > kParallelMin)
    for (int64_t v = 0; v < n; ++v) {
      const int32_t a = part[size_t(v)];
      for (int64_t j = adj_ptr[v]; j < adj_ptr[v + 1]; ++j)
        if (part[size_t(adj[j])] != a) {
          active[size_t(v)] = 1;
          break;
        }
    }
    std::vector<int64_t> cnt(size_t(n_parts), 0);
    std::vector<int64_t> touched;
    for (int64_t v = 0; v < n; ++v) {
      if (v + 8 < n && active[size_t(v + 8)])  // neighbours' parts of a vertex 8 ahead
        for (int64_t j = adj_ptr[v + 8]; j < adj_ptr[v + 9]; ++j) __builtin_prefetch(part.data() + adj[j]);
      if (!active[size_t(v)]) continue;
      int64_t a = part[v];
      touched.clear();
      for (int64_t j = adj_ptr[v]; j < adj_ptr[v + 1]; ++j) {
        int64_t q = part[adj[j]];
        if (cnt[size_t(q)]++ == 0) touched.push_back(q);
      }
      int64_t internal = cnt[size_t(a)];
      int64_t movable_any = nonfull - (sizes[a] < capacity ? 1 : 0);
      int64_t best = -1, best_sc = 0;
      if (movable_any > 0) {
        for (int64_t q : touched) {
          if (q == a || sizes[q] >= capacity) continue;
          int64_t sc = cnt[size_t(q)];
          if (sc > best_sc || (sc == best_sc && q < best)) { best = q; best_sc = sc; }
        }
      }
      for (int64_t q : touched) cnt[size_t(q)] = 0;
      if (best >= 0 && best_sc > internal) {
        bool a_was_full = sizes[a] >= capacity;
        part[v] = int32_t(best);
        sizes[a] -= 1;
        sizes[best] += 1;
        if (a_was_full && sizes[a] < capacity) ++nonfull;
        if (sizes[best] >= capacity) --nonfull;
        for (int64_t j = adj_ptr[v]; j < adj_ptr[v + 1]; ++j)
          if (adj[j] > v) active[size_t(adj[j])] = 1;
      }
    }
#pragma omp parallel for schedule(static) if (n > kParallelMin)
    for (int64_t v = 0; v < n; ++v) assignment[v] = part[size_t(v)];
    return 0;
  }
  EHYB_CATCH
}

EHYB_API int ehyb_rebalance_partition(int64_t n, const int64_t* adj_ptr, const int32_t* adj,
                                      int64_t n_parts, int64_t capacity,
                                      const int64_t* assignment_in, int64_t* assignment,
                                      int64_t* sizes) {
  EHYB_TRY {
    if (n_parts * capacity < n) return ehyb::fail("infeasible capacity");
    for (int64_t p = 0; p < n_parts; ++p) sizes[p] = 0;
    for (int64_t v = 0; v < n; ++v) {
      int64_t p = assignment_in[v];
      if (p < 0 || p >= n_parts) return ehyb::fail("partition id out of range");
      assignment[v] = p;
      sizes[p] += 1;
    }
    std::vector<int64_t> targets;
    for (;;) {
      int64_t pid = -1;
      for (int64_t p = 0; p < n_parts; ++p)
        if (sizes[p] > capacity && (pid < 0 || sizes[p] > sizes[pid])) pid = p;
      if (pid < 0) break;
      int64_t best_v = -1, best_ext = -1;
      for (int64_t v = 0; v < n; ++v) {
        if (assignment[v] != pid) continue;
        int64_t ext = 0;
        for (int64_t j = adj_ptr[v]; j < adj_ptr[v + 1]; ++j) ext += assignment[adj[j]] != pid;
        if (ext > best_ext) { best_v = v; best_ext = ext; }
      }
      int64_t target = -1;
      for (int64_t j = adj_ptr[best_v]; j < adj_ptr[best_v + 1]; ++j) {
        int64_t t = assignment[adj[j]];
        if (t == pid || sizes[t] >= capacity) continue;
        if (target < 0 || sizes[t] < sizes[target] || (sizes[t] == sizes[target] && t < target))
          target = t;
      }
      if (target < 0)
        for (int64_t p = 0; p < n_parts; ++p)
          if (sizes[p] < capacity && (target < 0 || sizes[p] < sizes[target])) target = p;
      assignment[best_v] = target;
      sizes[pid] -= 1;
      sizes[target] += 1;
    }
    return 0;
  }
  EHYB_CATCH
}

EHYB_API int ehyb_classify_rows(int64_t n, int64_t nnz, const int64_t* rows, const int64_t* cols,
                                const int64_t* assignment, int64_t n_parts, int64_t* inner,
                                int64_t* outer, int64_t* row_order, int64_t** out_er_row_order,
                                int64_t* out_n_er) {
  EHYB_TRY {
    std::vector<std::atomic<int64_t>> ic(static_cast<size_t>(n)), oc(static_cast<size_t>(n));
#pragma omp parallel for schedule(static) if (n > kParallelMin)
    for (int64_t i = 0; i < n; ++i) {
      ic[size_t(i)].store(0, std::memory_order_relaxed);
      oc[size_t(i)].store(0, std::memory_order_relaxed);
    }
#pragma omp parallel for schedule(static) if (nnz > kParallelMin)
    for (int64_t e = 0; e < nnz; ++e) {
      int64_t r = rows[e];
      if (assignment[r] == assignment[cols[e]])
        ic[size_t(r)].fetch_add(1, std::memory_order_relaxed);
      else
        oc[size_t(r)].fetch_add(1, std::memory_order_relaxed);
    }
#pragma omp parallel for schedule(static) if (n > kParallelMin)
    for (int64_t i = 0; i < n; ++i) {
      inner[i] = ic[size_t(i)].load(std::memory_order_relaxed);
      outer[i] = oc[size_t(i)].load(std::memory_order_relaxed);
    }
    // row_order = lexsort((rows, -inner, part)): partition-major, inner
    // descending, original row ascending. Stable bucket by part, then a
    // stable sort by -inner inside each part.
    std::vector<int64_t> pstart(size_t(n_parts) + 1, 0);
    for (int64_t i = 0; i < n; ++i) {
      int64_t p = assignment[i];
      if (p < 0 || p >= n_parts) return ehyb::fail("partition id out of range");
      pstart[size_t(p) + 1]++;
    }
    for (int64_t p = 0; p < n_parts; ++p) pstart[size_t(p) + 1] += pstart[size_t(p)];
    {
      std::vector<int64_t> fill(pstart.begin(), pstart.end() - 1);
      for (int64_t i = 0; i < n; ++i) row_order[fill[size_t(assignment[i])]++] = i;
    }
#pragma omp parallel for schedule(dynamic, 1) if (n > kParallelMin)
    for (int64_t p = 0; p < n_parts; ++p)
      std::stable_sort(row_order + pstart[size_t(p)], row_order + pstart[size_t(p) + 1],
                       [&](int64_t a, int64_t b) { return inner[a] > inner[b]; });
    // er_row_order: rows with outer > 0, outer descending then row ascending
    int64_t n_er = 0;
    for (int64_t i = 0; i < n; ++i) n_er += outer[i] > 0;
    int64_t* er = static_cast<int64_t*>(std::malloc(size_t(std::max<int64_t>(n_er, 1)) * 8));
    if (!er) return ehyb::fail_oom();
    int64_t j = 0;
    for (int64_t i = 0; i < n; ++i)
      if (outer[i] > 0) er[j++] = i;
    std::stable_sort(er, er + n_er, [&](int64_t a, int64_t b) { return outer[a] > outer[b]; });
    *out_er_row_order = er;
    *out_n_er = n_er;
    return 0;
  }
  EHYB_CATCH
}

EHYB_API int ehyb_build_reorder_plan(int64_t n, int64_t n_parts, int64_t vec,
                                     const int64_t* assignment, const int64_t* part_sizes,
                                     const int64_t* row_order, const int64_t* er_row_order,
                                     int64_t n_er, int64_t* reorder, int64_t* inverse,
                                     int64_t* arrange, int64_t* y_idx_er) {
  EHYB_TRY {
    int64_t maxsz = 0;
    for (int64_t p = 0; p < n_parts; ++p) maxsz = std::max(maxsz, part_sizes[p]);
    if (maxsz > vec) return ehyb::fail("a partition exceeds the vector cache capacity");
    const int64_t padded = n_parts * vec;
    // actual occupancy per part from the row order (row_order is part-major)
    std::vector<int64_t> occ(size_t(n_parts) + 1, 0);
    for (int64_t i = 0; i < n; ++i) occ[size_t(assignment[i]) + 1]++;
    for (int64_t p = 0; p < n_parts; ++p)
      if (occ[size_t(p) + 1] > vec) return ehyb::fail("a partition exceeds the vector cache capacity");
    std::vector<int64_t> start(size_t(n_parts) + 1, 0);
    for (int64_t p = 0; p < n_parts; ++p) start[size_t(p) + 1] = start[size_t(p)] + occ[size_t(p) + 1];
#pragma omp parallel for schedule(static) if (n > kParallelMin)
    for (int64_t i = 0; i < n; ++i) {
      int64_t r = row_order[i];
      int64_t p = assignment[r];
      reorder[r] = p * vec + (i - start[size_t(p)]);
    }
    // padding rows n..padded-1 take the free new ids in ascending order: the
    // tail [p*vec + occ_p, (p+1)*vec) of every part, parts ascending
    std::vector<int64_t> free_start(size_t(n_parts) + 1, 0);
    for (int64_t p = 0; p < n_parts; ++p)
      free_start[size_t(p) + 1] = free_start[size_t(p)] + (vec - occ[size_t(p) + 1]);
#pragma omp parallel for schedule(dynamic, 1) if (padded > kParallelMin)
    for (int64_t p = 0; p < n_parts; ++p) {
      int64_t k = n + free_start[size_t(p)];
      for (int64_t id = p * vec + occ[size_t(p) + 1]; id < (p + 1) * vec; ++id) reorder[k++] = id;
    }
#pragma omp parallel for schedule(static) if (padded > kParallelMin)
    for (int64_t i = 0; i < padded; ++i) inverse[reorder[i]] = i;
#pragma omp parallel for schedule(static) if (n > kParallelMin)
    for (int64_t i = 0; i < n; ++i) arrange[i] = -1;
#pragma omp parallel for schedule(static) if (n_er > kParallelMin)
    for (int64_t s = 0; s < n_er; ++s) {
      arrange[er_row_order[s]] = s;
      y_idx_er[s] = reorder[er_row_order[s]];
    }
    return 0;
  }
  EHYB_CATCH
}

EHYB_API int ehyb_assemble(int64_t n, int64_t nnz, const int64_t* rows, const int64_t* cols,
                           const double* values, const int64_t* assignment,
                           const int64_t* reorder, const int64_t* arrange, int64_t n_er,
                           int64_t warp, int64_t vec, int64_t n_parts, int32_t tau,
                           int32_t* position_ell, int32_t* width_ell, int32_t* ell_row_widths,
                           int32_t* part_boundary, int32_t* position_er, int32_t* width_er,
                           int32_t* er_row_widths, void** out_val_ell, uint16_t** out_col_ell,
                           int64_t* out_slots_ell, void** out_val_er, uint32_t** out_col_er,
                           int64_t* out_slots_er) {
  EHYB_TRY {
    if (tau != 4 && tau != 8) return ehyb::fail("tau must be 4 or 8");
    const int64_t padded = n_parts * vec;
    const int64_t n_sl = padded / warp;
    const int64_t n_er_sl = n_er ? cdiv(n_er, warp) : 0;
    std::vector<int64_t> rptr;
    std::unique_ptr<int32_t[]> scol;
    std::unique_ptr<double[]> sval;
    group_rows(n, nnz, rows, cols, values, rptr, scol, sval);
    // row widths
#pragma omp parallel for schedule(static) if (padded > kParallelMin)
    for (int64_t i = 0; i < padded; ++i) ell_row_widths[i] = 0;
#pragma omp parallel for schedule(static) if (n_er > kParallelMin)
    for (int64_t i = 0; i < n_er; ++i) er_row_widths[i] = 0;
#pragma omp parallel for schedule(dynamic, 1024) if (n > kParallelMin)
    for (int64_t r = 0; r < n; ++r) {
      int64_t ni = 0;
      for (int64_t j = rptr[size_t(r)]; j < rptr[size_t(r) + 1]; ++j)
        ni += assignment[scol[size_t(j)]] == assignment[r];
      ell_row_widths[reorder[r]] = int32_t(ni);
      if (arrange[r] >= 0) er_row_widths[arrange[r]] = int32_t(rptr[size_t(r) + 1] - rptr[size_t(r)] - ni);
    }
    // slice widths and int32 prefix positions (SELL-P)
#pragma omp parallel for schedule(static) if (n_sl > kParallelMin)
    for (int64_t s = 0; s < n_sl; ++s) {
      int32_t w = 0;
      for (int64_t l = 0; l < warp; ++l) w = std::max(w, ell_row_widths[s * warp + l]);
      width_ell[s] = w;
    }
    for (int64_t s = 0; s < n_er_sl; ++s) {
      int32_t w = 0;
      for (int64_t l = s * warp; l < std::min(n_er, (s + 1) * warp); ++l) w = std::max(w, er_row_widths[l]);
      width_er[s] = w;
    }
    int64_t acc = 0;
    position_ell[0] = 0;
    for (int64_t s = 0; s < n_sl; ++s) {
      acc += warp * int64_t(width_ell[s]);
      if (acc > INT32_MAX) return ehyb::fail("ELL slot count exceeds the int32 position range");
      position_ell[s + 1] = int32_t(acc);
    }
    const int64_t slots_ell = acc;
    acc = 0;
    position_er[0] = 0;
    for (int64_t s = 0; s < n_er_sl; ++s) {
      acc += warp * int64_t(width_er[s]);
      if (acc > INT32_MAX) return ehyb::fail("ER slot count exceeds the int32 position range");
      position_er[s + 1] = int32_t(acc);
    }
    const int64_t slots_er = acc;
    for (int64_t p = 0; p <= n_parts; ++p) part_boundary[p] = int32_t(p * vec);

    const size_t vb = size_t(tau);
    void* val_ell = std::calloc(size_t(std::max<int64_t>(slots_ell, 1)), vb);
    uint16_t* col_ell = static_cast<uint16_t*>(std::calloc(size_t(std::max<int64_t>(slots_ell, 1)), 2));
    void* val_er = std::calloc(size_t(std::max<int64_t>(slots_er, 1)), vb);
    uint32_t* col_er = static_cast<uint32_t*>(std::calloc(size_t(std::max<int64_t>(slots_er, 1)), 4));
    if (!val_ell || !col_ell || !val_er || !col_er) {
      std::free(val_ell); std::free(col_ell); std::free(val_er); std::free(col_er);
      return ehyb::fail_oom();
    }
    const int64_t lim = std::min<int64_t>(vec, EHYB_MAX_LOCAL_INDEX);
    std::atomic<int> bad{0};
#pragma omp parallel for schedule(dynamic, 1024) if (n > kParallelMin)
    for (int64_t r = 0; r < n; ++r) {
      const int64_t nr = reorder[r];
      const int64_t base = (nr / vec) * vec;
      const int64_t slot = arrange[r];
      int64_t ki = 0, ko = 0;
      for (int64_t j = rptr[size_t(r)]; j < rptr[size_t(r) + 1]; ++j) {
        const int64_t c = scol[size_t(j)];
        const double x = sval[size_t(j)];
        int64_t d;
        if (assignment[c] == assignment[r]) {
          const int64_t loc = reorder[c] - base;
          if (loc < 0 || loc >= lim) { bad.store(1); continue; }
          d = position_ell[nr / warp] + nr % warp + ki * warp;
          ++ki;
          col_ell[d] = uint16_t(loc);
          if (tau == 4) static_cast<float*>(val_ell)[d] = float(x);
          else static_cast<double*>(val_ell)[d] = x;
        } else {
          if (slot < 0) { bad.store(2); continue; }
          d = position_er[slot / warp] + slot % warp + ko * warp;
          ++ko;
          col_er[d] = uint32_t(reorder[c]);
          if (tau == 4) static_cast<float*>(val_er)[d] = float(x);
          else static_cast<double*>(val_er)[d] = x;
        }
      }
    }
    if (bad.load()) {
      std::free(val_ell); std::free(col_ell); std::free(val_er); std::free(col_er);
      return ehyb::fail(bad.load() == 1 ? "inner entry maps outside its partition cache window"
                                        : "outer entry in a row missing from the ER arrangement");
    }
    *out_val_ell = val_ell;
    *out_col_ell = col_ell;
    *out_slots_ell = slots_ell;
    *out_val_er = val_er;
    *out_col_er = col_er;
    *out_slots_er = slots_er;
    return 0;
  }
  EHYB_CATCH
}

// format.py:250-299 structural invariants, O(size) (the permutation test is a
// visit-once bitmap instead of a sort). Messages are the reference's.
EHYB_API int ehyb_check(const ehyb_host_matrix* m) {
  EHYB_TRY {
    const int64_t warp = m->warp_size, vec = m->vec_cache_size, n_parts = m->n_parts;
    const int64_t padded = m->padded_dimension;
    if (padded != n_parts * vec) return ehyb::fail("padded_dimension must equal n_parts * vec_cache_size");
    if (m->plan_padded_dimension != padded) return ehyb::fail("plan and matrix disagree on padded_dimension");
    const int64_t n_sl = padded / warp;
    if (m->n_width_ell != n_sl || m->n_position_ell != n_sl + 1)
      return ehyb::fail("bad ELL slice metadata length");
    for (int64_t s = 0; s < n_sl; ++s)
      if (int64_t(m->position_ell[s + 1]) - m->position_ell[s] != warp * int64_t(m->width_ell[s]))
        return ehyb::fail("position_ell deltas must equal warp_size * width_ell");
    if (m->slots_ell != (n_sl ? int64_t(m->position_ell[n_sl]) : 0))
      return ehyb::fail("val_ell length inconsistent with position_ell");
    if (m->n_col_ell != m->slots_ell) return ehyb::fail("col_ell and val_ell must have equal length");
    for (int64_t i = 0; i < m->n_col_ell; ++i)
      if (int64_t(m->col_ell[i]) >= vec) return ehyb::fail("col_ell offset outside the cache window");
    if (m->n_part_boundary != n_parts + 1) return ehyb::fail("part_boundary must step by vec_cache_size");
    for (int64_t p = 0; p <= n_parts; ++p)
      if (int64_t(m->part_boundary[p]) != p * vec) return ehyb::fail("part_boundary must step by vec_cache_size");
    if (m->n_ell_row_widths != padded) return ehyb::fail("ell_row_widths must cover every padded row");
    if (m->n_reorder != padded || m->n_inverse != padded) return ehyb::fail("reorder_table is not a permutation");
    {
      std::vector<uint8_t> seen(size_t(padded), 0);
      for (int64_t i = 0; i < padded; ++i) {
        int64_t v = m->reorder[i];
        if (v < 0 || v >= padded || seen[size_t(v)]) return ehyb::fail("reorder_table is not a permutation");
        seen[size_t(v)] = 1;
      }
      for (int64_t i = 0; i < padded; ++i)
        if (m->inverse[m->reorder[i]] != i) return ehyb::fail("inverse_table does not invert reorder_table");
    }
    const int64_t n_er = m->n_er_rows;
    const int64_t n_er_sl = m->n_width_er;
    if (m->n_position_er != n_er_sl + 1) return ehyb::fail("bad ER slice metadata length");
    if (n_er_sl != (n_er ? cdiv(n_er, warp) : 0)) return ehyb::fail("ER slice count inconsistent with n_er_rows");
    for (int64_t s = 0; s < n_er_sl; ++s)
      if (int64_t(m->position_er[s + 1]) - m->position_er[s] != warp * int64_t(m->width_er[s]))
        return ehyb::fail("position_er deltas must equal warp_size * width_er");
    if (m->slots_er != (m->n_position_er ? int64_t(m->position_er[m->n_position_er - 1]) : 0))
      return ehyb::fail("val_er length inconsistent with position_er");
    if (m->n_col_er != m->slots_er) return ehyb::fail("col_er and val_er must have equal length");
    if (m->n_er_row_widths != n_er || m->n_y_idx_er != n_er)
      return ehyb::fail("ER per-row metadata must have n_er_rows entries");
    for (int64_t i = 0; i < n_er; ++i)
      if (m->y_idx_er[i] >= padded) return ehyb::fail("y_idx_er points outside the padded row space");
    return 0;
  }
  EHYB_CATCH
}

EHYB_API void ehyb_free(void* p) { std::free(p); }

EHYB_API int ehyb_num_threads(void) { return omp_get_max_threads(); }

}  // extern "C"
