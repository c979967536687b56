/*
 * ORACLE — test / CPU-baseline infrastructure only. NOT part of the product.
 *
 * Plain-C restatement of the reference simulated engine `spmv_ehyb`
 * (/root/reference/pkg/src/ehyb/engine.py:108-216): phase 1 runs every
 * partition's ELL slices against its cached x window (run_block, 134-144),
 * a barrier, then phase 2 runs the ER slices on uncached x and accumulates
 * into y[y_idx_er] (run_er_slice, 146-154). Partitions / ER slices are dealt
 * to OpenMP threads like the reference's "static" worker sweep (163-177);
 * each output row gets exactly one phase-1 write and at most one phase-2
 * add, so the result is bit-identical for every thread count. Arithmetic is
 * the reference's: accumulator from +0.0, separately rounded multiply and
 * add per slot (compiled with -ffp-contract=off), padding slots included.
 *
 * [part_lo, part_hi) / [er_lo, er_hi) bound the work to a sample of the
 * partitions and ER slices (full product: 0..n_parts, 0..n_er_slices).
 *
 * Used by tests/ (parity), bench.py's cpu_baseline leg and
 * `bench.py --impl reference`. Pinned by tests/test_oracle_c.py against the
 * reference's own y digests (tests/golden/config_*.json, small_cases.npz).
 */
#include <stdint.h>
#include <string.h>

#include <omp.h>

#define DEFINE_SPMV(NAME, T)                                                                    \
  int NAME(int64_t n_parts, int64_t vec, int64_t warp, const T* val_ell, const uint16_t* col_ell, \
           const int32_t* position_ell, const int32_t* width_ell, int64_t n_er,                 \
           const T* val_er, const uint32_t* col_er, const int32_t* position_er,                 \
           const int32_t* width_er, const int64_t* y_idx_er, const T* x, T* y, int threads,   \
           int64_t part_lo, int64_t part_hi, int64_t er_lo, int64_t er_hi) {                    \
    const int64_t padded = n_parts * vec;                                                       \
    const int64_t slices_per_block = vec / warp;                                                \
    const int64_t n_er_slices = n_er ? (n_er + warp - 1) / warp : 0;                            \
    if (threads < 1) threads = 1;                                                               \
    if (part_hi > n_parts) part_hi = n_parts;                                                   \
    if (er_hi > n_er_slices) er_hi = n_er_slices;                                               \
    memset(y, 0, (size_t)padded * sizeof(T));                                                   \
    /* phase 1: run_block per partition */                                                      \
    _Pragma("omp parallel for schedule(static, 1) num_threads(threads)")                       \
    for (int64_t b = part_lo; b < part_hi; ++b) {                                               \
      const T* cache = x + b * vec;                                                             \
      T acc[32];                                                                                \
      for (int64_t s = b * slices_per_block; s < (b + 1) * slices_per_block; ++s) {           \
        const int64_t pos = position_ell[s];                                                    \
        for (int64_t l = 0; l < warp; ++l) acc[l] = (T)0;                                       \
        for (int64_t k = 0; k < width_ell[s]; ++k) {                                            \
          const int64_t seg = pos + k * warp;                                                   \
          for (int64_t l = 0; l < warp; ++l) {                                                  \
            T prod = val_ell[seg + l] * cache[col_ell[seg + l]];                                \
            acc[l] = acc[l] + prod;                                                             \
          }                                                                                     \
        }                                                                                       \
        for (int64_t l = 0; l < warp; ++l) y[s * warp + l] = acc[l];                           \
      }                                                                                         \
    }                                                                                           \
    /* barrier (end of the parallel region), then phase 2: run_er_slice */                     \
    _Pragma("omp parallel for schedule(static, 1) num_threads(threads)")                       \
    for (int64_t j = er_lo; j < er_hi; ++j) {                                                   \
      T acc[32];                                                                                \
      const int64_t pos = position_er[j];                                                       \
      for (int64_t l = 0; l < warp; ++l) acc[l] = (T)0;                                         \
      for (int64_t k = 0; k < width_er[j]; ++k) {                                               \
        const int64_t seg = pos + k * warp;                                                     \
        for (int64_t l = 0; l < warp; ++l) {                                                    \
          T prod = val_er[seg + l] * x[col_er[seg + l]];                                        \
          acc[l] = acc[l] + prod;                                                               \
        }                                                                                       \
      }                                                                                         \
      int64_t lanes = n_er - j * warp;                                                          \
      if (lanes > warp) lanes = warp;                                                           \
      for (int64_t l = 0; l < lanes; ++l) {                                                     \
        const int64_t r = y_idx_er[j * warp + l];                                               \
        y[r] = y[r] + acc[l];                                                                   \
      }                                                                                         \
    }                                                                                           \
    return 0;                                                                                   \
  }

/* slice height is at most 32 on every profile the reference tests use
 * (warp 1/4/8/32); larger heights are rejected by the Python wrapper */
DEFINE_SPMV(oracle_spmv_ehyb_f64, double)
DEFINE_SPMV(oracle_spmv_ehyb_f32, float)

int oracle_max_threads(void) { return omp_get_max_threads(); }
