/*
 * ORACLE — test / CPU-baseline infrastructure only. NOT part of the product.
 *
 * Plain-C restatement of the reference preprocessing pipeline, so the
 * reference arm of bench.py (and the tests) can build EHYB arrays without
 * the product library:
 *
 *   oracle_build_graph      partition.py:77-98   symmetrized off-diagonal
 *                                                adjacency, neighbours sorted
 *                                                ascending, duplicates removed
 *   oracle_partition_graph  partition.py:101-204 BFS region growing seeded at
 *                                                the min-degree unassigned
 *                                                vertex (CPython MT19937
 *                                                randrange among ties), fill,
 *                                                round-robin isolated vertices,
 *                                                one refinement pass
 *   oracle_assemble         format.py:123-137 (classify_rows),
 *                           format.py:161-199 (build_reorder_plan),
 *                           format.py:302-409 (assemble_ehyb)
 *
 * Written from the reference's Python semantics (SURVEY.md 8a gotchas 1-8),
 * serial except for the embarrassingly parallel per-row sorts; pinned by
 * tests/test_oracle_c.py against the digests the reference itself produced
 * (tests/golden/). Outputs are allocated here and released with oracle_free.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include <omp.h>

void oracle_free(void* p) { free(p); }

/* ------------------------------------------------------------ utilities */
static int cmp_i32(const void* a, const void* b) {
  const int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
  return (x > y) - (x < y);
}

typedef struct {
  int64_t key, idx;
} kv64;
static int cmp_kv64(const void* a, const void* b) {
  const kv64* x = (const kv64*)a;
  const kv64* y = (const kv64*)b;
  if (x->key != y->key) return (x->key > y->key) - (x->key < y->key);
  return (x->idx > y->idx) - (x->idx < y->idx);
}

/* ------------------------------------------------- build_graph (77-98) */
/* Returns the number of adjacency entries; *adj_out is malloc'd (int32). */
int64_t oracle_build_graph(int64_t n, int64_t nnz, const int64_t* rows, const int64_t* cols,
                           int64_t* adj_ptr, int32_t** adj_out) {
  int64_t* cnt = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
  for (int64_t e = 0; e < nnz; ++e)
    if (rows[e] != cols[e]) {
      cnt[rows[e] + 1]++;
      cnt[cols[e] + 1]++;
    }
  for (int64_t i = 0; i < n; ++i) cnt[i + 1] += cnt[i];
  const int64_t total = cnt[n];
  int32_t* tmp = (int32_t*)malloc((size_t)(total > 0 ? total : 1) * sizeof(int32_t));
  int64_t* fill = (int64_t*)malloc((size_t)(n > 0 ? n : 1) * sizeof(int64_t));
  memcpy(fill, cnt, (size_t)n * sizeof(int64_t));
  for (int64_t e = 0; e < nnz; ++e)
    if (rows[e] != cols[e]) {
      tmp[fill[rows[e]]++] = (int32_t)cols[e];
      tmp[fill[cols[e]]++] = (int32_t)rows[e];
    }
  /* per vertex: sort ascending, drop duplicates (np.unique of src*n+dst) */
  int64_t* uniq = fill;
#pragma omp parallel for schedule(dynamic, 1024)
  for (int64_t v = 0; v < n; ++v) {
    int32_t* seg = tmp + cnt[v];
    const int64_t len = cnt[v + 1] - cnt[v];
    if (len > 1) qsort(seg, (size_t)len, sizeof(int32_t), cmp_i32);
    int64_t u = 0;
    for (int64_t i = 0; i < len; ++i)
      if (i == 0 || seg[i] != seg[i - 1]) seg[u++] = seg[i];
    uniq[v] = u;
  }
  adj_ptr[0] = 0;
  for (int64_t v = 0; v < n; ++v) adj_ptr[v + 1] = adj_ptr[v] + uniq[v];
  int32_t* adj = (int32_t*)malloc((size_t)(adj_ptr[n] > 0 ? adj_ptr[n] : 1) * sizeof(int32_t));
#pragma omp parallel for schedule(static)
  for (int64_t v = 0; v < n; ++v)
    memcpy(adj + adj_ptr[v], tmp + cnt[v], (size_t)uniq[v] * sizeof(int32_t));
  free(tmp);
  free(fill);
  free(cnt);
  *adj_out = adj;
  return adj_ptr[n];
}

/* ------------------------------------- CPython random.Random (MT19937) */
typedef struct {
  uint32_t mt[624];
  int mti;
} mt_state;

static void mt_init_genrand(mt_state* s, uint32_t seed) {
  s->mt[0] = seed;
  for (int i = 1; i < 624; i++)
    s->mt[i] = 1812433253u * (s->mt[i - 1] ^ (s->mt[i - 1] >> 30)) + (uint32_t)i;
  s->mti = 624;
}

static void mt_init_by_array(mt_state* s, const uint32_t* key, int len) {
  mt_init_genrand(s, 19650218u);
  int i = 1, j = 0;
  for (int k = 624 > len ? 624 : len; k; k--) {
    s->mt[i] = (s->mt[i] ^ ((s->mt[i - 1] ^ (s->mt[i - 1] >> 30)) * 1664525u)) + key[j] + (uint32_t)j;
    i++;
    j++;
    if (i >= 624) {
      s->mt[0] = s->mt[623];
      i = 1;
    }
    if (j >= len) j = 0;
  }
  for (int k = 623; k; k--) {
    s->mt[i] = (s->mt[i] ^ ((s->mt[i - 1] ^ (s->mt[i - 1] >> 30)) * 1566083941u)) - (uint32_t)i;
    i++;
    if (i >= 624) {
      s->mt[0] = s->mt[623];
      i = 1;
    }
  }
  s->mt[0] = 0x80000000u;
}

static uint32_t mt_next(mt_state* s) {
  static const uint32_t mag01[2] = {0u, 0x9908b0dfu};
  uint32_t y;
  if (s->mti >= 624) {
    int kk;
    for (kk = 0; kk < 624 - 397; kk++) {
      y = (s->mt[kk] & 0x80000000u) | (s->mt[kk + 1] & 0x7fffffffu);
      s->mt[kk] = s->mt[kk + 397] ^ (y >> 1) ^ mag01[y & 1u];
    }
    for (; kk < 623; kk++) {
      y = (s->mt[kk] & 0x80000000u) | (s->mt[kk + 1] & 0x7fffffffu);
      s->mt[kk] = s->mt[kk + (397 - 624)] ^ (y >> 1) ^ mag01[y & 1u];
    }
    y = (s->mt[623] & 0x80000000u) | (s->mt[0] & 0x7fffffffu);
    s->mt[623] = s->mt[396] ^ (y >> 1) ^ mag01[y & 1u];
    s->mti = 0;
  }
  y = s->mt[s->mti++];
  y ^= (y >> 11);
  y ^= (y << 7) & 0x9d2c5680u;
  y ^= (y << 15) & 0xefc60000u;
  y ^= (y >> 18);
  return y;
}

/* random.Random(seed): init_by_array over the 32-bit words of |seed| */
static void mt_seed(mt_state* s, int64_t seed) {
  uint64_t a = seed < 0 ? (uint64_t)(-seed) : (uint64_t)seed;
  uint32_t key[2];
  int len = 0;
  do {
    key[len++] = (uint32_t)(a & 0xffffffffu);
    a >>= 32;
  } while (a && len < 2);
  mt_init_by_array(s, key, len);
}

/* randrange(m) = _randbelow_with_getrandbits(m), m < 2^32 */
static int64_t mt_randbelow(mt_state* s, int64_t m) {
  int k = 0;
  while ((((int64_t)1) << k) <= m) ++k; /* m.bit_length() */
  for (;;) {
    const int64_t r = (int64_t)(mt_next(s) >> (32 - k));
    if (r < m) return r;
  }
}

/* ------------------------------------------------------ Fenwick tree */
typedef struct {
  int64_t n;
  int64_t* t;
} fenwick;

static void fw_add(fenwick* f, int64_t i, int64_t d) {
  for (++i; i <= f->n; i += i & -i) f->t[i] += d;
}
static int64_t fw_prefix(const fenwick* f, int64_t i) { /* sum of [0, i) */
  int64_t s = 0;
  for (; i > 0; i -= i & -i) s += f->t[i];
  return s;
}
static int64_t fw_find(const fenwick* f, int64_t k) { /* smallest i with prefix(i+1) >= k */
  int64_t pos = 0, step = 1;
  while (step * 2 <= f->n) step *= 2;
  for (; step; step >>= 1)
    if (pos + step <= f->n && f->t[pos + step] < k) {
      pos += step;
      k -= f->t[pos];
    }
  return pos;
}

/* -------------------------------------------- partition_graph (101-204) */
int oracle_partition_graph(int64_t n, const int64_t* adj_ptr, const int32_t* adj, int64_t n_parts,
                           int64_t capacity, int64_t seed, int64_t* assignment, int64_t* sizes) {
  if (n_parts < 1 || capacity < 1 || n_parts * capacity < n) return 1;
  mt_state rng;
  mt_seed(&rng, seed);
  for (int64_t v = 0; v < n; ++v) assignment[v] = -1;
  memset(sizes, 0, (size_t)n_parts * sizeof(int64_t));

  /* by_degree: connected vertices, stable argsort by degree */
  int64_t maxdeg = 0;
  for (int64_t v = 0; v < n; ++v) {
    const int64_t d = adj_ptr[v + 1] - adj_ptr[v];
    if (d > maxdeg) maxdeg = d;
  }
  int64_t* dcnt = (int64_t*)calloc((size_t)maxdeg + 2, sizeof(int64_t));
  for (int64_t v = 0; v < n; ++v) dcnt[adj_ptr[v + 1] - adj_ptr[v] + 1]++;
  for (int64_t d = 0; d <= maxdeg; ++d) dcnt[d + 1] += dcnt[d];
  const int64_t n_iso = dcnt[1];
  const int64_t m = n - n_iso;
  int64_t* by_degree = (int64_t*)malloc((size_t)(m > 0 ? m : 1) * sizeof(int64_t));
  int64_t* pos_of = (int64_t*)malloc((size_t)(n > 0 ? n : 1) * sizeof(int64_t));
  int64_t* grp_end = (int64_t*)malloc((size_t)(m > 0 ? m : 1) * sizeof(int64_t));
  for (int64_t v = 0; v < n; ++v) {
    const int64_t d = adj_ptr[v + 1] - adj_ptr[v];
    if (d == 0) continue;
    const int64_t p = dcnt[d]++ - n_iso;
    by_degree[p] = v;
    pos_of[v] = p;
  }
  for (int64_t p = m - 1; p >= 0; --p) {
    const int64_t d = adj_ptr[by_degree[p] + 1] - adj_ptr[by_degree[p]];
    const int same = p + 1 < m &&
                     adj_ptr[by_degree[p + 1] + 1] - adj_ptr[by_degree[p + 1]] == d;
    grp_end[p] = same ? grp_end[p + 1] : p + 1;
  }
  free(dcnt);
  fenwick fw = {m, (int64_t*)calloc((size_t)m + 1, sizeof(int64_t))};
  for (int64_t p = 0; p < m; ++p) fw_add(&fw, p, 1); /* 1 = unassigned */

  int64_t cursor = 0;
  int64_t* queue = (int64_t*)malloc((size_t)(n > 0 ? n : 1) * sizeof(int64_t));

#define ASSIGN(v, pid)                                          \
  do {                                                          \
    assignment[(v)] = (pid);                                    \
    sizes[(pid)] += 1;                                          \
    if (adj_ptr[(v) + 1] > adj_ptr[(v)]) fw_add(&fw, pos_of[(v)], -1); \
  } while (0)

  int64_t left = m;
  int64_t pid_first = 0;
  for (int64_t step = 0;; ++step) {
    int64_t pid;
    if (pid_first < n_parts) {
      if (left == 0) break;
      pid = pid_first++;
    } else {
      if (left <= 0) break;
      pid = -1;
      for (int64_t q = 0; q < n_parts; ++q)
        if (sizes[q] < capacity && (pid < 0 || sizes[q] < sizes[pid])) pid = q;
      if (pid < 0) break;
    }
    /* next_seed */
    while (cursor < m && assignment[by_degree[cursor]] >= 0) ++cursor;
    if (cursor >= m) continue; /* grow() returns 0 */
    const int64_t run_n = fw_prefix(&fw, grp_end[cursor]) - fw_prefix(&fw, cursor);
    int64_t start;
    if (run_n > 1) {
      const int64_t pick = mt_randbelow(&rng, run_n);
      start = by_degree[fw_find(&fw, fw_prefix(&fw, cursor) + pick + 1)];
    } else {
      start = by_degree[cursor];
    }
    /* grow: BFS, vertices assigned on enqueue, neighbours ascending */
    int64_t grown = 1, qh = 0, qt = 0;
    ASSIGN(start, pid);
    queue[qt++] = start;
    while (qh < qt && sizes[pid] < capacity) {
      const int64_t u = queue[qh++];
      for (int64_t k = adj_ptr[u]; k < adj_ptr[u + 1]; ++k) {
        const int64_t w = adj[k];
        if (assignment[w] < 0) {
          ASSIGN(w, pid);
          grown++;
          queue[qt++] = w;
          if (sizes[pid] == capacity) break;
        }
      }
    }
    left -= grown;
  }
#undef ASSIGN
  /* isolated vertices, round-robin over non-full parts */
  {
    int64_t pid = 0;
    for (int64_t v = 0; v < n; ++v) {
      if (adj_ptr[v + 1] > adj_ptr[v]) continue;
      while (sizes[pid] >= capacity) pid = (pid + 1) % n_parts;
      assignment[v] = pid;
      sizes[pid] += 1;
      pid = (pid + 1) % n_parts;
    }
  }
  /* one refinement pass in vertex order, sizes updated live */
  {
    int64_t* cnt = (int64_t*)calloc((size_t)n_parts, sizeof(int64_t));
    int64_t* touched = (int64_t*)malloc((size_t)(maxdeg > 0 ? maxdeg : 1) * sizeof(int64_t));
    for (int64_t v = 0; v < n; ++v) {
      const int64_t lo = adj_ptr[v], hi = adj_ptr[v + 1];
      if (hi == lo) continue;
      const int64_t a = assignment[v];
      int64_t nt = 0;
      for (int64_t k = lo; k < hi; ++k) {
        const int64_t p = assignment[adj[k]];
        if (cnt[p]++ == 0) touched[nt++] = p;
      }
      const int64_t internal = cnt[a];
      int64_t b = -1, best = -1;
      for (int64_t t = 0; t < nt; ++t) {
        const int64_t p = touched[t];
        if (p == a || sizes[p] >= capacity) continue;
        if (cnt[p] > best || (cnt[p] == best && p < b)) {
          best = cnt[p];
          b = p;
        }
      }
      for (int64_t t = 0; t < nt; ++t) cnt[touched[t]] = 0;
      if (b >= 0 && best > internal) {
        assignment[v] = b;
        sizes[a] -= 1;
        sizes[b] += 1;
      }
    }
    free(cnt);
    free(touched);
  }
  free(queue);
  free(fw.t);
  free(grp_end);
  free(pos_of);
  free(by_degree);
  return 0;
}

/* ------------------------- classify_rows + build_reorder_plan + assemble */
typedef struct {
  int64_t n, padded, n_parts, vec, warp, tau, n_er, slots_ell, slots_er;
  int64_t *inner_counts, *outer_counts, *row_order, *er_row_order;  /* classify */
  int64_t *reorder, *inverse, *arrange, *y_idx_er;                  /* plan */
  int32_t *ell_row_widths, *width_ell, *position_ell, *part_boundary;
  int32_t *er_row_widths, *width_er, *position_er;
  void* val_ell;
  uint16_t* col_ell;
  void* val_er;
  uint32_t* col_er;
} oracle_ehyb;

void oracle_ehyb_free(oracle_ehyb* o) {
  void* ps[] = {o->inner_counts, o->outer_counts, o->row_order, o->er_row_order, o->reorder,
                o->inverse, o->arrange, o->y_idx_er, o->ell_row_widths, o->width_ell,
                o->position_ell, o->part_boundary, o->er_row_widths, o->width_er,
                o->position_er, o->val_ell, o->col_ell, o->val_er, o->col_er};
  for (size_t i = 0; i < sizeof(ps) / sizeof(ps[0]); ++i) free(ps[i]);
  memset(o, 0, sizeof(*o));
}

static const int64_t* g_key1; /* qsort context (single-threaded uses only) */
static const int64_t* g_key2;
static int cmp_rows_inner(const void* a, const void* b) { /* -inner, then row */
  const int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
  if (g_key1[x] != g_key1[y]) return g_key1[x] > g_key1[y] ? -1 : 1;
  return (x > y) - (x < y);
}

/* returns 0, or 1 = a part exceeds vec, 2 = local index out of range,
 * 3 = int32 position overflow */
int oracle_assemble(int64_t n, int64_t nnz, const int64_t* rows, const int64_t* cols,
                    const double* vals, const int64_t* assignment, int64_t n_parts, int64_t vec,
                    int64_t warp, int64_t tau, oracle_ehyb* o) {
  memset(o, 0, sizeof(*o));
  const int64_t padded = n_parts * vec;
  o->n = n;
  o->padded = padded;
  o->n_parts = n_parts;
  o->vec = vec;
  o->warp = warp;
  o->tau = tau;
  /* ---- classify_rows (123-137) */
  int64_t* inner = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
  int64_t* outer = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
  for (int64_t e = 0; e < nnz; ++e) {
    if (assignment[rows[e]] == assignment[cols[e]]) inner[rows[e]]++;
    else outer[rows[e]]++;
  }
  /* row_order = lexsort((rows, -inner, part)) */
  int64_t* pstart = (int64_t*)calloc((size_t)n_parts + 1, sizeof(int64_t));
  for (int64_t r = 0; r < n; ++r) pstart[assignment[r] + 1]++;
  for (int64_t p = 0; p < n_parts; ++p) {
    if (pstart[p + 1] > vec) {
      free(inner);
      free(outer);
      free(pstart);
      return 1; /* "capacity" */
    }
    pstart[p + 1] += pstart[p];
  }
  int64_t* row_order = (int64_t*)malloc((size_t)(n > 0 ? n : 1) * sizeof(int64_t));
  {
    int64_t* f = (int64_t*)malloc((size_t)(n_parts + 1) * sizeof(int64_t));
    memcpy(f, pstart, (size_t)n_parts * sizeof(int64_t));
    for (int64_t r = 0; r < n; ++r) row_order[f[assignment[r]]++] = r;
    free(f);
    g_key1 = inner;
    for (int64_t p = 0; p < n_parts; ++p)
      qsort(row_order + pstart[p], (size_t)(pstart[p + 1] - pstart[p]), sizeof(int64_t),
            cmp_rows_inner);
  }
  /* er_row_order: rows with outer > 0, outer descending, then row */
  int64_t n_er = 0;
  for (int64_t r = 0; r < n; ++r) n_er += outer[r] > 0;
  int64_t* er_order = (int64_t*)malloc((size_t)(n_er > 0 ? n_er : 1) * sizeof(int64_t));
  {
    int64_t k = 0;
    for (int64_t r = 0; r < n; ++r)
      if (outer[r] > 0) er_order[k++] = r;
    g_key1 = outer;
    qsort(er_order, (size_t)n_er, sizeof(int64_t), cmp_rows_inner);
  }
  o->inner_counts = inner;
  o->outer_counts = outer;
  o->row_order = row_order;
  o->er_row_order = er_order;
  o->n_er = n_er;

  /* ---- build_reorder_plan (161-199) */
  int64_t* reorder = (int64_t*)malloc((size_t)(padded > 0 ? padded : 1) * sizeof(int64_t));
  int64_t* inverse = (int64_t*)malloc((size_t)(padded > 0 ? padded : 1) * sizeof(int64_t));
  unsigned char* taken = (unsigned char*)calloc((size_t)padded + 1, 1);
  for (int64_t p = 0; p < n_parts; ++p)
    for (int64_t i = pstart[p]; i < pstart[p + 1]; ++i) {
      const int64_t nr = p * vec + (i - pstart[p]);
      reorder[row_order[i]] = nr;
      taken[nr] = 1;
    }
  {
    int64_t k = n;
    for (int64_t i = 0; i < padded; ++i)
      if (!taken[i]) reorder[k++] = i;
  }
  free(taken);
  free(pstart);
  for (int64_t i = 0; i < padded; ++i) inverse[reorder[i]] = i;
  int64_t* arrange = (int64_t*)malloc((size_t)(n > 0 ? n : 1) * sizeof(int64_t));
  int64_t* y_idx_er = (int64_t*)malloc((size_t)(n_er > 0 ? n_er : 1) * sizeof(int64_t));
  for (int64_t r = 0; r < n; ++r) arrange[r] = -1;
  for (int64_t k = 0; k < n_er; ++k) {
    arrange[er_order[k]] = k;
    y_idx_er[k] = reorder[er_order[k]];
  }
  o->reorder = reorder;
  o->inverse = inverse;
  o->arrange = arrange;
  o->y_idx_er = y_idx_er;

  /* ---- assemble_ehyb (302-409): entries by (row, original col), stable */
  int64_t* rs = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
  for (int64_t e = 0; e < nnz; ++e) rs[rows[e] + 1]++;
  for (int64_t r = 0; r < n; ++r) rs[r + 1] += rs[r];
  kv64* ent = (kv64*)malloc((size_t)(nnz > 0 ? nnz : 1) * sizeof(kv64));
  {
    int64_t* f = (int64_t*)malloc((size_t)(n > 0 ? n : 1) * sizeof(int64_t));
    memcpy(f, rs, (size_t)n * sizeof(int64_t));
    for (int64_t e = 0; e < nnz; ++e) {
      kv64 x = {cols[e], e};
      ent[f[rows[e]]++] = x;
    }
    free(f);
  }
#pragma omp parallel for schedule(dynamic, 1024)
  for (int64_t r = 0; r < n; ++r)
    if (rs[r + 1] - rs[r] > 1) qsort(ent + rs[r], (size_t)(rs[r + 1] - rs[r]), sizeof(kv64), cmp_kv64);

  const int64_t n_slices = padded / warp;
  int32_t* ell_w = (int32_t*)calloc((size_t)padded + 1, sizeof(int32_t));
  for (int64_t r = 0; r < n; ++r) ell_w[reorder[r]] = (int32_t)inner[r];
  int32_t* width_ell = (int32_t*)calloc((size_t)n_slices + 1, sizeof(int32_t));
  int32_t* pos_ell = (int32_t*)calloc((size_t)n_slices + 1, sizeof(int32_t));
  int64_t acc = 0;
  for (int64_t s = 0; s < n_slices; ++s) {
    int32_t w = 0;
    for (int64_t l = 0; l < warp; ++l)
      if (ell_w[s * warp + l] > w) w = ell_w[s * warp + l];
    width_ell[s] = w;
    acc += warp * (int64_t)w;
    if (acc >= ((int64_t)1 << 31)) return 3;
    pos_ell[s + 1] = (int32_t)acc;
  }
  const int64_t slots_ell = acc;
  int32_t* pb = (int32_t*)malloc((size_t)(n_parts + 1) * sizeof(int32_t));
  for (int64_t p = 0; p <= n_parts; ++p) pb[p] = (int32_t)(p * vec);

  int32_t* er_w = (int32_t*)calloc((size_t)n_er + 1, sizeof(int32_t));
  for (int64_t k = 0; k < n_er; ++k) er_w[k] = (int32_t)outer[er_order[k]];
  const int64_t n_er_slices = n_er ? (n_er + warp - 1) / warp : 0;
  int32_t* width_er = (int32_t*)calloc((size_t)n_er_slices + 1, sizeof(int32_t));
  int32_t* pos_er = (int32_t*)calloc((size_t)n_er_slices + 1, sizeof(int32_t));
  acc = 0;
  for (int64_t s = 0; s < n_er_slices; ++s) {
    int32_t w = 0;
    for (int64_t l = 0; l < warp && s * warp + l < n_er; ++l)
      if (er_w[s * warp + l] > w) w = er_w[s * warp + l];
    width_er[s] = w;
    acc += warp * (int64_t)w;
    if (acc >= ((int64_t)1 << 31)) return 3;
    pos_er[s + 1] = (int32_t)acc;
  }
  const int64_t slots_er = acc;
  const size_t tb = (size_t)tau;
  void* val_ell = calloc((size_t)(slots_ell > 0 ? slots_ell : 1), tb);
  uint16_t* col_ell = (uint16_t*)calloc((size_t)(slots_ell > 0 ? slots_ell : 1), 2);
  void* val_er = calloc((size_t)(slots_er > 0 ? slots_er : 1), tb);
  uint32_t* col_er = (uint32_t*)calloc((size_t)(slots_er > 0 ? slots_er : 1), 4);
  int bad_local = 0;
  for (int64_t r = 0; r < n; ++r) {
    const int64_t nr = reorder[r];
    const int64_t slot = arrange[r];
    int64_t ki = 0, ko = 0;
    for (int64_t i = rs[r]; i < rs[r + 1]; ++i) {
      const int64_t c = ent[i].key;
      const double v = vals[ent[i].idx];
      int64_t dest;
      if (assignment[r] == assignment[c]) {
        const int64_t local = reorder[c] - (nr / vec) * vec;
        if (local < 0 || local >= vec || local >= 65536) bad_local = 1;
        dest = pos_ell[nr / warp] + nr % warp + ki * warp;
        ki++;
        if (tau == 4) ((float*)val_ell)[dest] = (float)v;
        else ((double*)val_ell)[dest] = v;
        col_ell[dest] = (uint16_t)local;
      } else {
        dest = pos_er[slot / warp] + slot % warp + ko * warp;
        ko++;
        if (tau == 4) ((float*)val_er)[dest] = (float)v;
        else ((double*)val_er)[dest] = v;
        col_er[dest] = (uint32_t)reorder[c];
      }
    }
  }
  free(ent);
  free(rs);
  o->ell_row_widths = ell_w;
  o->width_ell = width_ell;
  o->position_ell = pos_ell;
  o->part_boundary = pb;
  o->er_row_widths = er_w;
  o->width_er = width_er;
  o->position_er = pos_er;
  o->val_ell = val_ell;
  o->col_ell = col_ell;
  o->val_er = val_er;
  o->col_er = col_er;
  o->slots_ell = slots_ell;
  o->slots_er = slots_er;
  return bad_local ? 2 : 0;
}
