/*
 * testgen.c -- test-matrix generators restated from the reference so the
 * GPU parity tests run on exactly the matrices the reference tests use.
 *
 * TEST INFRASTRUCTURE ONLY (see csr5_oracle.h).
 *
 *  - orc_mt64_*: the MT19937-64 engine (std::mt19937_64, the RNG every
 *    reference test and generator uses), restated from its published
 *    definition (Matsumoto & Nishimura 2000, 64-bit parameters).
 *  - orc_random_csr / orc_random_x: tests/test_helpers.hpp:13-29.
 *  - orc_coo_to_csr: csr.cpp:35-72 (stable (row,col) sort, duplicates summed).
 *  - orc_generate_synthetic: synthetic.cpp:101-181.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define MT_N 312
#define MT_M 156

typedef struct {
  uint64_t mt[MT_N];
  int idx;
} orc_mt64;

void orc_mt64_seed(orc_mt64 *g, uint64_t seed) {
  g->mt[0] = seed;
  for (int i = 1; i < MT_N; ++i)
    g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
  g->idx = MT_N;
}

orc_mt64 *orc_mt64_new(uint64_t seed) {
  orc_mt64 *g = (orc_mt64 *)malloc(sizeof(orc_mt64));
  orc_mt64_seed(g, seed);
  return g;
}

void orc_mt64_delete(orc_mt64 *g) { free(g); }

uint64_t orc_mt64_next(orc_mt64 *g) {
  static const uint64_t UPPER = 0xFFFFFFFF80000000ULL, LOWER = 0x7FFFFFFFULL;
  static const uint64_t MATRIX_A = 0xB5026F5AA96619E9ULL;
  if (g->idx >= MT_N) {
    for (int i = 0; i < MT_N; ++i) {
      const uint64_t y = (g->mt[i] & UPPER) | (g->mt[(i + 1) % MT_N] & LOWER);
      uint64_t v = g->mt[(i + MT_M) % MT_N] ^ (y >> 1);
      if (y & 1) v ^= MATRIX_A;
      g->mt[i] = v;
    }
    g->idx = 0;
  }
  uint64_t x = g->mt[g->idx++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= x >> 43;
  return x;
}

static double unit_double(orc_mt64 *g) { return (double)(orc_mt64_next(g) >> 11) * 0x1.0p-53; }

/* CSR result of the generators; arrays malloc'd, free with orc_csr_free. */
typedef struct {
  int64_t m, n, nnz;
  int64_t *row_ptr;
  int64_t *col_idx;
  double *val;
} orc_csr;

void orc_csr_free(orc_csr *a) {
  free(a->row_ptr);
  free(a->col_idx);
  free(a->val);
  memset(a, 0, sizeof *a);
}

typedef struct {
  int64_t row, col;
  double v;
  int64_t ord;
} coo_e;

static int coo_cmp(const void *pa, const void *pb) {
  const coo_e *a = (const coo_e *)pa, *b = (const coo_e *)pb;
  if (a->row != b->row) return a->row < b->row ? -1 : 1;
  if (a->col != b->col) return a->col < b->col ? -1 : 1;
  return a->ord < b->ord ? -1 : (a->ord > b->ord);
}

/* csr.cpp:35-72; entries must be in bounds (callers here guarantee it). */
static void coo_to_csr(coo_e *e, int64_t cnt, int64_t m, int64_t n, orc_csr *out) {
  for (int64_t k = 0; k < cnt; ++k) e[k].ord = k;
  qsort(e, (size_t)cnt, sizeof(coo_e), coo_cmp);
  out->m = m;
  out->n = n;
  out->row_ptr = (int64_t *)calloc((size_t)(m + 1), sizeof(int64_t));
  out->col_idx = (int64_t *)malloc(sizeof(int64_t) * (size_t)(cnt ? cnt : 1));
  out->val = (double *)malloc(sizeof(double) * (size_t)(cnt ? cnt : 1));
  int64_t nnz = 0;
  for (int64_t k = 0; k < cnt;) {
    const int64_t row = e[k].row, col = e[k].col;
    double sum = 0.0;
    while (k < cnt && e[k].row == row && e[k].col == col) sum += e[k++].v;
    out->col_idx[nnz] = col;
    out->val[nnz] = sum;
    ++nnz;
    out->row_ptr[row + 1] += 1;
  }
  for (int64_t i = 0; i < m; ++i) out->row_ptr[i + 1] += out->row_ptr[i];
  out->nnz = nnz;
}

/* Public COO->CSR for tests: rows/cols/vals arrays of length cnt. */
void orc_coo_to_csr(const int64_t *rows, const int64_t *cols, const double *vals, int64_t cnt,
                    int64_t m, int64_t n, orc_csr *out) {
  coo_e *e = (coo_e *)malloc(sizeof(coo_e) * (size_t)(cnt ? cnt : 1));
  for (int64_t k = 0; k < cnt; ++k) {
    e[k].row = rows[k];
    e[k].col = cols[k];
    e[k].v = vals[k];
  }
  coo_to_csr(e, cnt, m, n, out);
  free(e);
}

/* tests/test_helpers.hpp:13-24 */
void orc_random_csr(orc_mt64 *g, int64_t m, int64_t n, int64_t nnz_target, orc_csr *out) {
  coo_e *e = (coo_e *)malloc(sizeof(coo_e) * (size_t)(nnz_target ? nnz_target : 1));
  for (int64_t k = 0; k < nnz_target; ++k) {
    e[k].row = (int64_t)(orc_mt64_next(g) % (uint64_t)m);
    e[k].col = (int64_t)(orc_mt64_next(g) % (uint64_t)n);
    e[k].v = 0.5 + unit_double(g);
  }
  coo_to_csr(e, nnz_target, m, n, out);
  free(e);
}

/* tests/test_helpers.hpp:26-29, bench.cpp:103-105 */
void orc_random_x(orc_mt64 *g, int64_t n, double *x) {
  for (int64_t i = 0; i < n; ++i) x[i] = 0.5 + unit_double(g);
}

/* synthetic.cpp:27-47: l distinct sorted columns of [0, n). */
static void sample_columns(orc_mt64 *g, int64_t l, int64_t n, int64_t *out) {
  if (l == n) {
    for (int64_t c = 0; c < n; ++c) out[c] = c;
    return;
  }
  uint8_t *mark = (uint8_t *)calloc((size_t)n, 1);
  if (l <= n / 2) {
    int64_t got = 0;
    while (got < l) {
      const int64_t c = (int64_t)(orc_mt64_next(g) % (uint64_t)n);
      if (!mark[c]) {
        mark[c] = 1;
        ++got;
      }
    }
    int64_t k = 0;
    for (int64_t c = 0; c < n; ++c)
      if (mark[c]) out[k++] = c;
  } else {
    int64_t got = 0;
    while (got < n - l) {
      const int64_t c = (int64_t)(orc_mt64_next(g) % (uint64_t)n);
      if (!mark[c]) {
        mark[c] = 1;
        ++got;
      }
    }
    int64_t k = 0;
    for (int64_t c = 0; c < n; ++c)
      if (!mark[c]) out[k++] = c;
  }
  free(mark);
}

/* synthetic.cpp:54-80 */
static void from_lengths(const int64_t *len, int64_t m, int64_t n, orc_mt64 *g, int random_cols,
                         orc_csr *out) {
  out->m = m;
  out->n = n;
  out->row_ptr = (int64_t *)calloc((size_t)(m + 1), sizeof(int64_t));
  for (int64_t i = 0; i < m; ++i) out->row_ptr[i + 1] = out->row_ptr[i] + len[i];
  const int64_t nnz = out->row_ptr[m];
  out->nnz = nnz;
  out->col_idx = (int64_t *)malloc(sizeof(int64_t) * (size_t)(nnz ? nnz : 1));
  out->val = (double *)malloc(sizeof(double) * (size_t)(nnz ? nnz : 1));
  for (int64_t i = 0; i < m; ++i) {
    const int64_t l = len[i], base = out->row_ptr[i];
    if (l == 0) continue;
    if (random_cols)
      sample_columns(g, l, n, out->col_idx + base);
    else
      for (int64_t j = 0; j < l; ++j) out->col_idx[base + j] = j * n / l;
    for (int64_t j = 0; j < l; ++j) out->val[base + j] = 0.5 + unit_double(g);
  }
}

/* synthetic.cpp:101-181.  kind: 0 regular, 1 one_long_row, 2 random_skew.
 * Returns 0 on success, 1 when the target is infeasible. */
int orc_generate_synthetic(int kind, int64_t m, int64_t n, int64_t nnz_target, uint64_t seed,
                           double long_row_fraction, orc_csr *out) {
  memset(out, 0, sizeof *out);
  if (m < 1 || n < 1 || nnz_target < 0 || nnz_target > m * n) return 1;
  orc_mt64 g;
  orc_mt64_seed(&g, seed);
  int64_t *len = (int64_t *)calloc((size_t)m, sizeof(int64_t));
  int rc = 0;
  if (kind == 0) {
    const int64_t base = nnz_target / m, extra = nnz_target % m;
    for (int64_t i = 0; i < m; ++i) len[i] = base + (i < extra ? 1 : 0);
    if (base + (extra ? 1 : 0) > n) rc = 1;
    if (!rc) from_lengths(len, m, n, &g, 0, out);
  } else if (kind == 1) {
    if (long_row_fraction < 0.0 || long_row_fraction > 1.0) rc = 1;
    int64_t long_len = (int64_t)llround(long_row_fraction * (double)nnz_target);
    if (long_len > nnz_target) long_len = nnz_target;
    if (!rc && long_len > n) rc = 1;
    const int64_t rest = nnz_target - long_len;
    if (!rc && m == 1) {
      len[0] = nnz_target;
      if (nnz_target > n) rc = 1;
    } else if (!rc) {
      if (rest > (m - 1) * n) rc = 1;
      if (!rc) {
        const int64_t long_row = (int64_t)(orc_mt64_next(&g) % (uint64_t)m);
        const int64_t base = rest / (m - 1), extra = rest % (m - 1);
        if (base + (extra ? 1 : 0) > n) rc = 1;
        int64_t k = 0;
        for (int64_t i = 0; i < m && !rc; ++i) {
          if (i == long_row)
            len[i] = long_len;
          else
            len[i] = base + (k++ < extra ? 1 : 0);
        }
      }
    }
    if (!rc) from_lengths(len, m, n, &g, 0, out);
  } else {
    const double mean = (double)nnz_target / (double)m;
    int64_t total = 0;
    for (int64_t i = 0; i < m; ++i) {
      const double u = unit_double(&g);
      int64_t d = (int64_t)(-mean * log1p(-u));
      if (d < 0) d = 0;
      if (d > n) d = n;
      len[i] = d;
      total += d;
    }
    while (total < nnz_target) {
      const int64_t i = (int64_t)(orc_mt64_next(&g) % (uint64_t)m);
      if (len[i] < n) {
        ++len[i];
        ++total;
      }
    }
    while (total > nnz_target) {
      const int64_t i = (int64_t)(orc_mt64_next(&g) % (uint64_t)m);
      if (len[i] > 0) {
        --len[i];
        --total;
      }
    }
    from_lengths(len, m, n, &g, 1, out);
  }
  free(len);
  return rc;
}

/* Host twin of csr5g_stencil_box_fill (paper_1503_05032_b200/csrc/synth.cu)
 * for the reference arm of bench.py: kind 0 = 2D 5-point (a x layers), kind 1
 * = 3D 27-point (a x a x layers); layers = a is the square / cube.  Caller
 * buffers: row_ptr[m+1], col_idx[nnz], val[nnz]. */
void orc_stencil_box(int kind, int64_t a, int64_t layers, int64_t *row_ptr, int64_t *col_idx,
                     double *val) {
  const int64_t m = kind == 0 ? a * layers : a * a * layers;
  int64_t q = 0;
  row_ptr[0] = 0;
  for (int64_t r = 0; r < m; ++r) {
    if (kind == 0) {
      const int64_t iy = r / a, ix = r - iy * a;
      const int64_t cand[5] = {r - a, r - 1, r, r + 1, r + a};
      const int ok[5] = {iy > 0, ix > 0, 1, ix < a - 1, iy < layers - 1};
      for (int k = 0; k < 5; ++k)
        if (ok[k]) {
          col_idx[q] = cand[k];
          val[q] = cand[k] == r ? 4.0 : -1.0;
          ++q;
        }
    } else {
      const int64_t z = r / (a * a), rem = r - z * a * a, y = rem / a, x = rem - y * a;
      for (int dz = -1; dz <= 1; ++dz) {
        if (z + dz < 0 || z + dz >= layers) continue;
        for (int dy = -1; dy <= 1; ++dy) {
          if (y + dy < 0 || y + dy >= a) continue;
          for (int dx = -1; dx <= 1; ++dx) {
            if (x + dx < 0 || x + dx >= a) continue;
            col_idx[q] = r + dz * a * a + dy * a + dx;
            val[q] = (dz == 0 && dy == 0 && dx == 0) ? 26.0 : -1.0;
            ++q;
          }
        }
      }
    }
    row_ptr[r + 1] = q;
  }
}

void orc_stencil(int kind, int64_t a, int64_t *row_ptr, int64_t *col_idx, double *val) {
  orc_stencil_box(kind, a, a, row_ptr, col_idx, val);
}
