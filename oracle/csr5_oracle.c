/*
 * csr5_oracle.c -- sequential C restatement of the reference CSR5 path.
 *
 * TEST INFRASTRUCTURE ONLY (see csr5_oracle.h).  Each function cites the
 * reference file:line it restates; paths are relative to
 * /root/reference/proj/core/src.  Written from the reference's behaviour,
 * not translated line by line: the tile walks below work on packed words
 * and flat arrays instead of per-tile std::vectors.
 */
#include "csr5_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static void set_err(char *err, size_t len, const char *msg) {
  if (err && len) {
    strncpy(err, msg, len - 1);
    err[len - 1] = '\0';
  }
}

static int bit_width_u64(uint64_t x) { return x ? 64 - __builtin_clzll(x) : 0; }

static uint64_t low_mask(int bits) { return bits >= 64 ? ~(uint64_t)0 : (((uint64_t)1 << bits) - 1); }

/* tuning.cpp:8-15 */
int orc_validate_params(int64_t omega, int64_t sigma, int64_t r, int64_t s, int64_t t,
                        int64_t u, char *err, size_t errlen) {
  if (omega < 1 || sigma < 1) {
    set_err(err, errlen, "tuning: omega and sigma must be >= 1");
    return ORC_EINVAL;
  }
  if (omega * sigma < 2) {
    set_err(err, errlen,
            "tuning: omega * sigma must be >= 2; a tile needs at least two entries for "
            "segmentation");
    return ORC_EINVAL;
  }
  if (!(r <= s && s <= t)) {
    set_err(err, errlen, "tuning: bounds must satisfy r <= s <= t");
    return ORC_EINVAL;
  }
  if (u < 1) {
    set_err(err, errlen, "tuning: u must be >= 1");
    return ORC_EINVAL;
  }
  return ORC_OK;
}

/* tuning.cpp:25-34: piecewise rule on the average row length. */
int orc_select_sigma(double nnz_per_row, int64_t r, int64_t s, int64_t t, int64_t u,
                     int64_t *out, char *err, size_t errlen) {
  if (!(r <= s && s <= t)) {
    set_err(err, errlen, "select_sigma: bounds must satisfy r <= s <= t");
    return ORC_EINVAL;
  }
  if (nnz_per_row <= (double)r)
    *out = r;
  else if (nnz_per_row <= (double)s)
    *out = (int64_t)llround(nnz_per_row);
  else if (nnz_per_row <= (double)t)
    *out = s;
  else
    *out = u;
  return ORC_OK;
}

/* descriptor.cpp:17-20: bits needed for every value in [0, v). */
int orc_ceil_log2(int64_t v) { return v < 1 ? -1 : bit_width_u64((uint64_t)v - 1); }

/* descriptor.cpp:22-36 */
int orc_layout(int64_t omega, int64_t sigma, int *y_bits, int *seg_bits, int *word_bits,
               char *err, size_t errlen) {
  if (omega < 1 || sigma < 1) {
    set_err(err, errlen, "descriptor layout: omega and sigma must be >= 1");
    return ORC_EINVAL;
  }
  const int yb = orc_ceil_log2(omega * sigma);
  const int sb = orc_ceil_log2(omega);
  const int64_t total = yb + sb + sigma;
  if (total > 64) {
    char buf[160];
    snprintf(buf, sizeof buf,
             "descriptor layout: %lld bits per column exceed a 64-bit word; choose a smaller "
             "sigma",
             (long long)total);
    set_err(err, errlen, buf);
    return ORC_EINVAL;
  }
  *y_bits = yb;
  *seg_bits = sb;
  *word_bits = total <= 32 ? 32 : 64;
  return ORC_OK;
}

/* format.cpp:22-24 */
int orc_tile_ptr_bits(int64_t m) { return m < ((int64_t)1 << 31) ? 32 : 64; }

/* format.cpp:42-50: rightmost row whose row_ptr <= g, clamped to [0, m-1]. */
int64_t orc_row_of_nonzero(const int64_t *row_ptr, int64_t m, int64_t g) {
  if (m <= 0) return 0;
  /* upper_bound over the m+1 entries: first index with row_ptr[idx] > g. */
  int64_t lo = 0, hi = m + 1;
  while (lo < hi) {
    const int64_t mid = lo + (hi - lo) / 2;
    if (row_ptr[mid] <= g)
      lo = mid + 1;
    else
      hi = mid;
  }
  int64_t r = lo - 1;
  if (r < 0) r = 0;
  if (r > m - 1) r = m - 1;
  return r;
}

/* descriptor.cpp:38-62: word = y << (seg_bits + sigma) | seg << sigma | flags,
 * depth j at bit sigma-1-j. */
int orc_pack_desc(const int64_t *y_offset, const int64_t *seg_offset, const uint8_t *bf,
                  int64_t omega, int64_t sigma, int y_bits, int seg_bits, uint64_t *words) {
  for (int64_t i = 0; i < omega; ++i) {
    const uint64_t y = (uint64_t)y_offset[i];
    const uint64_t s = (uint64_t)seg_offset[i];
    if (y > low_mask(y_bits) || s > low_mask(seg_bits)) return ORC_EINVAL;
    uint64_t w = (y << (seg_bits + sigma)) | (s << sigma);
    for (int64_t j = 0; j < sigma; ++j)
      if (bf[i * sigma + j]) w |= (uint64_t)1 << (sigma - 1 - j);
    words[i] = w;
  }
  return ORC_OK;
}

/* descriptor.cpp:64-88 */
void orc_unpack_desc(const uint64_t *words, int64_t omega, int64_t sigma, int y_bits,
                     int seg_bits, int64_t *y_offset, int64_t *seg_offset, uint8_t *bf) {
  for (int64_t i = 0; i < omega; ++i) {
    const uint64_t w = words[i];
    y_offset[i] = (int64_t)((w >> (seg_bits + sigma)) & low_mask(y_bits));
    seg_offset[i] = (int64_t)((w >> sigma) & low_mask(seg_bits));
    for (int64_t j = 0; j < sigma; ++j) bf[i * sigma + j] = (uint8_t)((w >> (sigma - 1 - j)) & 1u);
  }
}

/* format.cpp:84-100: row starts inside the tile (empty-row runs collapse),
 * position 0 forced. */
void orc_bit_flag(const int64_t *row_ptr, int64_t m, int64_t tid, int64_t omega, int64_t sigma,
                  uint8_t *bf) {
  const int64_t block = omega * sigma;
  const int64_t start = tid * block, end = start + block;
  memset(bf, 0, (size_t)block);
  /* lower_bound over row_ptr[0..m) */
  int64_t lo = 0, hi = m;
  while (lo < hi) {
    const int64_t mid = lo + (hi - lo) / 2;
    if (row_ptr[mid] < start)
      lo = mid + 1;
    else
      hi = mid;
  }
  for (int64_t r = lo; r < m && row_ptr[r] < end; ++r) bf[row_ptr[r] - start] = 1;
  bf[0] = 1;
}

/* format.cpp:102-121: y_offset = exclusive scan of per-column head counts;
 * seg_offset = headless columns following a head-bearing column. */
void orc_y_seg_offset(const uint8_t *bf, int64_t omega, int64_t sigma, int64_t *y_offset,
                      int64_t *seg_offset) {
  /* The reference runs serial_segmented_sum over (data = !has_head,
   * flags = has_head); restated directly: a head-bearing column counts the
   * headless columns that follow it, every other column gets 0. */
  uint8_t *has = (uint8_t *)malloc((size_t)(omega ? omega : 1));
  int64_t acc = 0;
  for (int64_t i = 0; i < omega; ++i) {
    int64_t heads = 0;
    for (int64_t j = 0; j < sigma; ++j) heads += bf[i * sigma + j];
    y_offset[i] = acc;
    acc += heads;
    has[i] = heads > 0;
  }
  for (int64_t i = 0; i < omega; ++i) {
    int64_t k = 0;
    if (has[i])
      for (int64_t c = i + 1; c < omega && !has[c]; ++c) ++k;
    seg_offset[i] = k;
  }
  free(has);
}

/* segmented_sum.hpp:15-27 */
void orc_serial_segsum(double *data, const uint8_t *flags, int64_t n) {
  for (int64_t i = 0; i < n; ++i) {
    if (flags[i]) {
      for (int64_t j = i + 1; j < n && !flags[j]; ++j) data[i] += data[j];
    } else {
      data[i] = 0.0;
    }
  }
}

/* segmented_sum.cpp:25-48: out[i] = S[i+seg[i]] - S[i] + in[i], S the
 * left-to-right inclusive scan. */
int orc_fast_segsum(double *data, const int64_t *seg_offset, int64_t n) {
  for (int64_t i = 0; i < n; ++i)
    if (seg_offset[i] < 0 || i + seg_offset[i] >= n) return ORC_ERANGE;
  double *orig = (double *)malloc(sizeof(double) * (size_t)(n ? n : 1));
  memcpy(orig, data, sizeof(double) * (size_t)n);
  double acc = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    acc += data[i];
    data[i] = acc;
  }
  for (int64_t i = 0; i < n; ++i) data[i] = data[i + seg_offset[i]] - data[i] + orig[i];
  free(orig);
  return ORC_OK;
}

/* format.cpp:52-82: tile pointers with the empty-row flag in the MSB. */
static int build_tile_ptr(const int64_t *row_ptr, int64_t m, int64_t p, int64_t block, int bits,
                          uint64_t *out, char *err, size_t errlen) {
  const uint64_t flag = (uint64_t)1 << (bits - 1);
  int64_t *rows = (int64_t *)malloc(sizeof(int64_t) * (size_t)(p + 1));
  for (int64_t t = 0; t <= p; ++t) rows[t] = orc_row_of_nonzero(row_ptr, m, t * block);
  for (int64_t t = 0; t <= p; ++t) {
    int empty = 0;
    if (t < p) {
      /* inclusive right endpoint, rid < m (format.cpp:65-78) */
      for (int64_t rid = rows[t]; rid <= rows[t + 1] && rid < m; ++rid) {
        if (row_ptr[rid] == row_ptr[rid + 1]) {
          empty = 1;
          break;
        }
      }
    }
    if ((uint64_t)rows[t] >= flag) {
      char buf[96];
      snprintf(buf, sizeof buf, "tile_ptr: row index does not fit in %d bits", bits - 1);
      set_err(err, errlen, buf);
      free(rows);
      return ORC_EINVAL;
    }
    out[t] = (uint64_t)rows[t] | (empty ? flag : 0);
  }
  free(rows);
  return ORC_OK;
}

void orc_free(orc_csr5 *a) {
  free(a->tile_ptr);
  free(a->tile_desc);
  free(a->eo_ptr);
  free(a->eo);
  free(a->row_ptr);
  free(a->col_idx);
  free(a->val);
  memset(a, 0, sizeof *a);
}

static void *xmalloc(size_t n) { return malloc(n ? n : 1); }

/* format.cpp:165-252 */
int orc_build(int64_t m, int64_t n, const int64_t *row_ptr, const int64_t *col_idx,
              const double *val, int64_t omega, int64_t sigma, int64_t r, int64_t s, int64_t t,
              int64_t u, orc_csr5 *out, char *err, size_t errlen) {
  memset(out, 0, sizeof *out);
  int rc = orc_validate_params(omega, sigma, r, s, t, u, err, errlen);
  if (rc) return rc;
  int yb, sb, wb;
  rc = orc_layout(omega, sigma, &yb, &sb, &wb, err, errlen);
  if (rc) return rc;
  const int64_t block = omega * sigma;
  const int64_t nnz = row_ptr[m];
  out->m = m;
  out->n = n;
  out->nnz = nnz;
  out->omega = omega;
  out->sigma = sigma;
  out->p = (nnz + block - 1) / block;
  out->pc = nnz / block;
  out->tail_len = nnz % block;
  out->tile_ptr_bits = orc_tile_ptr_bits(m);
  out->y_bits = yb;
  out->seg_bits = sb;
  out->word_bits = wb;
  const int64_t p = out->p, pc = out->pc;

  out->row_ptr = (int64_t *)xmalloc(sizeof(int64_t) * (size_t)(m + 1));
  memcpy(out->row_ptr, row_ptr, sizeof(int64_t) * (size_t)(m + 1));
  out->col_idx = (int64_t *)xmalloc(sizeof(int64_t) * (size_t)nnz);
  out->val = (double *)xmalloc(sizeof(double) * (size_t)nnz);
  out->tile_ptr = (uint64_t *)xmalloc(sizeof(uint64_t) * (size_t)(p + 1));
  out->tile_desc = (uint64_t *)xmalloc(sizeof(uint64_t) * (size_t)(pc * omega));
  out->eo_ptr = (int64_t *)xmalloc(sizeof(int64_t) * (size_t)(pc + 1));

  rc = build_tile_ptr(row_ptr, m, p, block, out->tile_ptr_bits, out->tile_ptr, err, errlen);
  if (rc) {
    orc_free(out);
    return rc;
  }

  const uint64_t flag = (uint64_t)1 << (out->tile_ptr_bits - 1);
  uint8_t *bf = (uint8_t *)xmalloc((size_t)block);
  int64_t *yo = (int64_t *)xmalloc(sizeof(int64_t) * (size_t)omega);
  int64_t *so = (int64_t *)xmalloc(sizeof(int64_t) * (size_t)omega);

  /* Pass 1: descriptors + per-tile eo counts (format.cpp:196-210). */
  out->eo_ptr[0] = 0;
  for (int64_t tid = 0; tid < pc; ++tid) {
    orc_bit_flag(row_ptr, m, tid, omega, sigma, bf);
    orc_y_seg_offset(bf, omega, sigma, yo, so);
    orc_pack_desc(yo, so, bf, omega, sigma, yb, sb, out->tile_desc + tid * omega);
    int64_t heads = 0;
    if (out->tile_ptr[tid] & flag)
      for (int64_t k = 0; k < block; ++k) heads += bf[k];
    out->eo_ptr[tid + 1] = out->eo_ptr[tid] + heads;
  }
  /* Pass 2: empty_offset lists for flagged complete tiles (format.cpp:123-136). */
  out->eo = (int64_t *)xmalloc(sizeof(int64_t) * (size_t)out->eo_ptr[pc]);
  for (int64_t tid = 0; tid < pc; ++tid) {
    if (!(out->tile_ptr[tid] & flag)) continue;
    orc_bit_flag(row_ptr, m, tid, omega, sigma, bf);
    const int64_t tile_row = (int64_t)(out->tile_ptr[tid] & (flag - 1));
    int64_t k = out->eo_ptr[tid];
    for (int64_t pos = 0; pos < block; ++pos) /* logical order i*sigma+j */
      if (bf[pos]) out->eo[k++] = orc_row_of_nonzero(row_ptr, m, tid * block + pos) - tile_row;
  }
  /* Transposition of complete tiles, tail untouched (format.cpp:226-249). */
  memcpy(out->col_idx, col_idx, sizeof(int64_t) * (size_t)nnz);
  memcpy(out->val, val, sizeof(double) * (size_t)nnz);
  for (int64_t tid = 0; tid < pc; ++tid) {
    const int64_t base = tid * block;
    for (int64_t i = 0; i < omega; ++i)
      for (int64_t j = 0; j < sigma; ++j) {
        out->col_idx[base + j * omega + i] = col_idx[base + i * sigma + j];
        out->val[base + j * omega + i] = val[base + i * sigma + j];
      }
  }
  free(bf);
  free(yo);
  free(so);
  return ORC_OK;
}

typedef struct {
  int64_t *rows;
  double *vals;
  uint8_t *acc;
  int64_t count, cap;
} contrib_buf;

static void push(contrib_buf *b, int64_t row, double v, int accumulate) {
  if (b->count < b->cap) {
    b->rows[b->count] = row;
    b->vals[b->count] = v;
    b->acc[b->count] = (uint8_t)accumulate;
  }
  ++b->count;
}

/* spmv.cpp:42-106: Algorithm 8 on one complete tile.  The red piece of
 * column i lands in tmp[i-1]; greens close inside a column; blues are the
 * column bottoms spliced across headless columns by the fast segmented sum. */
static void run_tile(const orc_csr5 *a, int64_t tid, const double *x, contrib_buf *b) {
  const int64_t omega = a->omega, sigma = a->sigma;
  const uint64_t flagbit = (uint64_t)1 << (a->tile_ptr_bits - 1);
  const int64_t tile_row = (int64_t)(a->tile_ptr[tid] & (flagbit - 1));
  const int flagged = (a->tile_ptr[tid] & flagbit) != 0;
  const int64_t *eo = flagged ? a->eo + a->eo_ptr[tid] : NULL;
  double *tmp = (double *)calloc((size_t)omega, sizeof(double));
  double *last = (double *)calloc((size_t)omega, sizeof(double));
  int64_t *seg = (int64_t *)calloc((size_t)omega, sizeof(int64_t));
  int64_t *blue = (int64_t *)calloc((size_t)omega, sizeof(int64_t));
  uint8_t *has = (uint8_t *)calloc((size_t)omega, 1);
  const uint64_t fmask = low_mask((int)sigma);
  for (int64_t i = 0; i < omega; ++i) {
    const uint64_t w = a->tile_desc[tid * omega + i];
    int64_t head = (int64_t)((w >> (a->seg_bits + sigma)) & low_mask(a->y_bits));
    seg[i] = (int64_t)((w >> sigma) & low_mask(a->seg_bits));
    const uint64_t flags = w & fmask;
    double sum = 0.0;
    int seen = 0;
    for (int64_t j = 0; j < sigma; ++j) {
      if ((flags >> (sigma - 1 - j)) & 1u) {
        if (!seen) {
          if (i > 0) tmp[i - 1] = sum;
          seen = 1;
        } else {
          push(b, tile_row + (eo ? eo[head] : head), sum, head == 0);
          ++head;
        }
        sum = 0.0;
      }
      const int64_t ptr = tid * omega * sigma + j * omega + i;
      sum += a->val[ptr] * x[a->col_idx[ptr]];
    }
    last[i] = sum;
    has[i] = (uint8_t)seen;
    if (!seen && i > 0) tmp[i - 1] = sum;
    blue[i] = head;
  }
  orc_fast_segsum(tmp, seg, omega);
  for (int64_t i = 0; i < omega; ++i) {
    if (!has[i]) continue;
    push(b, tile_row + (eo ? eo[blue[i]] : blue[i]), last[i] + tmp[i], 1);
  }
  free(tmp);
  free(last);
  free(seg);
  free(blue);
  free(has);
}

int64_t orc_tile_contrib(const orc_csr5 *a, int64_t tid, const double *x, int64_t *rows,
                         double *vals, uint8_t *accumulate, int64_t cap) {
  if (tid < 0 || tid >= a->pc) return -1;
  contrib_buf b = {rows, vals, accumulate, 0, cap};
  run_tile(a, tid, x, &b);
  return b.count <= cap ? b.count : -1;
}

/* spmv.cpp:110-124 */
static void tail_add(const orc_csr5 *a, const double *x, double *y) {
  if (a->tail_len == 0) return;
  const uint64_t flagbit = (uint64_t)1 << (a->tile_ptr_bits - 1);
  const int64_t start = a->pc * a->omega * a->sigma;
  for (int64_t r = (int64_t)(a->tile_ptr[a->pc] & (flagbit - 1)); r < a->m; ++r) {
    const int64_t lo = a->row_ptr[r] > start ? a->row_ptr[r] : start;
    const int64_t hi = a->row_ptr[r + 1];
    if (lo >= hi) continue;
    double sum = 0.0;
    for (int64_t k = lo; k < hi; ++k) sum += a->val[k] * x[a->col_idx[k]];
    y[r] += sum;
  }
}

/* spmv.cpp:224-272: deterministic mode.  Exclusive contributions are stored
 * as they are produced; accumulate contributions are combined afterwards in
 * ascending tile order. */
void orc_spmv(const orc_csr5 *a, const double *x, double *y) {
  for (int64_t i = 0; i < a->m; ++i) y[i] = 0.0;
  if (a->nnz == 0) return;
  const int64_t cap = a->omega + 1; /* spmv.cpp:238 */
  const int64_t total = a->pc * cap;
  int64_t *acc_rows = (int64_t *)xmalloc(sizeof(int64_t) * (size_t)total);
  double *acc_vals = (double *)xmalloc(sizeof(double) * (size_t)total);
  int64_t *acc_cnt = (int64_t *)xmalloc(sizeof(int64_t) * (size_t)(a->pc));
  for (int64_t tid = 0; tid < a->pc; ++tid) {
    /* per-tile emission can exceed omega+1 only for exclusive entries; use a
     * generous buffer sized by the tile */
    const int64_t big = a->omega * a->sigma + 1;
    int64_t *r2 = (int64_t *)xmalloc(sizeof(int64_t) * (size_t)big);
    double *v2 = (double *)xmalloc(sizeof(double) * (size_t)big);
    uint8_t *a2 = (uint8_t *)xmalloc((size_t)big);
    contrib_buf b = {r2, v2, a2, 0, big};
    run_tile(a, tid, x, &b);
    int64_t c = 0;
    for (int64_t k = 0; k < b.count; ++k) {
      if (a2[k]) {
        acc_rows[tid * cap + c] = r2[k];
        acc_vals[tid * cap + c] = v2[k];
        ++c;
      } else {
        y[r2[k]] = v2[k];
      }
    }
    acc_cnt[tid] = c;
    free(r2);
    free(v2);
    free(a2);
  }
  for (int64_t tid = 0; tid < a->pc; ++tid)
    for (int64_t k = 0; k < acc_cnt[tid]; ++k) y[acc_rows[tid * cap + k]] += acc_vals[tid * cap + k];
  tail_add(a, x, y);
  free(acc_rows);
  free(acc_vals);
  free(acc_cnt);
}

/* csr.cpp:85-98 */
void orc_dense_spmv(int64_t m, const int64_t *row_ptr, const int64_t *col_idx,
                    const double *val, const double *x, double *y) {
  for (int64_t i = 0; i < m; ++i) {
    double sum = 0.0;
    for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k) sum += val[k] * x[col_idx[k]];
    y[i] = sum;
  }
}

/* format.cpp:254-265 with format.hpp:91-103 */
void orc_csr5_to_csr(const orc_csr5 *a, int64_t *col_idx_out, double *val_out) {
  const int64_t block = a->omega * a->sigma;
  memcpy(col_idx_out, a->col_idx, sizeof(int64_t) * (size_t)a->nnz);
  memcpy(val_out, a->val, sizeof(double) * (size_t)a->nnz);
  if (block <= 1) return;
  for (int64_t tid = 0; tid < a->pc; ++tid) {
    const int64_t base = tid * block;
    for (int64_t i = 0; i < a->omega; ++i)
      for (int64_t j = 0; j < a->sigma; ++j) {
        col_idx_out[base + i * a->sigma + j] = a->col_idx[base + j * a->omega + i];
        val_out[base + i * a->sigma + j] = a->val[base + j * a->omega + i];
      }
  }
}
