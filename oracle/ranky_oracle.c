/*
 * ranky_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the Ranky reference algorithm on the B200 hot
 * path (rank check + checker repair, block SVD, proxy merge, V recovery).
 * It is the CPU checker for the CUDA path: only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg may load it. The product path never calls it.
 *
 * Every routine names the reference routine it restates (paths relative to
 * /root/reference). Floating-point expressions keep the reference's operation
 * order and are compiled with -ffp-contract=off so that, on x86-64, results are
 * bit-identical to the reference build in oracle/_ref (checked by
 * tests/test_oracle.py).
 *
 * Data structures differ from the reference on purpose: the repair workspace
 * keeps the immutable CSR/CSC of the input plus a small overlay of inserted
 * edges, and the neighbor sets are bitmaps instead of sort+unique vectors.
 * The sets, their ascending order and the RNG draws are the same.
 */
#define _POSIX_C_SOURCE 199309L
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "or_result.h"


static const double kJacobiTol = 1e-14;   /* proj/src/svd.cpp:17 */
static const int kMaxSweeps = 60;         /* proj/src/svd.cpp:18 */
static const double kRankTol = 1e-10;     /* proj/include/ranky/svd.hpp:13 */
static const uint64_t kDensifyCap = (uint64_t)1 << 26; /* dense_matrix.hpp:45 */

/* ------------------------------------------------------------------------ */
/* result object shared with the Python wrapper (oracle/oracle.py mirrors it) */



static void set_err(or_result *res, int code, const char *msg) {
  if (res->status == OR_OK) {
    res->status = code;
    snprintf(res->message, sizeof res->message, "%s", msg);
  }
}

void or_free(or_result *res) {
  if (!res) return;
  free(res->e_block); free(res->e_row); free(res->e_col); free(res->e_mech);
  free(res->lonely); free(res->r); free(res->c); free(res->v);
  free(res->u); free(res->sigma); free(res->vm);
  free(res->rec_kept); free(res->rec_payload);
  free(res);
}

static or_result *new_result(void) { return (or_result *)calloc(1, sizeof(or_result)); }

/* ------------------------------------------------------------------------ */
/* KeyedRng -- proj/src/rng.cpp:8-38                                          */

static uint64_t mix64(uint64_t z) { /* rng.cpp:8-12, splitmix64 finalizer */
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

typedef struct { uint64_t s; } keyed_rng;

static keyed_rng rng_make(uint64_t seed, uint64_t block, uint64_t row) { /* rng.cpp:16-20 */
  keyed_rng g;
  g.s = mix64(seed + 0x9e3779b97f4a7c15ull);
  g.s = mix64(g.s ^ (block + 0xbf58476d1ce4e5b9ull));
  g.s = mix64(g.s ^ (row + 0x94d049bb133111ebull));
  return g;
}

static uint64_t rng_next(keyed_rng *g) { /* rng.cpp:22-25 */
  g->s += 0x9e3779b97f4a7c15ull;
  return mix64(g->s);
}

static uint64_t rng_below(keyed_rng *g, uint64_t bound) { /* rng.cpp:27-34 */
  const uint64_t threshold = (0 - bound) % bound;
  for (;;) {
    uint64_t x = rng_next(g);
    if (x >= threshold) return x % bound;
  }
}

static double rng_unit(keyed_rng *g) { /* rng.cpp:36-38 */
  return (double)(rng_next(g) >> 11) * 0x1.0p-53;
}

void or_rng_stream(uint64_t seed, uint64_t block, uint64_t row, uint64_t n, uint64_t *out) {
  keyed_rng g = rng_make(seed, block, row);
  for (uint64_t i = 0; i < n; ++i) out[i] = rng_next(&g);
}

uint64_t or_rng_below(uint64_t seed, uint64_t block, uint64_t row, uint64_t bound) {
  keyed_rng g = rng_make(seed, block, row);
  return rng_below(&g, bound);
}

double or_rng_unit(uint64_t seed, uint64_t block, uint64_t row, uint64_t skip) {
  keyed_rng g = rng_make(seed, block, row);
  for (uint64_t i = 0; i < skip; ++i) rng_next(&g);
  return rng_unit(&g);
}

/* ------------------------------------------------------------------------ */
/* sparse input: sorted COO (row, col) as SparseMatrix keeps it               */
/* (proj/src/sparse_matrix.cpp:9-34). Callers pass already-sorted entries.    */

typedef struct {
  uint64_t rows, cols, nnz;
  const uint64_t *r, *c;
  const double *v;
  uint64_t *row_ptr; /* rows + 1 */
} coo_view;

static int coo_open(coo_view *a, uint64_t rows, uint64_t cols, uint64_t nnz, const uint64_t *r,
                    const uint64_t *c, const double *v) {
  a->rows = rows; a->cols = cols; a->nnz = nnz; a->r = r; a->c = c; a->v = v;
  a->row_ptr = (uint64_t *)calloc(rows + 1, sizeof(uint64_t));
  if (!a->row_ptr) return OR_NOMEM;
  for (uint64_t i = 0; i < nnz; ++i) a->row_ptr[r[i] + 1]++;
  for (uint64_t i = 0; i < rows; ++i) a->row_ptr[i + 1] += a->row_ptr[i];
  return OR_OK;
}

static void coo_close(coo_view *a) { free(a->row_ptr); a->row_ptr = NULL; }

/* column partition -- proj/src/partition.cpp:38-51 */
static int partition_ok(uint64_t n_cols, uint64_t d, or_result *res) {
  if (d == 0 || d > n_cols) {
    char msg[160];
    snprintf(msg, sizeof msg, "cannot split %llu columns into %llu blocks",
             (unsigned long long)n_cols, (unsigned long long)d);
    set_err(res, OR_INVALID, msg);
    return 0;
  }
  return 1;
}
static uint64_t range_begin(uint64_t n, uint64_t d_count, uint64_t d) { return d * (n / d_count); }
static uint64_t range_end(uint64_t n, uint64_t d_count, uint64_t d) {
  return d + 1 == d_count ? n : (d + 1) * (n / d_count);
}

/* first index in sorted a[lo,hi) with a[i] >= key */
static uint64_t lower_u64(const uint64_t *a, uint64_t lo, uint64_t hi, uint64_t key) {
  while (lo < hi) {
    uint64_t mid = lo + (hi - lo) / 2;
    if (a[mid] < key) lo = mid + 1; else hi = mid;
  }
  return lo;
}

/* ------------------------------------------------------------------------ */
/* repair -- proj/src/repair.cpp:42-216                                       */
/* workspace: base CSR (the input, sorted) + base CSC + inserted-edge overlay */

typedef struct {
  uint64_t *cols; /* sorted inserted columns of one row */
  uint64_t n, cap;
} ins_list;

typedef struct {
  const coo_view *a;
  uint64_t *col_ptr, *col_rows; /* CSC of the input, rows ascending */
  ins_list *row_ins;            /* per row */
  uint64_t *ic_col, *ic_row;    /* inserted edges sorted by (col,row) */
  uint64_t n_ins, cap_ins;
} workspace;

static int ws_open(workspace *w, const coo_view *a) {
  memset(w, 0, sizeof *w);
  w->a = a;
  w->col_ptr = (uint64_t *)calloc(a->cols + 1, sizeof(uint64_t));
  w->col_rows = (uint64_t *)malloc((a->nnz ? a->nnz : 1) * sizeof(uint64_t));
  w->row_ins = (ins_list *)calloc(a->rows ? a->rows : 1, sizeof(ins_list));
  if (!w->col_ptr || !w->col_rows || !w->row_ins) return OR_NOMEM;
  for (uint64_t i = 0; i < a->nnz; ++i) w->col_ptr[a->c[i] + 1]++;
  for (uint64_t j = 0; j < a->cols; ++j) w->col_ptr[j + 1] += w->col_ptr[j];
  uint64_t *fill = (uint64_t *)malloc((a->cols ? a->cols : 1) * sizeof(uint64_t));
  if (!fill) return OR_NOMEM;
  memcpy(fill, w->col_ptr, a->cols * sizeof(uint64_t));
  for (uint64_t i = 0; i < a->nnz; ++i) w->col_rows[fill[a->c[i]]++] = a->r[i]; /* rows ascending */
  free(fill);
  return OR_OK;
}

static void ws_close(workspace *w) {
  free(w->col_ptr); free(w->col_rows);
  if (w->row_ins)
    for (uint64_t i = 0; i < w->a->rows; ++i) free(w->row_ins[i].cols);
  free(w->row_ins); free(w->ic_col); free(w->ic_row);
}

static int ws_has(const workspace *w, uint64_t row, uint64_t col) {
  const coo_view *a = w->a;
  uint64_t lo = a->row_ptr[row], hi = a->row_ptr[row + 1];
  uint64_t p = lower_u64(a->c, lo, hi, col);
  if (p < hi && a->c[p] == col) return 1;
  const ins_list *l = &w->row_ins[row];
  uint64_t q = lower_u64(l->cols, 0, l->n, col);
  return q < l->n && l->cols[q] == col;
}

/* RepairWorkspace::insert -- repair.cpp:85-93 (idempotent) */
static int ws_insert(workspace *w, uint64_t row, uint64_t col) {
  if (ws_has(w, row, col)) return OR_OK;
  ins_list *l = &w->row_ins[row];
  if (l->n == l->cap) {
    l->cap = l->cap ? 2 * l->cap : 4;
    l->cols = (uint64_t *)realloc(l->cols, l->cap * sizeof(uint64_t));
    if (!l->cols) return OR_NOMEM;
  }
  uint64_t q = lower_u64(l->cols, 0, l->n, col);
  memmove(l->cols + q + 1, l->cols + q, (l->n - q) * sizeof(uint64_t));
  l->cols[q] = col;
  l->n++;
  if (w->n_ins == w->cap_ins) {
    w->cap_ins = w->cap_ins ? 2 * w->cap_ins : 64;
    w->ic_col = (uint64_t *)realloc(w->ic_col, w->cap_ins * sizeof(uint64_t));
    w->ic_row = (uint64_t *)realloc(w->ic_row, w->cap_ins * sizeof(uint64_t));
    if (!w->ic_col || !w->ic_row) return OR_NOMEM;
  }
  /* position in (col,row) order */
  uint64_t lo = 0, hi = w->n_ins;
  while (lo < hi) {
    uint64_t mid = lo + (hi - lo) / 2;
    if (w->ic_col[mid] < col || (w->ic_col[mid] == col && w->ic_row[mid] < row)) lo = mid + 1;
    else hi = mid;
  }
  memmove(w->ic_col + lo + 1, w->ic_col + lo, (w->n_ins - lo) * sizeof(uint64_t));
  memmove(w->ic_row + lo + 1, w->ic_row + lo, (w->n_ins - lo) * sizeof(uint64_t));
  w->ic_col[lo] = col;
  w->ic_row[lo] = row;
  w->n_ins++;
  return OR_OK;
}

/* RepairWorkspace::row_lonely_in_block -- repair.cpp:70-75 */
static int ws_lonely(const workspace *w, uint64_t row, uint64_t b, uint64_t e) {
  const coo_view *a = w->a;
  uint64_t lo = a->row_ptr[row], hi = a->row_ptr[row + 1];
  uint64_t p = lower_u64(a->c, lo, hi, b);
  if (p < hi && a->c[p] < e) return 0;
  const ins_list *l = &w->row_ins[row];
  uint64_t q = lower_u64(l->cols, 0, l->n, b);
  return !(q < l->n && l->cols[q] < e);
}

#define BIT_SET(bm, i) ((bm)[(i) >> 6] |= (1ull << ((i)&63)))
#define BIT_GET(bm, i) (((bm)[(i) >> 6] >> ((i)&63)) & 1ull)

/* RepairWorkspace::apply_neighbor -- repair.cpp:103-135.
 * Returns 1 and sets *col when a neighbor column exists; 0 without consuming
 * a draw otherwise. cand (rows bits) and nb (width bits) are scratch. */
static int ws_apply_neighbor(workspace *w, uint64_t row, uint64_t b, uint64_t e, keyed_rng *g,
                             uint64_t *cand, uint64_t *nb, uint64_t *col_out, int *err) {
  const coo_view *a = w->a;
  const uint64_t M = a->rows, width = e - b;
  memset(cand, 0, ((M + 63) / 64) * sizeof(uint64_t));
  memset(nb, 0, ((width + 63) / 64) * sizeof(uint64_t));
  /* candidate rows: every row sharing a column with `row` outside [b,e) */
  const ins_list *own = &w->row_ins[row];
  for (int pass = 0; pass < 2; ++pass) {
    uint64_t n = pass == 0 ? a->row_ptr[row + 1] - a->row_ptr[row] : own->n;
    for (uint64_t i = 0; i < n; ++i) {
      uint64_t c = pass == 0 ? a->c[a->row_ptr[row] + i] : own->cols[i];
      if (c >= b && c < e) continue;
      for (uint64_t k = w->col_ptr[c]; k < w->col_ptr[c + 1]; ++k) BIT_SET(cand, w->col_rows[k]);
      /* inserted edges on column c */
      uint64_t lo = 0, hi = w->n_ins;
      while (lo < hi) {
        uint64_t mid = lo + (hi - lo) / 2;
        if (w->ic_col[mid] < c) lo = mid + 1; else hi = mid;
      }
      for (uint64_t k = lo; k < w->n_ins && w->ic_col[k] == c; ++k) BIT_SET(cand, w->ic_row[k]);
    }
  }
  /* their nonzero columns inside [b,e) */
  uint64_t count = 0;
  for (uint64_t m = 0; m < M; ++m) {
    if (!BIT_GET(cand, m)) continue;
    uint64_t lo = a->row_ptr[m], hi = a->row_ptr[m + 1];
    for (uint64_t p = lower_u64(a->c, lo, hi, b); p < hi && a->c[p] < e; ++p) {
      uint64_t j = a->c[p] - b;
      if (!BIT_GET(nb, j)) { BIT_SET(nb, j); count++; }
    }
    const ins_list *l = &w->row_ins[m];
    for (uint64_t q = lower_u64(l->cols, 0, l->n, b); q < l->n && l->cols[q] < e; ++q) {
      uint64_t j = l->cols[q] - b;
      if (!BIT_GET(nb, j)) { BIT_SET(nb, j); count++; }
    }
  }
  if (count == 0) return 0;
  uint64_t k = rng_below(g, count); /* k-th smallest column of the set */
  for (uint64_t word = 0;; ++word) {
    uint64_t bits = nb[word];
    uint64_t pc = (uint64_t)__builtin_popcountll(bits);
    if (k < pc) {
      while (k--) bits &= bits - 1;
      *col_out = b + word * 64 + (uint64_t)__builtin_ctzll(bits);
      break;
    }
    k -= pc;
  }
  *err = ws_insert(w, row, *col_out);
  return 1;
}

static int push_edge(or_result *res, uint64_t *cap, uint64_t d, uint64_t row, uint64_t col, int mech) {
  if (res->n_edges == *cap) {
    *cap = *cap ? 2 * *cap : 256;
    res->e_block = (uint64_t *)realloc(res->e_block, *cap * sizeof(uint64_t));
    res->e_row = (uint64_t *)realloc(res->e_row, *cap * sizeof(uint64_t));
    res->e_col = (uint64_t *)realloc(res->e_col, *cap * sizeof(uint64_t));
    res->e_mech = (int32_t *)realloc(res->e_mech, *cap * sizeof(int32_t));
    if (!res->e_block || !res->e_row || !res->e_col || !res->e_mech) return OR_NOMEM;
  }
  res->e_block[res->n_edges] = d;
  res->e_row[res->n_edges] = row;
  res->e_col[res->n_edges] = col;
  res->e_mech[res->n_edges] = mech;
  res->n_edges++;
  return OR_OK;
}

/* RepairWorkspace::to_matrix -- repair.cpp:147-160: input values preserved,
 * inserted edges carry 1.0, (row, col) order. */
static int ws_to_matrix(const workspace *w, or_result *res) {
  const coo_view *a = w->a;
  res->rows = a->rows; res->cols = a->cols;
  res->nnz = a->nnz + w->n_ins;
  uint64_t n = res->nnz ? res->nnz : 1;
  res->r = (uint64_t *)malloc(n * sizeof(uint64_t));
  res->c = (uint64_t *)malloc(n * sizeof(uint64_t));
  res->v = (double *)malloc(n * sizeof(double));
  if (!res->r || !res->c || !res->v) return OR_NOMEM;
  uint64_t o = 0;
  for (uint64_t row = 0; row < a->rows; ++row) {
    uint64_t p = a->row_ptr[row], pe = a->row_ptr[row + 1];
    const ins_list *l = &w->row_ins[row];
    uint64_t q = 0;
    while (p < pe || q < l->n) {
      if (q >= l->n || (p < pe && a->c[p] < l->cols[q])) {
        res->r[o] = row; res->c[o] = a->c[p]; res->v[o] = a->v[p]; ++p;
      } else {
        res->r[o] = row; res->c[o] = l->cols[q]; res->v[o] = 1.0; ++q;
      }
      ++o;
    }
  }
  return OR_OK;
}

/* repair -- repair.cpp:162-216. method: 0 random, 1 neighbor, 2 neighbor-random, 3 none */
static int repair_into(const coo_view *a, uint64_t D, int method, uint64_t seed, or_result *res) {
  if (!partition_ok(a->cols, D, res)) return res->status;
  res->n_blocks = D;
  res->lonely = (uint64_t *)calloc(D, sizeof(uint64_t));
  if (!res->lonely) return OR_NOMEM;
  if (method == 3) { /* kNone: the input unchanged, zero lonely counts */
    res->rows = a->rows; res->cols = a->cols; res->nnz = a->nnz;
    uint64_t n = a->nnz ? a->nnz : 1;
    res->r = (uint64_t *)malloc(n * sizeof(uint64_t));
    res->c = (uint64_t *)malloc(n * sizeof(uint64_t));
    res->v = (double *)malloc(n * sizeof(double));
    if (!res->r || !res->c || !res->v) return OR_NOMEM;
    memcpy(res->r, a->r, a->nnz * sizeof(uint64_t));
    memcpy(res->c, a->c, a->nnz * sizeof(uint64_t));
    memcpy(res->v, a->v, a->nnz * sizeof(double));
    return OR_OK;
  }
  workspace w;
  int st = ws_open(&w, a);
  uint64_t cap = 0;
  uint64_t *cand = NULL, *nb = NULL;
  uint64_t max_w = 0;
  for (uint64_t d = 0; d < D; ++d) {
    uint64_t wd = range_end(a->cols, D, d) - range_begin(a->cols, D, d);
    if (wd > max_w) max_w = wd;
  }
  cand = (uint64_t *)malloc(((a->rows + 63) / 64 + 1) * sizeof(uint64_t));
  nb = (uint64_t *)malloc(((max_w + 63) / 64 + 1) * sizeof(uint64_t));
  if (!cand || !nb) st = OR_NOMEM;
  for (uint64_t d = 0; d < D && st == OR_OK; ++d) {
    const uint64_t b = range_begin(a->cols, D, d), e = range_end(a->cols, D, d);
    /* the scan for block d runs before any block-d edge exists (repair.cpp:172-175) */
    uint64_t n_lonely = 0;
    for (uint64_t row = 0; row < a->rows; ++row) n_lonely += ws_lonely(&w, row, b, e);
    res->lonely[d] = n_lonely;
    for (uint64_t row = 0; row < a->rows && st == OR_OK; ++row) {
      /* rows of block d that were lonely before this block's repairs: edges
       * inserted below only touch this row, so re-testing later rows is safe */
      if (!ws_lonely(&w, row, b, e)) continue;
      keyed_rng g = rng_make(seed, d, row);
      uint64_t col = 0;
      int err = OR_OK;
      if (method == 0) { /* kRandom, repair.cpp:178-182 */
        col = b + rng_below(&g, e - b);
        st = ws_insert(&w, row, col);
        if (st == OR_OK) st = push_edge(res, &cap, d, row, col, 0);
      } else if (method == 1) { /* kNeighbor, repair.cpp:184-195 */
        if (ws_apply_neighbor(&w, row, b, e, &g, cand, nb, &col, &err)) {
          st = err;
          if (st == OR_OK) st = push_edge(res, &cap, d, row, col, 1);
        } else {
          col = b + rng_below(&g, e - b);
          st = ws_insert(&w, row, col);
          if (st == OR_OK) st = push_edge(res, &cap, d, row, col, 0);
          res->fallback++;
        }
      } else { /* kNeighborRandom, repair.cpp:196-209 */
        if (ws_apply_neighbor(&w, row, b, e, &g, cand, nb, &col, &err)) {
          st = err;
          if (st == OR_OK) st = push_edge(res, &cap, d, row, col, 1);
        }
        if (st != OR_OK) break;
        uint64_t rcol = b + rng_below(&g, e - b);
        st = ws_insert(&w, row, rcol);
        uint64_t k = res->n_edges;
        if (st == OR_OK && (k == 0 || res->e_block[k - 1] != d || res->e_row[k - 1] != row ||
                            res->e_col[k - 1] != rcol))
          st = push_edge(res, &cap, d, row, rcol, 0);
      }
    }
  }
  /* note: the lonely re-test above is equivalent to iterating the list taken
   * before the block's repairs, because repairs of row r only add entries to
   * row r and only rows that were lonely get repaired */
  if (st == OR_OK) st = ws_to_matrix(&w, res);
  free(cand); free(nb);
  ws_close(&w);
  if (st == OR_NOMEM) set_err(res, OR_NOMEM, "out of memory");
  return st;
}

or_result *or_repair(uint64_t rows, uint64_t cols, uint64_t nnz, const uint64_t *r, const uint64_t *c,
                     const double *v, uint64_t D, int method, uint64_t seed) {
  or_result *res = new_result();
  coo_view a;
  if (coo_open(&a, rows, cols, nnz, r, c, v) != OR_OK) { set_err(res, OR_NOMEM, "oom"); return res; }
  repair_into(&a, D, method, seed, res);
  coo_close(&a);
  return res;
}

/* find_lonely_rows -- repair.cpp:42-50; out must hold `rows` entries */
uint64_t or_find_lonely_rows(uint64_t rows, uint64_t cols, uint64_t nnz, const uint64_t *r,
                             const uint64_t *c, uint64_t D, uint64_t d, uint64_t *out) {
  coo_view a;
  if (coo_open(&a, rows, cols, nnz, r, c, NULL) != OR_OK) return 0;
  uint64_t b = range_begin(cols, D, d), e = range_end(cols, D, d), n = 0;
  for (uint64_t row = 0; row < rows; ++row) {
    uint64_t lo = a.row_ptr[row], hi = a.row_ptr[row + 1];
    uint64_t p = lower_u64(c, lo, hi, b);
    if (!(p < hi && c[p] < e)) out[n++] = row;
  }
  coo_close(&a);
  return n;
}

/* ------------------------------------------------------------------------ */
/* dense SVD -- proj/src/svd.cpp                                              */

typedef struct { uint64_t rows, cols; double *d; } cmat; /* column-major */

static int cmat_alloc(cmat *m, uint64_t r, uint64_t c) {
  m->rows = r; m->cols = c;
  m->d = (double *)calloc(r * c ? r * c : 1, sizeof(double));
  return m->d ? OR_OK : OR_NOMEM;
}
static double *ccol(const cmat *m, uint64_t j) { return m->d + j * m->rows; }

static double dot_n(const double *x, const double *y, uint64_t n) { /* svd.cpp:60-64 */
  double s = 0.0;
  for (uint64_t i = 0; i < n; ++i) s += x[i] * y[i];
  return s;
}

/* Householder QR of tall a in place -- svd.cpp:77-107. vs[k] is stored in
 * column k of `vs` (length rows - k, rest zero); betas[k] = 0 marks a skip. */
static void householder(cmat *a, cmat *vs, double *betas) {
  const uint64_t m = a->rows, n = a->cols;
  for (uint64_t k = 0; k < n; ++k) {
    double *ak = ccol(a, k);
    const uint64_t len = m - k;
    const double norm = sqrt(dot_n(ak + k, ak + k, len));
    double *v = ccol(vs, k);
    betas[k] = 0.0;
    if (norm == 0.0) continue;
    const double alpha = ak[k] >= 0.0 ? -norm : norm;
    for (uint64_t i = 0; i < len; ++i) v[i] = ak[k + i];
    v[0] -= alpha;
    const double vsq = dot_n(v, v, len);
    if (vsq == 0.0) { memset(v, 0, len * sizeof(double)); continue; }
    const double beta = 2.0 / vsq;
    betas[k] = beta;
    ak[k] = alpha;
    for (uint64_t i = 1; i < len; ++i) ak[k + i] = 0.0;
    for (uint64_t j = k + 1; j < n; ++j) {
      double *aj = ccol(a, j);
      const double wv = dot_n(v, aj + k, len);
      const double bw = beta * wv;
      for (uint64_t i = 0; i < len; ++i) aj[k + i] -= bw * v[i];
    }
  }
}

/* apply_q -- svd.cpp:111-132: out (m x x.cols) = H_0 ... H_{n-1} [x; 0] */
static int apply_q(const cmat *vs, const double *betas, uint64_t m, const cmat *x, cmat *out) {
  const uint64_t n = vs->cols;
  if (cmat_alloc(out, m, x->cols) != OR_OK) return OR_NOMEM;
  for (uint64_t j = 0; j < x->cols; ++j) memcpy(ccol(out, j), ccol(x, j), x->rows * sizeof(double));
  for (uint64_t j = 0; j < out->cols; ++j) {
    double *oj = ccol(out, j);
    for (uint64_t kk = n; kk-- > 0;) {
      const double beta = betas[kk];
      if (beta == 0.0) continue;
      const double *v = ccol(vs, kk);
      const uint64_t len = m - kk;
      const double wv = dot_n(v, oj + kk, len);
      const double bw = beta * wv;
      for (uint64_t i = 0; i < len; ++i) oj[kk + i] -= bw * v[i];
    }
  }
  return OR_OK;
}

/* complete_columns -- svd.cpp:150-201 */
static int complete_columns(cmat *u, const unsigned char *deficient, or_result *res) {
  const uint64_t m = u->rows, n = u->cols;
  double *w = (double *)calloc(m ? m : 1, sizeof(double));
  double *best = (double *)calloc(m ? m : 1, sizeof(double));
  if (!w || !best) { free(w); free(best); return OR_NOMEM; }
  for (uint64_t j = 0; j < n; ++j) {
    if (!deficient[j]) continue;
    double best_norm = -1.0;
    for (uint64_t cand = 0; cand < m; ++cand) {
      memset(w, 0, m * sizeof(double));
      w[cand] = 1.0;
      for (int pass = 0; pass < 2; ++pass) {
        for (uint64_t c = 0; c < n; ++c) {
          if (deficient[c] && c >= j) continue;
          const double *uc = ccol(u, c);
          const double proj = dot_n(uc, w, m);
          for (uint64_t i = 0; i < m; ++i) w[i] -= proj * uc[i];
        }
      }
      const double wn = sqrt(dot_n(w, w, m));
      if (wn > 0.5) { best_norm = wn; memcpy(best, w, m * sizeof(double)); break; }
      if (wn > best_norm) { best_norm = wn; memcpy(best, w, m * sizeof(double)); }
    }
    if (!(best_norm > 0.0)) {
      free(w); free(best);
      res->residual = best_norm;
      set_err(res, OR_CONVERGE, "orthonormal completion has no independent direction");
      return OR_CONVERGE;
    }
    double *uj = ccol(u, j);
    for (uint64_t i = 0; i < m; ++i) uj[i] = best[i] / best_norm;
    if (best_norm <= 0.5) {
      for (uint64_t c = 0; c < n; ++c) {
        if (deficient[c] && c >= j) continue;
        const double *uc = ccol(u, c);
        const double proj = dot_n(uc, uj, m);
        for (uint64_t i = 0; i < m; ++i) uj[i] -= proj * uc[i];
      }
      const double wn = sqrt(dot_n(uj, uj, m));
      for (uint64_t i = 0; i < m; ++i) uj[i] /= wn;
    }
  }
  free(w); free(best);
  return OR_OK;
}

typedef struct { cmat u; double *sigma; cmat v; } jac_out;

/* stable descending order of sigma (std::stable_sort with `>`) */
static void stable_desc(const double *s, uint64_t *order, uint64_t n) {
  for (uint64_t i = 0; i < n; ++i) order[i] = i;
  for (uint64_t i = 1; i < n; ++i) { /* insertion sort is stable */
    uint64_t x = order[i];
    uint64_t j = i;
    while (j > 0 && s[order[j - 1]] < s[x]) { order[j] = order[j - 1]; --j; }
    order[j] = x;
  }
}

/* jacobi_svd -- svd.cpp:214-306 (b is consumed) */
static int jacobi(cmat *b, int build_u, jac_out *out, or_result *res) {
  const uint64_t m = b->rows, n = b->cols;
  cmat v;
  if (cmat_alloc(&v, n, n) != OR_OK) return OR_NOMEM;
  for (uint64_t i = 0; i < n; ++i) v.d[i * n + i] = 1.0;
  double *alpha = (double *)calloc(n ? n : 1, sizeof(double));
  if (!alpha) return OR_NOMEM;
  double last_max_ratio = 0.0;
  int converged = n < 2;
  for (int sweep = 0; sweep < kMaxSweeps && !converged; ++sweep) {
    double alpha_max = 0.0;
    for (uint64_t j = 0; j < n; ++j) {
      alpha[j] = dot_n(ccol(b, j), ccol(b, j), m);
      if (alpha[j] > alpha_max) alpha_max = alpha[j];
    }
    const double freeze = kJacobiTol * kJacobiTol * alpha_max;
    uint64_t rotations = 0;
    double max_ratio = 0.0;
    for (uint64_t p = 0; p + 1 < n; ++p) {
      for (uint64_t q = p + 1; q < n; ++q) {
        if (alpha[p] <= freeze || alpha[q] <= freeze) continue;
        double *bp = ccol(b, p), *bq = ccol(b, q);
        const double gamma = dot_n(bp, bq, m);
        const double ratio = fabs(gamma) / sqrt(alpha[p] * alpha[q]);
        if (ratio > max_ratio) max_ratio = ratio;
        if (ratio <= kJacobiTol) continue;
        const double zeta = (alpha[q] - alpha[p]) / (2.0 * gamma);
        const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / sqrt(1.0 + t * t);
        const double s = c * t;
        for (uint64_t i = 0; i < m; ++i) {
          const double xp = bp[i], xq = bq[i];
          bp[i] = c * xp - s * xq;
          bq[i] = s * xp + c * xq;
        }
        double *vp = ccol(&v, p), *vq = ccol(&v, q);
        for (uint64_t i = 0; i < n; ++i) {
          const double xp = vp[i], xq = vq[i];
          vp[i] = c * xp - s * xq;
          vq[i] = s * xp + c * xq;
        }
        const double ap = alpha[p], aq = alpha[q];
        double na = c * c * ap - 2.0 * c * s * gamma + s * s * aq;
        double nq = s * s * ap + 2.0 * c * s * gamma + c * c * aq;
        alpha[p] = na > 0.0 ? na : 0.0;
        alpha[q] = nq > 0.0 ? nq : 0.0;
        ++rotations;
      }
    }
    last_max_ratio = max_ratio;
    if (rotations == 0) converged = 1;
  }
  free(alpha);
  if (!converged) {
    free(v.d);
    res->residual = last_max_ratio;
    set_err(res, OR_CONVERGE, "one-sided Jacobi did not converge");
    return OR_CONVERGE;
  }
  double *sig = (double *)calloc(n ? n : 1, sizeof(double));
  uint64_t *order = (uint64_t *)calloc(n ? n : 1, sizeof(uint64_t));
  for (uint64_t j = 0; j < n; ++j) sig[j] = sqrt(dot_n(ccol(b, j), ccol(b, j), m));
  stable_desc(sig, order, n);
  out->sigma = (double *)calloc(n ? n : 1, sizeof(double));
  cmat_alloc(&out->v, n, n);
  for (uint64_t j = 0; j < n; ++j) {
    out->sigma[j] = sig[order[j]];
    memcpy(ccol(&out->v, j), ccol(&v, order[j]), n * sizeof(double));
  }
  free(v.d);
  out->u.d = NULL;
  int st = OR_OK;
  if (build_u) {
    const double smax = n ? out->sigma[0] : 0.0;
    const double threshold = kRankTol * smax;
    cmat_alloc(&out->u, m, n);
    unsigned char *def = (unsigned char *)calloc(n ? n : 1, 1);
    for (uint64_t j = 0; j < n; ++j) {
      const double s = out->sigma[j];
      if (s > threshold && s > 0.0) {
        const double *src = ccol(b, order[j]);
        double *dst = ccol(&out->u, j);
        for (uint64_t i = 0; i < m; ++i) dst[i] = src[i] / s;
      } else {
        def[j] = 1;
      }
    }
    st = complete_columns(&out->u, def, res);
    free(def);
  }
  free(sig); free(order);
  return st;
}

typedef struct { cmat u; double *sigma; cmat v; } tall_out;

/* svd_tall -- svd.cpp:316-332 (b consumed) */
static int svd_tall(cmat *b, int want_u, tall_out *out, or_result *res) {
  memset(out, 0, sizeof *out);
  if (b->rows > b->cols) {
    cmat vs;
    if (cmat_alloc(&vs, b->rows, b->cols) != OR_OK) return OR_NOMEM;
    double *betas = (double *)calloc(b->cols ? b->cols : 1, sizeof(double));
    householder(b, &vs, betas);
    cmat r; /* extract_r, svd.cpp:134-143 */
    cmat_alloc(&r, b->cols, b->cols);
    for (uint64_t j = 0; j < b->cols; ++j)
      for (uint64_t i = 0; i <= j; ++i) ccol(&r, j)[i] = ccol(b, j)[i];
    jac_out j;
    memset(&j, 0, sizeof j);
    int st = jacobi(&r, want_u, &j, res);
    free(r.d);
    if (st == OR_OK) {
      out->sigma = j.sigma; out->v = j.v;
      if (want_u) st = apply_q(&vs, betas, b->rows, &j.u, &out->u);
    }
    free(j.u.d);
    free(vs.d); free(betas);
    return st;
  }
  jac_out j;
  memset(&j, 0, sizeof j);
  int st = jacobi(b, want_u, &j, res);
  if (st == OR_OK) { out->sigma = j.sigma; out->v = j.v; out->u = j.u; }
  return st;
}

/* apply_sign_convention -- svd.cpp:336-354 on row-major u (rows x cols) */
static void sign_convention(double *u, uint64_t rows, uint64_t cols, double *v, uint64_t vrows) {
  for (uint64_t j = 0; j < cols; ++j) {
    uint64_t arg = 0;
    double best = -1.0;
    for (uint64_t i = 0; i < rows; ++i) {
      const double mag = fabs(u[i * cols + j]);
      if (mag > best) { best = mag; arg = i; }
    }
    if (rows && u[arg * cols + j] < 0.0) {
      for (uint64_t i = 0; i < rows; ++i) u[i * cols + j] = -u[i * cols + j];
      if (v)
        for (uint64_t i = 0; i < vrows; ++i) v[i * cols + j] = -v[i * cols + j];
    }
  }
}

static int all_finite(const double *x, uint64_t n) {
  for (uint64_t i = 0; i < n; ++i) if (!isfinite(x[i])) return 0;
  return 1;
}

/* colmat_of -- svd.cpp:39-49 from row-major a (rows x cols) */
static int colmat_of(const double *a, uint64_t rows, uint64_t cols, int transpose, cmat *out) {
  if (cmat_alloc(out, transpose ? cols : rows, transpose ? rows : cols) != OR_OK) return OR_NOMEM;
  for (uint64_t r = 0; r < rows; ++r)
    for (uint64_t c = 0; c < cols; ++c) {
      if (transpose) ccol(out, r)[c] = a[r * cols + c];
      else ccol(out, c)[r] = a[r * cols + c];
    }
  return OR_OK;
}

/* row-major copy of a colmat -- dense_of_colmat, svd.cpp:51-58 */
static double *rowmajor_of(const cmat *a) {
  double *o = (double *)calloc(a->rows * a->cols ? a->rows * a->cols : 1, sizeof(double));
  for (uint64_t c = 0; c < a->cols; ++c)
    for (uint64_t r = 0; r < a->rows; ++r) o[r * a->cols + c] = ccol(a, c)[r];
  return o;
}

/* dense_svd -- svd.cpp:365-379 */
static int dense_svd_into(const double *a, uint64_t rows, uint64_t cols, or_result *res) {
  if (!all_finite(a, rows * cols)) {
    set_err(res, OR_INVALID, "dense_svd: input has non-finite values");
    return OR_INVALID;
  }
  const uint64_t k = rows < cols ? rows : cols;
  res->has_v = 1;
  if (k == 0) {
    res->u_rows = rows; res->u_cols = 0; res->n_sigma = 0;
    res->v_rows = cols; res->v_cols = 0;
    return OR_OK;
  }
  const int transposed = rows < cols;
  cmat b;
  if (colmat_of(a, rows, cols, transposed, &b) != OR_OK) return OR_NOMEM;
  tall_out t;
  int st = svd_tall(&b, 1, &t, res);
  free(b.d);
  if (st != OR_OK) { free(t.u.d); free(t.v.d); free(t.sigma); return st; }
  const cmat *uu = transposed ? &t.v : &t.u;
  const cmat *vv = transposed ? &t.u : &t.v;
  res->u = rowmajor_of(uu); res->u_rows = uu->rows; res->u_cols = uu->cols;
  res->vm = rowmajor_of(vv); res->v_rows = vv->rows; res->v_cols = vv->cols;
  res->sigma = t.sigma; res->n_sigma = k;
  sign_convention(res->u, res->u_rows, res->u_cols, res->vm, res->v_rows);
  free(t.u.d); free(t.v.d);
  return OR_OK;
}

or_result *or_dense_svd(uint64_t rows, uint64_t cols, const double *a) {
  or_result *res = new_result();
  dense_svd_into(a, rows, cols, res);
  return res;
}

/* block_svd -- svd.cpp:381-400. The block arrives as sorted COO. */
static int block_svd_into(uint64_t rows, uint64_t cols, uint64_t nnz, const uint64_t *r,
                          const uint64_t *c, const double *v, uint64_t keep, or_result *res) {
  if (keep == 0) { set_err(res, OR_INVALID, "block_svd: keep must be >= 1"); return OR_INVALID; }
  const uint64_t count = rows * cols; /* dense_of, dense_matrix.cpp:62-75 */
  if (rows != 0 && count / rows != cols) {
    set_err(res, OR_INVALID, "dense_of: dimension overflow");
    return OR_INVALID;
  }
  if (count > kDensifyCap) {
    char msg[160];
    snprintf(msg, sizeof msg, "dense_of: %llux%llu exceeds the densification cap",
             (unsigned long long)rows, (unsigned long long)cols);
    set_err(res, OR_INVALID, msg);
    return OR_INVALID;
  }
  double *dense = (double *)calloc(count ? count : 1, sizeof(double));
  if (!dense) return OR_NOMEM;
  for (uint64_t i = 0; i < nnz; ++i) dense[r[i] * cols + c[i]] = v[i];
  if (!all_finite(dense, count)) {
    free(dense);
    set_err(res, OR_INVALID, "block_svd: block has non-finite values");
    return OR_INVALID;
  }
  const uint64_t k_full = rows < cols ? rows : cols;
  res->has_v = 0;
  if (k_full == 0) { free(dense); res->u_rows = rows; res->u_cols = 0; res->n_sigma = 0; return OR_OK; }
  const uint64_t k = keep < k_full ? keep : k_full;
  const int transposed = rows < cols;
  cmat b;
  colmat_of(dense, rows, cols, transposed, &b);
  free(dense);
  tall_out t;
  int st = svd_tall(&b, !transposed, &t, res);
  free(b.d);
  if (st != OR_OK) { free(t.u.d); free(t.v.d); free(t.sigma); return st; }
  const cmat *uu = transposed ? &t.v : &t.u;
  double *u = rowmajor_of(uu);
  sign_convention(u, uu->rows, uu->cols, NULL, 0);
  res->u_rows = uu->rows; res->u_cols = k;
  res->u = (double *)calloc(uu->rows * k ? uu->rows * k : 1, sizeof(double));
  for (uint64_t i = 0; i < uu->rows; ++i)
    for (uint64_t j = 0; j < k; ++j) res->u[i * k + j] = u[i * uu->cols + j];
  res->n_sigma = k;
  res->sigma = t.sigma; /* first k of min(rows,cols) entries are the kept ones */
  free(u); free(t.u.d); free(t.v.d);
  return OR_OK;
}

or_result *or_block_svd(uint64_t rows, uint64_t cols, uint64_t nnz, const uint64_t *r,
                        const uint64_t *c, const double *v, uint64_t keep) {
  or_result *res = new_result();
  block_svd_into(rows, cols, nnz, r, c, v, keep, res);
  return res;
}

/* recover_right_vectors -- proj/src/proxy.cpp:48-72 */
or_result *or_recover_right_vectors(uint64_t rows, uint64_t cols, uint64_t nnz, const uint64_t *r,
                                    const uint64_t *c, const double *v, const double *u,
                                    uint64_t u_rows, uint64_t u_cols, const double *sigma,
                                    uint64_t n_sigma, double tol) {
  or_result *res = new_result();
  if (u_rows != rows || u_cols != n_sigma) {
    set_err(res, OR_INVALID, "recover_right_vectors: factor shapes disagree");
    return res;
  }
  double smax = 0.0;
  for (uint64_t j = 0; j < n_sigma; ++j) if (sigma[j] > smax) smax = sigma[j];
  uint64_t *ret = (uint64_t *)malloc((n_sigma ? n_sigma : 1) * sizeof(uint64_t));
  uint64_t nr = 0;
  for (uint64_t j = 0; j < n_sigma; ++j)
    if (sigma[j] > tol * smax && sigma[j] > 0.0) ret[nr++] = j;
  res->v_rows = cols; res->v_cols = nr; res->has_v = 1;
  res->vm = (double *)calloc(cols * nr ? cols * nr : 1, sizeof(double));
  if (!res->vm) { free(ret); set_err(res, OR_NOMEM, "oom"); return res; }
  for (uint64_t e = 0; e < nnz; ++e) {
    double *vr = res->vm + c[e] * nr;
    const double *ur = u + r[e] * u_cols;
    for (uint64_t jj = 0; jj < nr; ++jj) vr[jj] += v[e] * ur[ret[jj]];
  }
  for (uint64_t jj = 0; jj < nr; ++jj) {
    const double inv = 1.0 / sigma[ret[jj]];
    for (uint64_t i = 0; i < cols; ++i) res->vm[i * nr + jj] *= inv;
  }
  free(ret);
  return res;
}

/* ------------------------------------------------------------------------ */
/* run_pipeline -- proj/src/pipeline.cpp:61-121 (workers = 1: output is      */
/* worker-invariant in the reference, so the single-thread order is exact)   */

#include <time.h>
static double now_s(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

or_result *or_run_pipeline(uint64_t rows, uint64_t cols, uint64_t nnz, const uint64_t *r,
                           const uint64_t *c, const double *v, uint64_t D, int method,
                           uint64_t keep, uint64_t seed, uint64_t workers) {
  or_result *res = new_result();
  if (workers == 0) { set_err(res, OR_INVALID, "workers must be >= 1"); return res; }
  if (!partition_ok(cols, D, res)) return res;
  double t0 = now_s();
  coo_view a;
  coo_open(&a, rows, cols, nnz, r, c, v);
  if (repair_into(&a, D, method, seed, res) != OR_OK) { coo_close(&a); return res; }
  coo_close(&a);
  double t1 = now_s();
  /* repaired matrix is in res->r/c/v (sorted by row, col) */
  res->n_records = D;
  res->rec_kept = (uint32_t *)calloc(D, sizeof(uint32_t));
  uint64_t total_cols = 0;
  double **payloads = (double **)calloc(D, sizeof(double *));
  uint64_t *bidx = (uint64_t *)malloc((res->nnz ? res->nnz : 1) * sizeof(uint64_t));
  for (uint64_t d = 0; d < D; ++d) {
    const uint64_t b = range_begin(cols, D, d), e = range_end(cols, D, d);
    /* block_view -- partition.cpp:53-62 (entries stay in (row, col) order) */
    uint64_t n = 0;
    uint64_t *br = (uint64_t *)malloc((res->nnz ? res->nnz : 1) * sizeof(uint64_t));
    uint64_t *bc = (uint64_t *)malloc((res->nnz ? res->nnz : 1) * sizeof(uint64_t));
    double *bv = (double *)malloc((res->nnz ? res->nnz : 1) * sizeof(double));
    for (uint64_t i = 0; i < res->nnz; ++i)
      if (res->c[i] >= b && res->c[i] < e) { br[n] = res->r[i]; bc[n] = res->c[i] - b; bv[n] = res->v[i]; ++n; }
    /* run_block_task -- pipeline.cpp:11-16 */
    const uint64_t k_full = rows < (e - b) ? rows : (e - b);
    const uint64_t kk = keep == 0 ? k_full : (keep < k_full ? keep : k_full);
    or_result *br_res = new_result();
    block_svd_into(rows, e - b, n, br, bc, bv, kk, br_res);
    free(br); free(bc); free(bv);
    if (br_res->status != OR_OK) {
      char msg[700];
      snprintf(msg, sizeof msg, "block task %llu failed: %s", (unsigned long long)d, br_res->message);
      res->status = OR_OK;
      set_err(res, OR_RUNTIME, msg);
      or_free(br_res);
      for (uint64_t q = 0; q < D; ++q) free(payloads[q]);
      free(payloads); free(bidx);
      return res;
    }
    /* make_block_record -- block_record.cpp:69-84 */
    const uint64_t kept = br_res->u_cols;
    res->rec_kept[d] = (uint32_t)kept;
    payloads[d] = (double *)calloc(rows * kept ? rows * kept : 1, sizeof(double));
    for (uint64_t i = 0; i < rows; ++i)
      for (uint64_t j = 0; j < kept; ++j)
        payloads[d][i * kept + j] = br_res->u[i * kept + j] * br_res->sigma[j];
    total_cols += kept;
    or_free(br_res);
  }
  free(bidx);
  double t2 = now_s();
  /* proxy_from_records -- pipeline.cpp:18-59 (already in block order) */
  res->rec_payload = (double *)calloc(rows * total_cols ? rows * total_cols : 1, sizeof(double));
  double *P = (double *)calloc(rows * total_cols ? rows * total_cols : 1, sizeof(double));
  uint64_t off = 0, poff = 0;
  for (uint64_t d = 0; d < D; ++d) {
    const uint64_t kept = res->rec_kept[d];
    memcpy(res->rec_payload + poff, payloads[d], rows * kept * sizeof(double));
    poff += rows * kept;
    for (uint64_t i = 0; i < rows; ++i)
      for (uint64_t j = 0; j < kept; ++j) P[i * total_cols + off + j] = payloads[d][i * kept + j];
    off += kept;
    free(payloads[d]);
  }
  free(payloads);
  /* proxy_svd -> dense_svd -- proxy.cpp:40-46; V of P is dropped (pipeline.cpp:112) */
  dense_svd_into(P, rows, total_cols, res);
  free(P);
  free(res->vm); res->vm = NULL; res->has_v = 0; res->v_rows = res->v_cols = 0;
  double t3 = now_s();
  res->t_repair = t1 - t0; res->t_blocks = t2 - t1; res->t_proxy = t3 - t2;
  return res;
}

/* synth_bipartite -- proj/src/synth.cpp:14-29 (Bernoulli cells, value 1.0).
 * Two-call protocol: with out arrays NULL it only counts. */
uint64_t or_synth_bipartite(uint64_t rows, uint64_t cols, double density, uint64_t seed,
                            uint64_t *r, uint64_t *c, double *v) {
  uint64_t n = 0;
  for (uint64_t row = 0; row < rows; ++row) {
    keyed_rng g = rng_make(seed, 0x53594e5448ull, row);
    for (uint64_t col = 0; col < cols; ++col) {
      if (rng_unit(&g) < density) {
        if (r) { r[n] = row; c[n] = col; v[n] = 1.0; }
        ++n;
      }
    }
  }
  return n;
}
