/*
 * gen.c -- deterministic synthetic inputs for the five BASELINE.json configs.
 *
 * The reference ships only synth_bipartite (Bernoulli cells of value 1.0,
 * proj/src/synth.cpp:14-29); none of the BASELINE configs (real values, Zipf
 * column degrees, planted empty rows, planted spectrum) can be produced by it,
 * so the workloads are defined here, once, and fed byte-identically to the GPU
 * path and to the CPU oracles. All draws come from the reference's KeyedRng
 * (splitmix64 keyed by (seed, tag, index)), so a config is a pure function of
 * its parameters. Outputs are entry arrays sorted by (row, col) -- the layout of
 * ranky::Entry / rk_entry. Not part of the timed path.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct { uint64_t row, col; double value; } rkg_entry;

static uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
typedef struct { uint64_t s; } rng_t;
static rng_t rng_make(uint64_t seed, uint64_t a, uint64_t b) {
  rng_t g;
  g.s = mix64(seed + 0x9e3779b97f4a7c15ull);
  g.s = mix64(g.s ^ (a + 0xbf58476d1ce4e5b9ull));
  g.s = mix64(g.s ^ (b + 0x94d049bb133111ebull));
  return g;
}
static uint64_t rng_next(rng_t* g) { g->s += 0x9e3779b97f4a7c15ull; return mix64(g->s); }
static double rng_unit(rng_t* g) { return (double)(rng_next(g) >> 11) * 0x1.0p-53; }
static uint64_t rng_below(rng_t* g, uint64_t bound) {
  const uint64_t t = (0 - bound) % bound;
  for (;;) { uint64_t r = rng_next(g); if (r >= t) return r % bound; }
}

enum { VAL_ONE = 0, VAL_UNIFORM_PM1 = 1, VAL_NORMAL = 2, VAL_UNIFORM_01 = 3 };
enum { TAG_POS = 0x504f53, TAG_PLANT = 0x504c4e54, TAG_COL = 0x434f4c, TAG_ZIPF = 0x5a495046 };

static double draw_value(rng_t* g, int kind) {
  for (;;) {
    double x;
    switch (kind) {
      case VAL_UNIFORM_PM1: x = 2.0 * rng_unit(g) - 1.0; break;
      case VAL_NORMAL: {  /* Box-Muller, first variate */
        double u1 = rng_unit(g), u2 = rng_unit(g);
        if (u1 <= 0.0) continue;
        x = sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
        break;
      }
      case VAL_UNIFORM_01: x = rng_unit(g); break;
      default: x = 1.0;
    }
    if (x != 0.0) return x;
  }
}

typedef struct { rkg_entry* e; uint64_t n, cap; } vec_t;
static int push(vec_t* v, uint64_t r, uint64_t c, double x) {
  if (v->n == v->cap) {
    uint64_t cap = v->cap ? v->cap * 2 : 1024;
    rkg_entry* p = (rkg_entry*)realloc(v->e, cap * sizeof(rkg_entry));
    if (!p) return -1;
    v->e = p; v->cap = cap;
  }
  v->e[v->n].row = r; v->e[v->n].col = c; v->e[v->n].value = x;
  v->n++;
  return 0;
}

void rkg_free(void* p) { free(p); }

/* Uniform positions with density p per cell (row-wise geometric skipping),
 * values of `kind`; then `plant_blocks` distinct blocks of the D-block column
 * partition get `plant_rows` distinct rows emptied inside the block. */
rkg_entry* rkg_uniform(uint64_t rows, uint64_t cols, double density, int kind, uint64_t seed, uint64_t D,
                       uint64_t plant_blocks, uint64_t plant_rows, uint64_t* n_out) {
  vec_t v = {0, 0, 0};
  const double lq = log1p(-density);
  /* planted (block, row) pairs */
  uint64_t* pb = NULL; uint64_t* pr = NULL; uint64_t np = 0;
  if (plant_blocks && D) {
    pb = (uint64_t*)calloc(plant_blocks * plant_rows + 1, 8);
    pr = (uint64_t*)calloc(plant_blocks * plant_rows + 1, 8);
    uint64_t* blocks = (uint64_t*)calloc(plant_blocks + 1, 8);
    rng_t g = rng_make(seed, TAG_PLANT, 0);
    for (uint64_t i = 0; i < plant_blocks; ++i) {
      for (;;) {
        uint64_t b = rng_below(&g, D), dup = 0;
        for (uint64_t q = 0; q < i; ++q) dup |= blocks[q] == b;
        if (!dup) { blocks[i] = b; break; }
      }
      uint64_t first = np;
      for (uint64_t k = 0; k < plant_rows && k < rows; ++k) {
        for (;;) {
          uint64_t r = rng_below(&g, rows), dup = 0;
          for (uint64_t q = first; q < np; ++q) dup |= pr[q] == r;
          if (!dup) { pb[np] = blocks[i]; pr[np] = r; ++np; break; }
        }
      }
    }
    free(blocks);
  }
  const uint64_t width = D ? cols / D : cols;
  for (uint64_t r = 0; r < rows; ++r) {
    rng_t g = rng_make(seed, TAG_POS, r);
    int64_t c = -1;
    for (;;) {
      const double u = rng_unit(&g);
      const double gap = floor(log1p(-u) / lq);
      if (!(gap < (double)cols)) break;
      c += (int64_t)gap + 1;
      if ((uint64_t)c >= cols) break;
      const double x = draw_value(&g, kind);
      int planted = 0;
      if (np) {
        uint64_t d = (uint64_t)c / width;
        if (d >= D) d = D - 1;
        for (uint64_t q = 0; q < np; ++q) planted |= (pb[q] == d && pr[q] == r);
      }
      if (!planted && push(&v, r, (uint64_t)c, x)) { free(v.e); free(pb); free(pr); return NULL; }
    }
  }
  free(pb); free(pr);
  *n_out = v.n;
  return v.e;
}

/* Zipf column degrees: a column is nonempty with probability p_nonempty; a
 * nonempty column's degree k in [1, rows] has P(k) ~ k^-s; its rows are k
 * distinct uniform rows; values of `kind`. Entries are returned (row, col)-sorted. */
rkg_entry* rkg_zipf(uint64_t rows, uint64_t cols, double p_nonempty, double s, int kind, uint64_t seed,
                    uint64_t* n_out) {
  double* cdf = (double*)malloc((rows + 1) * sizeof(double));
  double z = 0.0;
  for (uint64_t k = 1; k <= rows; ++k) { z += pow((double)k, -s); cdf[k] = z; }
  for (uint64_t k = 1; k <= rows; ++k) cdf[k] /= z;
  vec_t v = {0, 0, 0};
  unsigned char* mark = (unsigned char*)calloc(rows, 1);
  uint64_t* pick = (uint64_t*)malloc(rows * sizeof(uint64_t));
  for (uint64_t c = 0; c < cols; ++c) {
    rng_t g = rng_make(seed, TAG_COL, c);
    if (!(rng_unit(&g) < p_nonempty)) continue;
    const double u = rng_unit(&g);
    uint64_t lo = 1, hi = rows;  /* smallest k with cdf[k] > u */
    while (lo < hi) { uint64_t mid = (lo + hi) / 2; if (cdf[mid] > u) hi = mid; else lo = mid + 1; }
    const uint64_t k = lo;
    uint64_t n = 0;
    if (k == rows) {
      for (uint64_t r = 0; r < rows; ++r) pick[n++] = r;
    } else {
      while (n < k) {
        uint64_t r = rng_below(&g, rows);
        if (!mark[r]) { mark[r] = 1; pick[n++] = r; }
      }
      for (uint64_t q = 0; q < n; ++q) mark[pick[q]] = 0;
    }
    for (uint64_t q = 0; q < n; ++q) push(&v, pick[q], c, draw_value(&g, kind));
  }
  free(cdf); free(mark); free(pick);
  /* counting sort by row (stable: columns stay ascending within a row) */
  uint64_t* cnt = (uint64_t*)calloc(rows + 1, sizeof(uint64_t));
  for (uint64_t i = 0; i < v.n; ++i) cnt[v.e[i].row + 1]++;
  for (uint64_t r = 0; r < rows; ++r) cnt[r + 1] += cnt[r];
  rkg_entry* out = (rkg_entry*)malloc((v.n ? v.n : 1) * sizeof(rkg_entry));
  for (uint64_t i = 0; i < v.n; ++i) out[cnt[v.e[i].row]++] = v.e[i];
  free(cnt); free(v.e);
  *n_out = v.n;
  return out;
}

/* mean degree of the Zipf(s) law on [1, rows] (for calibrating p_nonempty) */
double rkg_zipf_mean(uint64_t rows, double s) {
  double z = 0.0, m = 0.0;
  for (uint64_t k = 1; k <= rows; ++k) { double w = pow((double)k, -s); z += w; m += w * (double)k; }
  return m / z;
}

/* synth_bipartite -- proj/src/synth.cpp:14-29 (Bernoulli per cell, value 1.0) */
rkg_entry* rkg_synth_bipartite(uint64_t rows, uint64_t cols, double density, uint64_t seed, uint64_t* n_out) {
  vec_t v = {0, 0, 0};
  for (uint64_t r = 0; r < rows; ++r) {
    rng_t g = rng_make(seed, 0x53594e5448ull, r);
    for (uint64_t c = 0; c < cols; ++c)
      if (rng_unit(&g) < density) push(&v, r, c, 1.0);
  }
  *n_out = v.n;
  return v.e;
}

/* ---------------------------------------------------------------------------
 * c5: planted spectrum. P (rows x k) and Q (cols x k) have orthonormal columns,
 * obtained from seeded Gaussians by Cholesky QR (Q = G R^-1 with R = chol(G^T G);
 * P the same, twice); sigma_j = decay^j. A = mask o (P diag(sigma) Q^T) + noise *
 * N(0,1) on the nonzeros, the mask being uniform positions of the given density.
 * Since Q_c = G_c R^-1, A_ic = G_c . H_i with H = P diag(sigma) R^-T, so Q is
 * never stored: row c of G is regenerated from KeyedRng(seed, 'Q', c) for every
 * nonzero of column c. G^T G is accumulated over fixed chunks of rows and summed
 * in chunk order, so the result does not depend on the number of threads.
 * ------------------------------------------------------------------------- */
enum { TAG_P = 0x50, TAG_Q = 0x51, TAG_NOISE = 0x4e4f4953 };

static void gauss_row(uint64_t seed, uint64_t tag, uint64_t idx, uint64_t k, double* out) {
  rng_t g = rng_make(seed, tag, idx);
  for (uint64_t j = 0; j < k; j += 2) {
    double u1, u2;
    do { u1 = rng_unit(&g); } while (u1 <= 0.0);
    u2 = rng_unit(&g);
    const double r = sqrt(-2.0 * log(u1));
    out[j] = r * cos(6.283185307179586 * u2);
    if (j + 1 < k) out[j + 1] = r * sin(6.283185307179586 * u2);
  }
}

/* in place: S (k x k, row-major, symmetric positive definite) -> upper R, S = R^T R */
static int chol_upper(double* S, uint64_t k) {
  for (uint64_t i = 0; i < k; ++i) {
    double d = S[i * k + i];
    for (uint64_t p = 0; p < i; ++p) d -= S[p * k + i] * S[p * k + i];
    if (!(d > 0.0)) return -1;
    d = sqrt(d);
    S[i * k + i] = d;
    for (uint64_t j = i + 1; j < k; ++j) {
      double x = S[i * k + j];
      for (uint64_t p = 0; p < i; ++p) x -= S[p * k + i] * S[p * k + j];
      S[i * k + j] = x / d;
    }
    for (uint64_t j = 0; j < i; ++j) S[i * k + j] = 0.0;
  }
  return 0;
}

/* inverse of an upper-triangular R (row-major), in place */
static void inv_upper(double* R, uint64_t k) {
  double* X = (double*)calloc(k * k, sizeof(double));
  for (uint64_t j = 0; j < k; ++j) {  /* column j of R^-1: solve R x = e_j */
    for (int64_t i = (int64_t)j; i >= 0; --i) {
      double s = (i == (int64_t)j) ? 1.0 : 0.0;
      for (uint64_t p = (uint64_t)i + 1; p <= j; ++p) s -= R[i * k + p] * X[p * k + j];
      X[i * k + j] = s / R[i * k + i];
    }
  }
  memcpy(R, X, k * k * sizeof(double));
  free(X);
}

/* Gram of the Gaussian rows [0, n) of stream `tag`: chunked, deterministic */
static void gauss_gram(uint64_t seed, uint64_t tag, uint64_t n, uint64_t k, double* S) {
  const uint64_t chunk = 1ull << 15;
  const uint64_t nc = (n + chunk - 1) / chunk;
  double* part = (double*)calloc(nc * k * k, sizeof(double));
#pragma omp parallel for schedule(dynamic, 4)
  for (int64_t c = 0; c < (int64_t)nc; ++c) {
    double* row = (double*)malloc(k * sizeof(double));
    double* acc = part + (uint64_t)c * k * k;
    const uint64_t r1 = ((uint64_t)c + 1) * chunk < n ? ((uint64_t)c + 1) * chunk : n;
    for (uint64_t r = (uint64_t)c * chunk; r < r1; ++r) {
      gauss_row(seed, tag, r, k, row);
      for (uint64_t i = 0; i < k; ++i) {
        const double x = row[i];
        for (uint64_t j = i; j < k; ++j) acc[i * k + j] += x * row[j];
      }
    }
    free(row);
  }
  memset(S, 0, k * k * sizeof(double));
  for (uint64_t c = 0; c < nc; ++c)
    for (uint64_t i = 0; i < k; ++i)
      for (uint64_t j = i; j < k; ++j) S[i * k + j] += part[c * k * k + i * k + j];
  for (uint64_t i = 0; i < k; ++i)
    for (uint64_t j = 0; j < i; ++j) S[i * k + j] = S[j * k + i];
  free(part);
}

rkg_entry* rkg_planted(uint64_t rows, uint64_t cols, double density, uint64_t k, double decay, double noise,
                       uint64_t seed, uint64_t* n_out) {
  *n_out = 0;
  if (k == 0 || k > rows || k > cols) return NULL;
  /* P: rows x k, orthonormal columns (Cholesky QR applied twice) */
  double* P = (double*)malloc(rows * k * sizeof(double));
  for (uint64_t r = 0; r < rows; ++r) gauss_row(seed, TAG_P, r, k, P + r * k);
  double* S = (double*)malloc(k * k * sizeof(double));
  double* T = (double*)malloc(rows * k * sizeof(double));
  for (int pass = 0; pass < 2; ++pass) {
    memset(S, 0, k * k * sizeof(double));
    for (uint64_t r = 0; r < rows; ++r)
      for (uint64_t i = 0; i < k; ++i)
        for (uint64_t j = 0; j < k; ++j) S[i * k + j] += P[r * k + i] * P[r * k + j];
    if (chol_upper(S, k)) { free(P); free(S); free(T); return NULL; }
    inv_upper(S, k);
    for (uint64_t r = 0; r < rows; ++r)
      for (uint64_t j = 0; j < k; ++j) {
        double x = 0.0;
        for (uint64_t i = 0; i <= j; ++i) x += P[r * k + i] * S[i * k + j];
        T[r * k + j] = x;
      }
    memcpy(P, T, rows * k * sizeof(double));
  }
  free(T);
  /* Q = G R^-1 with G^T G = R^T R */
  gauss_gram(seed, TAG_Q, cols, k, S);
  if (chol_upper(S, k)) { free(P); free(S); return NULL; }
  inv_upper(S, k); /* S = R^-1 (upper) */
  /* H = P diag(sigma) R^-T : H[i][l] = sum_j Rinv[l][j] sigma_j P[i][j] */
  double* H = (double*)calloc(rows * k, sizeof(double));
  double sig = 1.0;
  double* sigma = (double*)malloc(k * sizeof(double));
  for (uint64_t j = 0; j < k; ++j) { sigma[j] = sig; sig *= decay; }
  for (uint64_t i = 0; i < rows; ++i)
    for (uint64_t l = 0; l < k; ++l) {
      double x = 0.0;
      for (uint64_t j = l; j < k; ++j) x += S[l * k + j] * sigma[j] * P[i * k + j];
      H[i * k + l] = x;
    }
  free(P); free(S); free(sigma);
  /* mask positions per row (geometric skipping); counts first, then values */
  const double lq = log1p(-density);
  uint64_t* cnt = (uint64_t*)calloc(rows + 1, sizeof(uint64_t));
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t r = 0; r < (int64_t)rows; ++r) {
    rng_t g = rng_make(seed, TAG_POS, (uint64_t)r);
    int64_t c = -1;
    uint64_t n = 0;
    for (;;) {
      const double gap = floor(log1p(-rng_unit(&g)) / lq);
      if (!(gap < (double)cols)) break;
      c += (int64_t)gap + 1;
      if ((uint64_t)c >= cols) break;
      ++n;
    }
    cnt[r + 1] = n;
  }
  for (uint64_t r = 0; r < rows; ++r) cnt[r + 1] += cnt[r];
  const uint64_t nnz = cnt[rows];
  rkg_entry* out = (rkg_entry*)malloc((nnz ? nnz : 1) * sizeof(rkg_entry));
  if (!out) { free(H); free(cnt); return NULL; }
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t r = 0; r < (int64_t)rows; ++r) {
    rng_t g = rng_make(seed, TAG_POS, (uint64_t)r);
    rng_t gn = rng_make(seed, TAG_NOISE, (uint64_t)r);
    double* grow = (double*)malloc(k * sizeof(double));
    const double* h = H + (uint64_t)r * k;
    int64_t c = -1;
    uint64_t o = cnt[r];
    for (;;) {
      const double gap = floor(log1p(-rng_unit(&g)) / lq);
      if (!(gap < (double)cols)) break;
      c += (int64_t)gap + 1;
      if ((uint64_t)c >= cols) break;
      gauss_row(seed, TAG_Q, (uint64_t)c, k, grow);
      double x = 0.0;
      for (uint64_t l = 0; l < k; ++l) x += h[l] * grow[l];
      x += noise * draw_value(&gn, VAL_NORMAL);
      if (x == 0.0) x = noise;  /* keep the mask exact (probability ~0) */
      out[o].row = (uint64_t)r; out[o].col = (uint64_t)c; out[o].value = x;
      ++o;
    }
    free(grow);
  }
  free(H); free(cnt);
  *n_out = nnz;
  return out;
}
