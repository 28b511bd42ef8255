/* Plain C against include/ranky_b200.h (no Python, no C++): the boundary as a
 * cgo / JNI / N-API binding would see it. Builds a small matrix with two lonely
 * rows, runs rk_run_pipeline with V, checks sigma against the dense SVD entry
 * point, V's shape and the repair report, and prints one line. Exit 0 = pass. */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "ranky_b200.h"

#define CHECK(x)                                                        \
  do {                                                                  \
    rk_status st_ = (x);                                                \
    if (st_ != RK_OK) {                                                 \
      fprintf(stderr, "%s -> %d: %s\n", #x, (int)st_, rk_last_error()); \
      return 1;                                                         \
    }                                                                   \
  } while (0)

int main(void) {
  enum { ROWS = 8, COLS = 64, D = 4 };
  rk_entry* e = malloc(sizeof(rk_entry) * ROWS * COLS);
  double* dense = calloc(ROWS * COLS, sizeof(double));
  uint64_t n = 0;
  for (uint64_t r = 0; r < ROWS; ++r)
    for (uint64_t c = 0; c < COLS; ++c) {
      if ((r == 3 && c < 16) || (r == 6 && c >= 48)) continue; /* lonely in blocks 0 and 3 */
      if ((r * 31 + c * 17) % 5 == 0) continue;
      const double v = 1.0 + (double)((r * 7 + c * 13) % 11) / 8.0;
      e[n].row = r;
      e[n].col = c;
      e[n].value = v;
      dense[r * COLS + c] = v;
      ++n;
    }
  rk_ctx* ctx = NULL;
  CHECK(rk_ctx_create(0, &ctx));
  rk_sparse_view a = {ROWS, COLS, n, e};
  rk_pipeline_result res;
  CHECK(rk_run_pipeline(ctx, &a, D, RK_RANDOM, 0, 7, 1, RK_WANT_V | RK_WANT_REPAIRED, 0, &res));
  if (res.report.n_edges != 2 || res.svd.v_rows != COLS || res.svd.n_sigma != ROWS) {
    fprintf(stderr, "unexpected shapes: edges %llu, v_rows %llu, k %llu\n", (unsigned long long)res.report.n_edges,
            (unsigned long long)res.svd.v_rows, (unsigned long long)res.svd.n_sigma);
    return 1;
  }
  /* sigma of the repaired matrix from the dense entry point */
  double* rep = calloc(ROWS * COLS, sizeof(double));
  for (uint64_t i = 0; i < res.repaired.nnz; ++i)
    rep[res.repaired.entries[i].row * COLS + res.repaired.entries[i].col] = res.repaired.entries[i].value;
  rk_svd ds;
  CHECK(rk_dense_svd(ctx, ROWS, COLS, rep, &ds));
  double worst = 0.0;
  for (uint64_t j = 0; j < ROWS; ++j) {
    const double rel = fabs(ds.sigma[j] - res.svd.sigma[j]) / ds.sigma[j];
    if (rel > worst) worst = rel;
  }
  printf("c abi smoke: %llu nnz, %llu repair edges, sigma_max %.6f, worst rel sigma diff %.2e\n",
         (unsigned long long)n, (unsigned long long)res.report.n_edges, res.svd.sigma[0], worst);
  rk_svd_free(&ds);
  rk_pipeline_result_free(&res);
  rk_ctx_destroy(ctx);
  free(e);
  free(dense);
  free(rep);
  return worst <= 1e-10 ? 0 : 1;
}
