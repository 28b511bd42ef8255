/* or_result.h -- TEST INFRASTRUCTURE ONLY. Result record shared by the C
 * restatement (ranky_oracle.c) and the reference wrapper (ref_capi.cpp);
 * oracle/oracle.py mirrors the layout with ctypes. */
#pragma once
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

#define OR_OK 0
#define OR_INVALID 1    /* std::invalid_argument */
#define OR_RANGE 2      /* std::out_of_range */
#define OR_CONVERGE 3   /* ranky::ConvergenceError */
#define OR_RUNTIME 4    /* std::runtime_error */
#define OR_NOMEM 5

typedef struct or_result {
  int status;
  char message[512];
  double residual; /* ConvergenceError::residual */
  /* repair report */
  uint64_t n_edges;
  uint64_t *e_block, *e_row, *e_col;
  int32_t *e_mech; /* 0 random, 1 neighbor */
  uint64_t n_blocks;
  uint64_t *lonely;
  uint64_t fallback;
  /* a sparse matrix (repaired) in sorted COO */
  uint64_t rows, cols, nnz;
  uint64_t *r, *c;
  double *v;
  /* SVD */
  uint64_t u_rows, u_cols;
  double *u;
  uint64_t n_sigma;
  double *sigma;
  int has_v;
  uint64_t v_rows, v_cols;
  double *vm;
  /* block records (pipeline) */
  uint64_t n_records;
  uint32_t *rec_kept;
  double *rec_payload; /* concatenated, record d at offset sum_{e<d} rows*kept_e */
  /* timing breakdown, seconds (filled by or_run_pipeline) */
  double t_repair, t_blocks, t_proxy;
} or_result;

#ifdef __cplusplus
}
#endif
