/*
 * ranky_b200.h -- C ABI of the B200-native Ranky hot path.
 *
 * Each entry point replaces one reference routine of /root/reference/proj
 * (cited as include-or-source file:line). Plain pointers and sizes only; no
 * C++ or torch types cross this boundary. Host-pointer entry points take the
 * reference's value semantics (inputs are read, results are returned in
 * library-owned records released with rk_*_free); rk_dev_* entry points work
 * on device-resident data for callers that keep the matrix in HBM.
 *
 * Errors: every function returns an rk_status. The message of the last
 * failure on the calling thread is rk_last_error(); for RK_CONVERGENCE the
 * reference's ConvergenceError::residual() is rk_last_residual(). Status
 * codes map one-to-one onto the reference's exception types
 * (proj/include/ranky/errors.hpp:10-38 and the std:: exceptions it throws).
 *
 * Sparse inputs are the reference's SparseMatrix entries: an array of
 * rk_entry {row, col, value} without duplicates, explicit zeros or out-of-range
 * indices (proj/include/ranky/sparse_matrix.hpp:9-48). Any order is accepted:
 * like the reference constructor (sparse_matrix.cpp:12-30), unsorted entries
 * are sorted by (row, col) -- on the device -- before validation, and the first
 * invalid entry in sorted order is reported with the reference's message.
 * rk_entry has the exact layout of ranky::Entry, so a C++ caller passes
 * SparseMatrix::entries().data() unchanged.
 *
 * Dense matrices are row-major doubles, as ranky::DenseMatrix
 * (proj/include/ranky/dense_matrix.hpp:11-39).
 *
 * Every GPU entry point runs on the context's CUDA device and stream; there is
 * no CPU fallback. Calls on one context are not thread-safe; use one context
 * per thread.
 */
#ifndef RANKY_B200_H
#define RANKY_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RK_ABI_VERSION 1

#if defined(__GNUC__)
#define RK_API __attribute__((visibility("default")))
#else
#define RK_API
#endif

typedef enum rk_status {
  RK_OK = 0,
  RK_INVALID_ARGUMENT = 1, /* std::invalid_argument */
  RK_OUT_OF_RANGE = 2,     /* std::out_of_range */
  RK_CONVERGENCE = 3,      /* ranky::ConvergenceError (proj/include/ranky/errors.hpp:29-38) */
  RK_RUNTIME = 4,          /* std::runtime_error ("block task d failed: ...") */
  RK_CUDA = 5,             /* CUDA runtime failure or no usable device */
  RK_NOMEM = 6,            /* device or host allocation failed */
  RK_RECORD = 7,           /* ranky::RecordError: damaged or truncated block record file */
  RK_GRAM_REJECTED = 8,    /* sharded Gram route not applicable: take the TSQR path (rk_dev_shard_tsqr) */
  RK_PARSE = 9             /* ranky::ParseError (errors.hpp:9-20); the line is rk_last_error_line() */
} rk_status;

/* RepairMethod -- proj/include/ranky/repair.hpp:15-20 (same numbering) */
typedef enum rk_method { RK_RANDOM = 0, RK_NEIGHBOR = 1, RK_NEIGHBOR_RANDOM = 2, RK_NONE = 3 } rk_method;

/* Entry -- proj/include/ranky/sparse_matrix.hpp:9-15 */
typedef struct rk_entry {
  uint64_t row;
  uint64_t col;
  double value;
} rk_entry;

typedef struct rk_sparse_view {
  uint64_t rows, cols, nnz;
  const rk_entry* entries; /* host; any order (sorted on the device if needed) */
} rk_sparse_view;

/* SvdResult -- proj/include/ranky/svd.hpp:15-19. u: u_rows x u_cols row-major,
 * sigma: n_sigma descending, v (when has_v): v_rows x v_cols row-major. */
typedef struct rk_svd {
  uint64_t u_rows, u_cols;
  double* u;
  uint64_t n_sigma;
  double* sigma;
  int32_t has_v;
  uint64_t v_rows, v_cols;
  double* v;
} rk_svd;

/* RepairReport -- proj/include/ranky/repair.hpp:25-48. mechanism: 0 random, 1 neighbor */
typedef struct rk_repair_report {
  uint64_t n_edges;
  uint64_t *block, *row, *col;
  int32_t* mechanism;
  uint64_t n_blocks;
  uint64_t* lonely_counts;
  uint64_t fallback_count;
} rk_repair_report;

/* A library-owned sparse matrix in entry order (the repaired matrix). */
typedef struct rk_sparse {
  uint64_t rows, cols, nnz;
  rk_entry* entries;
} rk_sparse;

/* BlockResultRecord payloads -- proj/include/ranky/block_record.hpp:15-22:
 * record d is rows x kept[d] row-major at payload + offset[d]. */
typedef struct rk_records {
  uint64_t n_records, rows;
  uint32_t* kept;
  uint64_t* offset;
  double* payload;
} rk_records;

/* Per-stage device times of the last pipeline call, milliseconds (CUDA events). */
typedef struct rk_timing {
  double repair_ms, blocks_ms, merge_ms, recover_ms, total_ms;
  double qr_ms, jacobi_ms;       /* inside blocks_ms */
  uint64_t jacobi_sweeps_max;    /* over all block factorizations */
  uint64_t jacobi_rotations;     /* over all block factorizations */
  uint64_t kernel_launches;      /* kernels this library launched in the call */
  uint64_t jacobi_sweeps_sum;    /* sweeps summed over the block factorizations */
  double qr_flops;               /* algorithmic FP64 flops of the block QRs: sum 2 n_d M^2 - 2/3 M^3 */
  double jacobi_flops;           /* algorithmic FP64 flops of the block Jacobi: per block
                                    sweeps*(c(c-1)/2*2M + 2Mc) + rotations*6M, c = active columns */
  uint64_t merge_sweeps;         /* the merge's Jacobi */
  uint64_t merge_rotations;
  double merge_flops;            /* algorithmic FP64 flops of the merge: Gram route M(M+1)*sum k (SYRK) +
                                    M^3/3 (Cholesky), TSQR route 2*sum k*M^2; + its Jacobi as above */
} rk_timing;

/* PipelineResult (+ V) -- proj/include/ranky/pipeline.hpp:30-36 */
typedef struct rk_pipeline_result {
  rk_svd svd;              /* sigma + U of the input; v = V = A^T U Sigma^-1 when requested */
  rk_repair_report report;
  rk_sparse repaired;      /* filled only when want_repaired */
  rk_records records;
  rk_timing timing;
} rk_pipeline_result;

/* ---- errors & context ---------------------------------------------------- */
RK_API const char* rk_last_error(void);
RK_API double rk_last_residual(void);
RK_API uint64_t rk_last_error_line(void); /* ParseError::line() of the last RK_PARSE */
/* Re-read the RK_* tuning/debug environment switches (read once per process
 * otherwise). Not thread-safe against calls in flight. */
RK_API void rk_reload_tuning(void);
/* Build flags: bit 0 = experiments build (RK_EXPERIMENTS: the measured-and-not-kept
 * variants RK_PRECOND, RK_CHOL=r, RK_GRAM_PAIRS are compiled in). */
RK_API uint32_t rk_build_flags(void);
RK_API int32_t rk_abi_version(void);

typedef struct rk_ctx rk_ctx;
/* device = CUDA ordinal; the context owns a non-blocking stream */
RK_API rk_status rk_ctx_create(int32_t device, rk_ctx** out);
RK_API rk_status rk_ctx_destroy(rk_ctx* ctx);
/* run subsequent work on a caller stream (cudaStream_t); NULL restores the own stream */
RK_API rk_status rk_ctx_set_stream(rk_ctx* ctx, void* cuda_stream);
RK_API rk_status rk_ctx_synchronize(rk_ctx* ctx);
/* kernels launched through this context since creation */
RK_API uint64_t rk_ctx_kernel_launches(const rk_ctx* ctx);

/* release one library-allocated host buffer (e.g. a field taken over from a result
 * record, which must then be set to NULL before the record is freed) */
RK_API void rk_host_free(void* p);
RK_API void rk_svd_free(rk_svd* s);
RK_API void rk_repair_report_free(rk_repair_report* r);
RK_API void rk_sparse_free(rk_sparse* s);
RK_API void rk_records_free(rk_records* r);
RK_API void rk_pipeline_result_free(rk_pipeline_result* r);

/* ---- KeyedRng -- proj/include/ranky/rng.hpp:11-25, proj/src/rng.cpp:16-38 ----
 * Streams evaluated on the device (the same routine the repair kernels use).
 * out[i] = i-th next() of KeyedRng(seed, block[i], row[i]) after skip[i] draws. */
RK_API rk_status rk_keyed_rng_next(rk_ctx* ctx, uint64_t n, uint64_t seed, const uint64_t* block,
                            const uint64_t* row, uint64_t draws, uint64_t* out /* n x draws */);
/* out[i] = KeyedRng(seed, block[i], row[i]).below(bound[i]) */
RK_API rk_status rk_keyed_rng_below(rk_ctx* ctx, uint64_t n, uint64_t seed, const uint64_t* block,
                             const uint64_t* row, const uint64_t* bound, uint64_t* out);

/* ---- rank check & repair -- proj/include/ranky/repair.hpp:50-96 ------------- */
/* find_lonely_rows(a, partition_columns(a.cols, block_count), d) -- repair.hpp:51-52.
 * out must hold a.rows entries; *n_out receives the count. */
RK_API rk_status rk_find_lonely_rows(rk_ctx* ctx, const rk_sparse_view* a, uint64_t block_count,
                              uint64_t d, uint64_t* out, uint64_t* n_out);
/* repair(a, partition_columns(a.cols, block_count), method, seed) -- repair.hpp:93-96 */
RK_API rk_status rk_repair(rk_ctx* ctx, const rk_sparse_view* a, uint64_t block_count, rk_method method,
                    uint64_t seed, rk_sparse* repaired, rk_repair_report* report);

/* ---- SVD kernels -- proj/include/ranky/svd.hpp:25-29 ------------------------ */
/* dense_svd(a) -- svd.hpp:25; a is rows x cols row-major */
RK_API rk_status rk_dense_svd(rk_ctx* ctx, uint64_t rows, uint64_t cols, const double* a, rk_svd* out);
/* block_svd(block, keep) -- svd.hpp:29 (no V, U truncated to min(keep, rows, cols)) */
RK_API rk_status rk_block_svd(rk_ctx* ctx, const rk_sparse_view* block, uint64_t keep, rk_svd* out);

/* ---- proxy -- proj/include/ranky/proxy.hpp:18-27 ---------------------------- */
/* proxy_svd(proxy) -- proxy.hpp:22; proxy rows x total_cols row-major with
 * n_offsets = blocks + 1 block offsets (the trailing one must equal total_cols) */
RK_API rk_status rk_proxy_svd(rk_ctx* ctx, uint64_t rows, uint64_t total_cols, const double* proxy,
                       uint64_t n_offsets, const uint64_t* block_offsets, rk_svd* out);
/* recover_right_vectors(a, u, sigma, tol) -- proxy.hpp:26-27; V is a.cols x retained
 * row-major, written into out->v (out->u / sigma stay empty) */
RK_API rk_status rk_recover_right_vectors(rk_ctx* ctx, const rk_sparse_view* a, uint64_t u_rows,
                                   uint64_t u_cols, const double* u, uint64_t n_sigma,
                                   const double* sigma, double tol, rk_svd* out);

/* ---- pipeline -- proj/include/ranky/pipeline.hpp:23-44 ---------------------- */
/* run_block_task for every block of partition_columns(a.cols, block_count) of an
 * already-repaired matrix, in block order (records only) -- pipeline.hpp:23 */
RK_API rk_status rk_run_block_tasks(rk_ctx* ctx, const rk_sparse_view* a, uint64_t block_count,
                             uint64_t keep, rk_records* out);
/* run_pipeline(a, block_count, method, keep, seed, workers) -- pipeline.hpp:42-44.
 * workers is validated (0 is invalid) and otherwise ignored: block tasks run as
 * batched kernels and the result is identical for any value, as in the reference.
 * flags: RK_WANT_V adds V = recover_right_vectors(repaired, U[:, :top_k],
 * sigma[:top_k], 1e-10) (top_k = 0: all); RK_WANT_REPAIRED returns the repaired
 * matrix; RK_WANT_RECORDS returns the block records. */
#define RK_WANT_V 1u
#define RK_WANT_REPAIRED 2u
#define RK_WANT_RECORDS 4u
RK_API rk_status rk_run_pipeline(rk_ctx* ctx, const rk_sparse_view* a, uint64_t block_count,
                          rk_method method, uint64_t keep, uint64_t seed, uint64_t workers,
                          uint32_t flags, uint64_t top_k, rk_pipeline_result* out);

/* ---- device-resident path (inputs already in HBM) --------------------------- */
typedef struct rk_dev_matrix rk_dev_matrix;
/* upload host entries once and build the device CSR/CSC */
RK_API rk_status rk_dev_matrix_create(rk_ctx* ctx, const rk_sparse_view* a, rk_dev_matrix** out);
RK_API rk_status rk_dev_matrix_destroy(rk_dev_matrix* m);
RK_API uint64_t rk_dev_matrix_nnz(const rk_dev_matrix* m);

/* Device-resident outputs of rk_dev_full_svd (owned by the library). */
typedef struct rk_dev_outputs {
  uint64_t rows, cols, k_sigma, k_v;
  const double* d_sigma;  /* k_sigma, device */
  const double* d_u;      /* rows x k_sigma row-major, device */
  const double* d_v;      /* cols x k_v row-major, device (NULL without RK_WANT_V) */
  uint64_t n_edges;
} rk_dev_outputs;

/* The whole hot path on a device-resident matrix: repair -> block SVDs -> merge ->
 * (V). Results stay in HBM until rk_dev_outputs_free. Same flags as rk_run_pipeline
 * (RK_WANT_REPAIRED / RK_WANT_RECORDS are ignored here). */
RK_API rk_status rk_dev_full_svd(rk_ctx* ctx, const rk_dev_matrix* a, uint64_t block_count,
                          rk_method method, uint64_t keep, uint64_t seed, uint32_t flags,
                          uint64_t top_k, rk_dev_outputs** out, rk_timing* timing);
RK_API rk_status rk_dev_outputs_free(rk_dev_outputs* o);

/* Reconstruction of device-resident outputs (the reference's test metric,
 * proj/tests/test_support.hpp:57-70): residual = ||A - U[:, :k_v] diag(sigma) V^T||_F
 * formed exactly on the device (no dense N x M copy), A being the repaired matrix
 * the outputs were computed from (the input `a` when no repair edge was added);
 * a_norm = ||A||_F. Requires RK_WANT_V. */
RK_API rk_status rk_dev_residual(rk_ctx* ctx, const rk_dev_matrix* a, const rk_dev_outputs* out, double* residual,
                                 double* a_norm);

/* ---- Matrix Market (proj/src/matrix_market.cpp:38-132) ----------------------------
 * `%%MatrixMarket matrix coordinate real general`, 1-based. Loading validates as the
 * reference (RK_PARSE with its messages and line numbers; the (row, col) sort that
 * finds duplicates runs on the device) and returns the entries sorted; saving writes
 * the reference's bytes (shortest round-trip values). Free with rk_sparse_free. */
RK_API rk_status rk_load_matrix_market(rk_ctx* ctx, const char* path, rk_sparse* out);
RK_API rk_status rk_save_matrix_market(const rk_sparse_view* a, const char* path);

/* ---- RepairWorkspace (proj/include/ranky/repair.hpp:56-87, proj/src/repair.cpp:52-160) ----
 * The single-row checker API on a device workspace: the matrix (device CSR + CSC)
 * plus the edges inserted so far. Partitions are partition_columns(cols, block_count).
 * The draws stay with the caller's KeyedRng, where the reference makes them:
 *   apply_random(d, row, rng):   col = begin(d) + rng.below(width(d)); rk_workspace_insert
 *   apply_neighbor(d, row, rng): rk_workspace_neighbor_columns -> n; n == 0: no edge and no
 *                                draw; else col = cols[rng.below(n)]; rk_workspace_insert
 * rk_workspace_neighbor_columns writes the ascending distinct columns of block d held by
 * rows sharing a column with `row` outside block d (the row itself included), as
 * repair.cpp:107-125 builds neighbor_cols; `cols` must hold width(d) entries.
 * Insertion is idempotent. rk_workspace_to_matrix: original values kept, inserted 1.0. */
typedef struct rk_workspace rk_workspace;
RK_API rk_status rk_workspace_create(rk_ctx* ctx, const rk_sparse_view* a, uint64_t block_count,
                                     rk_workspace** out);
RK_API rk_status rk_workspace_destroy(rk_workspace* ws);
RK_API rk_status rk_workspace_has_entry(rk_workspace* ws, uint64_t row, uint64_t col, int32_t* out);
RK_API rk_status rk_workspace_row_lonely_in_block(rk_workspace* ws, uint64_t d, uint64_t row, int32_t* out);
RK_API rk_status rk_workspace_lonely_rows(rk_workspace* ws, uint64_t d, uint64_t* rows_out, uint64_t* n_out);
RK_API rk_status rk_workspace_neighbor_columns(rk_workspace* ws, uint64_t d, uint64_t row, uint64_t* cols_out,
                                               uint64_t* n_out);
RK_API rk_status rk_workspace_insert(rk_workspace* ws, uint64_t row, uint64_t col);
RK_API rk_status rk_workspace_to_matrix(rk_workspace* ws, rk_sparse* out);

/* ---- evaluation metrics (proj/include/ranky/metrics.hpp, proj/src/metrics.cpp) ----
 * Matrices are row-major (DenseMatrix layout). The rk_dev_* forms take device
 * pointers (e.g. rk_dev_outputs' d_u / d_sigma) and return scalars to the host;
 * the plain forms take host pointers (upload, compute on the device, download).
 *   sigma_error        metrics.cpp:32-42   sum |a_i - b_i|, the shorter list zero-padded
 *   align_signs        metrics.cpp:44-93   sign flips; Procrustes on clusters of sigma_ref
 *                                          (n_sigma = 0: no sigma, flips only)
 *   left_vector_error  metrics.cpp:95-103  sum |align_signs(u_hat) - u_ref|
 *   numerical_rank     metrics.cpp:105-114 #{sigma > tol sigma_max} of dense_svd(a) */
RK_API rk_status rk_dev_sigma_error(rk_ctx* ctx, const double* d_sigma_hat, uint64_t n_hat,
                                    const double* d_sigma_ref, uint64_t n_ref, double* out);
RK_API rk_status rk_dev_align_signs(rk_ctx* ctx, const double* d_u_hat, const double* d_u_ref, uint64_t rows,
                                    uint64_t cols, const double* d_sigma_ref, uint64_t n_sigma, double* d_out);
RK_API rk_status rk_dev_left_vector_error(rk_ctx* ctx, const double* d_u_hat, const double* d_u_ref, uint64_t rows,
                                          uint64_t cols, const double* d_sigma_ref, uint64_t n_sigma, double* out);
RK_API rk_status rk_dev_numerical_rank(rk_ctx* ctx, const double* d_a, uint64_t rows, uint64_t cols, double tol,
                                       uint64_t* out);
RK_API rk_status rk_sigma_error(rk_ctx* ctx, const double* sigma_hat, uint64_t n_hat, const double* sigma_ref,
                                uint64_t n_ref, double* out);
RK_API rk_status rk_align_signs(rk_ctx* ctx, const double* u_hat, const double* u_ref, uint64_t rows, uint64_t cols,
                                const double* sigma_ref, uint64_t n_sigma, double* out);
RK_API rk_status rk_left_vector_error(rk_ctx* ctx, const double* u_hat, const double* u_ref, uint64_t rows,
                                      uint64_t cols, const double* sigma_ref, uint64_t n_sigma, double* out);
RK_API rk_status rk_numerical_rank(rk_ctx* ctx, const double* a, uint64_t rows, uint64_t cols, double tol,
                                   uint64_t* out);

/* ---- sharded path (one process per GPU) --------------------------------------
 * Column blocks are sharded over G ranks by merge-tree leaves. Rank g repairs the
 * whole matrix (the replay is deterministic, so every rank holds the same repaired
 * matrix without communication), factors the blocks of leaves [leaf_lo, leaf_hi)
 * and reduces their records to the R factor of that subtree of the fixed merge tree
 * (rk_merge_tree_leaves) -- or, on the Gram route below, to the subtree's Gram. The
 * caller all-gathers the G factors (NCCL) and every rank finishes the same top of
 * the tree, then recovers V for its own columns. With (leaves / G) a power of two
 * the results are bitwise identical for every G. */
RK_API uint64_t rk_merge_tree_leaves(uint64_t rows, uint64_t cols, uint64_t block_count, uint64_t keep);
typedef struct rk_dev_shard rk_dev_shard;
/* d_root_out: device, rows*rows doubles, column-major upper-triangular R */
RK_API rk_status rk_dev_shard_factor(rk_ctx* ctx, const rk_dev_matrix* a, uint64_t block_count, rk_method method,
                              uint64_t keep, uint64_t seed, uint64_t leaf_lo, uint64_t leaf_hi,
                              double* d_root_out, rk_dev_shard** shard_out, rk_timing* timing);
/* d_roots: device, n_roots x rows x rows (leaf order); V for columns [col_lo, col_hi) */
RK_API rk_status rk_dev_shard_finish(rk_ctx* ctx, rk_dev_shard* shard, const double* d_roots, uint64_t n_roots,
                              uint32_t flags, uint64_t top_k, uint64_t col_lo, uint64_t col_hi,
                              rk_dev_outputs** out, rk_timing* timing);
RK_API rk_status rk_dev_shard_destroy(rk_dev_shard* shard);
/* Gram route of the sharded merge (the single-GPU merge's route, merge_records):
 * rk_dev_shard_factor_gram does the same repair and block stage and writes
 * d_gram_out = the Gram (rows x rows, column-major, full) of the shard's stacked
 * records -- each leaf's records, then the leaves by the fixed pairwise tree, so an
 * aligned power-of-two run of leaves is a node of the whole matrix's tree; it
 * returns RK_GRAM_REJECTED without a shard when the route does not apply (rows >
 * 1280 or not a multiple of 8, RK_BLOCK_ROUTE=householder). The caller all-gathers
 * the G partials; rk_dev_shard_finish_gram finishes the pairwise tree, Cholesky, the
 * kappa guard and the Jacobi, then V for [col_lo, col_hi). When the guard rejects
 * (RK_GRAM_REJECTED, identically on every rank) each rank calls rk_dev_shard_tsqr
 * for its subtree's R factor, the caller all-gathers those and rk_dev_shard_finish
 * completes as on the TSQR path. One 512 KiB all-gather per rank at c2 either way. */
RK_API rk_status rk_dev_shard_factor_gram(rk_ctx* ctx, const rk_dev_matrix* a, uint64_t block_count,
                                          rk_method method, uint64_t keep, uint64_t seed, uint64_t leaf_lo,
                                          uint64_t leaf_hi, double* d_gram_out, rk_dev_shard** shard_out,
                                          rk_timing* timing);
RK_API rk_status rk_dev_shard_finish_gram(rk_ctx* ctx, rk_dev_shard* shard, const double* d_grams, uint64_t n_roots,
                                          uint32_t flags, uint64_t top_k, uint64_t col_lo, uint64_t col_hi,
                                          rk_dev_outputs** out, rk_timing* timing);
RK_API rk_status rk_dev_shard_tsqr(rk_ctx* ctx, rk_dev_shard* shard, double* d_root_out);

/* ---- RNKY block records (proj/src/block_record.cpp:51-144) ----------------------
 * Files byte-identical to ranky::write_block_record: "RNKY", version u16 = 1,
 * block index u32, rows u32, k u32, rows*k doubles row-major, CRC32 of the payload
 * bytes, little-endian. Reader failures return RK_RECORD with the reference's
 * RecordError message. */
RK_API uint32_t rk_crc32(const void* data, uint64_t size); /* block_record.cpp:53-68 */
/* CRC32 of n device-resident byte ranges [d_data + offsets[i], + lengths[i]) (GPU;
 * offsets/lengths/crcs are host arrays) */
RK_API rk_status rk_dev_crc32(rk_ctx* ctx, const void* d_data, const uint64_t* offsets, const uint64_t* lengths,
                              uint64_t n, uint32_t* crcs);
RK_API rk_status rk_write_block_record(uint32_t block_index, uint32_t rows, uint32_t kept, const double* payload,
                                       const char* path);
/* *payload (rows*kept doubles) is library-owned: rk_host_free */
RK_API rk_status rk_read_block_record(const char* path, uint32_t* block_index, uint32_t* rows, uint32_t* kept,
                                      double** payload);
/* every record of `records` to "<path_prefix><block index>.rnky", payload CRCs on the GPU */
RK_API rk_status rk_write_records(rk_ctx* ctx, const rk_records* records, const char* path_prefix);

/* ---- library-owned multi-GPU runs --------------------------------------------
 * The sharded protocol above, orchestrated by the library (DESIGN.md (e)):
 *
 * rk_multi_*: one process drives several devices (`devices` may repeat one device:
 * its shards then share it). rk_multi_run_pipeline is rk_run_pipeline over the whole
 * box -- every device uploads the matrix, factors its leaves; the M x M factors are
 * exchanged by peer copies (NVLink with peer access), every shard finishes the same
 * tree top; V rows and records are copied back from their owners concurrently.
 * Results are bitwise those of one process per GPU with the same shard count.
 *
 * rk_dist_*: one process per GPU with the library's own NCCL communicator (NCCL
 * opened at run time from libnccl.so.2). rank 0 makes the id (rk_nccl_unique_id),
 * the caller ships it to the other ranks. rk_dist_full_svd returns this rank's
 * outputs (sigma, U and V rows [col_lo, col_hi)).
 *
 * rk_dev_sharded_full_svd: the same with the caller's all-gather: allgather(user,
 * d_mine, d_all, count) must gather `count` doubles from every rank into d_all in
 * rank order (device pointers on the context's device, the context's stream
 * synchronized before the call; the data must be in d_all when it returns). */
typedef struct rk_multi rk_multi;
typedef struct rk_dist rk_dist;
typedef void (*rk_allgather_fn)(void* user, const double* d_mine, double* d_all, uint64_t count);
RK_API int32_t rk_device_count(void); /* visible CUDA devices (0 when none) */
RK_API rk_status rk_multi_create(const int32_t* devices, uint32_t n, rk_multi** out);
RK_API rk_status rk_multi_destroy(rk_multi* m);
RK_API rk_status rk_multi_run_pipeline(rk_multi* m, const rk_sparse_view* a, uint64_t block_count,
                                       rk_method method, uint64_t keep, uint64_t seed, uint32_t flags,
                                       uint64_t top_k, rk_pipeline_result* out);
RK_API rk_status rk_nccl_unique_id(uint8_t id_out[128]);
RK_API rk_status rk_dist_create(rk_ctx* ctx, int32_t world, int32_t rank, const uint8_t id[128], rk_dist** out);
RK_API rk_status rk_dist_destroy(rk_dist* d);
RK_API rk_status rk_dist_full_svd(rk_dist* d, const rk_dev_matrix* a, uint64_t block_count, rk_method method,
                                  uint64_t keep, uint64_t seed, uint32_t flags, uint64_t top_k,
                                  rk_dev_outputs** out, rk_timing* timing, uint64_t* col_lo, uint64_t* col_hi);
RK_API rk_status rk_dev_sharded_full_svd(rk_ctx* ctx, const rk_dev_matrix* a, uint64_t block_count,
                                         rk_method method, uint64_t keep, uint64_t seed, uint32_t flags,
                                         uint64_t top_k, int32_t world, int32_t rank, rk_allgather_fn allgather,
                                         void* user, rk_dev_outputs** out, rk_timing* timing, uint64_t* col_lo,
                                         uint64_t* col_hi);

#ifdef __cplusplus
}
#endif
#endif /* RANKY_B200_H */
