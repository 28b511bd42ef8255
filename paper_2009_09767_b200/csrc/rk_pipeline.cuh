// rk_pipeline.cuh -- orchestration interfaces shared by rk_pipeline.cu and rk_api.cu
#pragma once

#include <utility>

#include "rk_internal.cuh"

namespace rk {

// optional per-block outputs for the block_svd API (U, sigma, deficient flags)
struct BlockApiOut {
  DBuf<double> u;          // per block: M x kept row-major at offset_u[i]
  DBuf<double> sigma;      // per block: M entries (first kept valid)
  DBuf<uint8_t> deficient; // per block: M flags
};

struct BlockStageResult {
  DBuf<double> payload;               // records back to back (M x kept row-major each)
  std::vector<uint64_t> offset;       // doubles into payload, per block
  std::vector<uint32_t> kept;
  // per block: columns past eff are zero by construction (a block of n_d < kept nonzero columns); the
  // merge reads only those and need not scan the records for it (record_eff_cols)
  std::vector<uint32_t> eff;
  std::vector<std::string> failures;  // per block, empty = ok (reference "block task d failed: ...")
  double conv_residual = 0.0;
  uint64_t sweeps_max = 0, rotations = 0, sweeps_sum = 0;
  double qr_flops = 0, jacobi_flops = 0;
  float qr_ms = 0, jacobi_ms = 0;
};

void block_stage(Ctx& c, const DevMatrix& a, const Partition& p, uint64_t d_lo, uint64_t d_hi, uint64_t keep,
                 BlockStageResult& out, BlockApiOut* api);

struct MergeOut {
  uint32_t k = 0;          // min(M, total kept)
  DBuf<double> sigma;      // k, descending
  DBuf<double> u;          // M x k row-major, sign convention applied
  uint64_t sweeps = 0, rotations = 0;
  double flops = 0.0;      // algorithmic FP64 flops (rk_timing::merge_flops)
};

// TSQR over a forest: every tree's leaves (column-major, factored in place) are
// reduced by a fixed pairwise tree to one R factor (n x n column-major, upper)
struct LeafRef {
  double* a;
  uint64_t lda;
  uint32_t m;
  uint32_t split;  // see QrJob::split
};
void tsqr_forest(Ctx& c, uint32_t n, std::vector<std::vector<LeafRef>>& leaves, std::vector<DBuf<double>>& roots);

// leaves of the merge tree: consecutive records, each leaf at least M rows of P^T
struct TreeLeaf {
  uint32_t r0, r1, height;
};
std::vector<TreeLeaf> merge_leaves(const std::vector<uint32_t>& kept, uint32_t M);

// R factor (M x M column-major, upper) of the stacked leaves [leaf_lo, leaf_hi)
void merge_subtree(Ctx& c, const double* payload, const std::vector<uint64_t>& offset,
                   const std::vector<uint32_t>& kept, uint32_t M, const std::vector<TreeLeaf>& leaves,
                   size_t leaf_lo, size_t leaf_hi, DBuf<double>& r_out, const std::vector<uint32_t>* eff_hint = nullptr);
// top of the tree over R factors (each M x M column-major), then Jacobi on R^T
void merge_finish(Ctx& c, std::vector<DBuf<double>>& roots, uint32_t M, MergeOut& out);
// the whole proxy SVD of the records (sigma, U of P)
void merge_records(Ctx& c, const double* payload, const std::vector<uint64_t>& offset,
                   const std::vector<uint32_t>& kept, uint32_t M, MergeOut& out,
                   const std::vector<uint32_t>* eff_hint = nullptr);

// the merge's Gram route (see merge_records): eligibility, and the finish from
// W = P P^T (M x jacobi_cols_pad slot, consumed); false when the kappa guard rejects
bool gram_merge_eligible(uint32_t M);
// the reference-algorithm flop count of a Jacobi run (rk_timing::jacobi_flops)
double jacobi_flops_of(uint64_t sweeps, uint64_t rotations, uint32_t rows, uint32_t cols);
bool gram_merge(Ctx& c, DBuf<double>& W, uint32_t M, MergeOut& out);
// rk_eig.cu: the Gram route by a symmetric eigensolver (tridiagonalisation in one
// cluster, bisection, inverse iteration); false (out untouched) when it declines
bool eig_merge_eligible(uint32_t M);
bool gram_merge_eig(Ctx& c, const double* G, uint32_t M, MergeOut& out);

// dense_svd on the device: a is rows x cols row-major (device). Outputs row-major.
struct DenseSvdOut {
  uint32_t k = 0;
  DBuf<double> u, sigma, v;  // u rows x k, v cols x k
};
void dense_svd_dev(Ctx& c, const double* a, uint32_t rows, uint32_t cols, DenseSvdOut& out);

// rk_gram.cu: Gram + Cholesky route (see the file header)
void sparse_gram(const DevMatrix& a, const Partition& p, uint64_t d_lo, uint64_t nblk, double* G, uint64_t stride,
                 cudaStream_t s);
// eff[d] for records [r_lo, r_hi) (0 elsewhere): 1 + the last column of record d with
// a nonzero; the finalize writes columns by descending sigma and a sigma-0 column is
// exactly zero, so the columns past eff[d] are zero
std::vector<uint32_t> record_eff_cols(const double* payload, const std::vector<uint64_t>& offset,
                                      const std::vector<uint32_t>& kept, uint32_t M, uint32_t r_lo, uint32_t r_hi,
                                      cudaStream_t s, const std::vector<uint32_t>* hint = nullptr);
void records_gram(const double* payload, const std::vector<uint64_t>& offset, const std::vector<uint32_t>& kept,
                  uint32_t M, double* G, cudaStream_t s, const std::vector<uint32_t>* eff_hint = nullptr);
void cholesky_batched(double* const* d_mats, uint32_t n_mats, uint32_t M, uint32_t* d_status, double* d_ratio,
                      cudaStream_t s);
// the Gram of the stacked records of the given leaves (block ranges [first, second)):
// each leaf's records summed in chunk order, the leaves combined by the fixed
// pairwise tree -- so a rank's aligned power-of-two run of leaves is a node of the
// whole matrix's tree. G: M x M column-major (full).
void leaf_gram_tree(const double* payload, const std::vector<uint64_t>& offset, const std::vector<uint32_t>& kept,
                    uint32_t M, const std::vector<std::pair<uint32_t, uint32_t>>& leaves, double* G, cudaStream_t s,
                    const std::vector<uint32_t>* eff_hint = nullptr);
// pairwise tree sum of n M x M matrices stored back to back; the result in mats[0, M*M)
void gram_tree_sum(double* mats, uint64_t n, uint32_t M, cudaStream_t s);
// symmetric diagonal ordering of nb Grams (slots of `stride` doubles, M x M,
// ld M): perm (nb x M, position -> original row), Gp = the permuted Grams
void diag_order(const double* G, uint64_t stride, uint32_t M, uint64_t nb, uint32_t* perm, double* Gp,
                cudaStream_t s);
bool diag_order_enabled();  // RK_DIAG_ORDER=0 turns it off
double kappa_max(uint32_t M);
uint32_t cholesky_max_rows();
bool gram_route_enabled();

// rk_eval.cu: the reference's evaluation metrics (proj/src/metrics.cpp:32-114) on the device
double sigma_error_device(const double* a, uint64_t na, const double* b, uint64_t nb, cudaStream_t s);
void align_signs_device(Ctx& c, const double* hat, const double* ref, uint64_t rows, uint64_t cols,
                        const double* sigma_ref, uint64_t n_sigma, double* out);
double left_vector_error_device(Ctx& c, const double* hat, const double* ref, uint64_t rows, uint64_t cols,
                                const double* sigma_ref, uint64_t n_sigma);
uint64_t numerical_rank_device(Ctx& c, const double* a, uint64_t rows, uint64_t cols, double tol);

// small launch helpers
void sign_rows(double* u, uint32_t rows, uint32_t k, double* v, uint32_t vrows, cudaStream_t s);
void check_finite_or_throw(const double* x, uint64_t n, const char* what, cudaStream_t s);

}  // namespace rk
