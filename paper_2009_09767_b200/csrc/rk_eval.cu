// rk_eval.cu -- the reference's evaluation metrics on the device
// (proj/src/metrics.cpp:32-114, proj/include/ranky/metrics.hpp):
//
//   sigma_error        sum |sigma_hat_i - sigma_ref_i|, the shorter list zero-padded (:32-42)
//   align_signs        per column: flip u_hat_j when <u_hat_j, u_ref_j> < 0; with sigma_ref,
//                      a degenerate cluster (consecutive sigma_ref within 1e-9 sigma_max) is
//                      aligned as a block by orthogonal Procrustes: W = U_c V_c^T from the SVD
//                      of C = hat_c^T ref_c, hat_c <- hat_c W (:44-93)
//   left_vector_error  sum |align_signs(u_hat) - u_ref| (:95-103)
//   numerical_rank     #{sigma > tol sigma_max, sigma > 0} of dense_svd(a) (:105-114)
//
// U matrices are row-major rows x cols (as DenseMatrix). Column dots and the
// cluster products run one thread per output element with the row loop inside
// (coalesced across columns); the absolute-difference sums are reduced per CTA
// in a fixed tree and the CTA partials added in CTA order, so every metric is
// deterministic run to run. The Procrustes SVD is dense_svd_dev (the device
// dense_svd), exactly the routine the reference calls (svd.cpp:365-379).
#include "rk_pipeline.cuh"

namespace rk {
namespace {

constexpr int kET = 256;

__device__ __forceinline__ double block_sum(double x, double* sh) {
#pragma unroll
  for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) sh[w] = x;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x < 32) {
    t = threadIdx.x < (kET >> 5) ? sh[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  }
  return t;
}

// partial[b] = sum over this CTA's grid-stride elements of |a_i - b_i| (missing = 0)
__global__ void absdiff_partial(const double* __restrict__ a, uint64_t na, const double* __restrict__ b, uint64_t nb,
                                uint64_t n, double* __restrict__ partial) {
  __shared__ double sh[kET / 32];
  double acc = 0.0;
  for (uint64_t i = blockIdx.x * (uint64_t)kET + threadIdx.x; i < n; i += (uint64_t)gridDim.x * kET) {
    const double x = i < na ? a[i] : 0.0, y = i < nb ? b[i] : 0.0;
    acc += fabs(x - y);
  }
  const double t = block_sum(acc, sh);
  if (threadIdx.x == 0) partial[blockIdx.x] = t;
}

__global__ void sum_in_order(const double* __restrict__ partial, uint32_t n, double* __restrict__ out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double s = 0.0;
    for (uint32_t i = 0; i < n; ++i) s += partial[i];
    *out = s;
  }
}

// dots[j] = <hat[:, j], ref[:, j]>, j in [0, cols)
__global__ void column_dots(const double* __restrict__ hat, const double* __restrict__ ref, uint64_t rows,
                            uint64_t cols, double* __restrict__ dots) {
  const uint64_t j = blockIdx.x * (uint64_t)kET + threadIdx.x;
  if (j >= cols) return;
  double s = 0.0;
  for (uint64_t i = 0; i < rows; ++i) s = fma(hat[i * cols + j], ref[i * cols + j], s);
  dots[j] = s;
}

// out = hat with column j negated where flip[j] (singleton columns; cluster columns are
// overwritten afterwards)
__global__ void apply_flips(const double* __restrict__ hat, const double* __restrict__ dots, uint64_t rows,
                            uint64_t cols, double* __restrict__ out) {
  const uint64_t total = rows * cols;
  for (uint64_t t = blockIdx.x * (uint64_t)kET + threadIdx.x; t < total; t += (uint64_t)gridDim.x * kET) {
    const uint64_t j = t % cols;
    out[t] = dots[j] < 0.0 ? -hat[t] : hat[t];
  }
}

// C (c x c row-major) = hat[:, lo:lo+c]^T ref[:, lo:lo+c]
__global__ void cluster_cross(const double* __restrict__ hat, const double* __restrict__ ref, uint64_t rows,
                              uint64_t cols, uint64_t lo, uint32_t c, double* __restrict__ C) {
  const uint64_t t = blockIdx.x * (uint64_t)kET + threadIdx.x;
  if (t >= (uint64_t)c * c) return;
  const uint64_t p = t / c, q = t % c;
  double s = 0.0;
  for (uint64_t i = 0; i < rows; ++i) s = fma(hat[i * cols + lo + p], ref[i * cols + lo + q], s);
  C[t] = s;
}

// W (c x c row-major) = U V^T (U, V c x c row-major)
__global__ void procrustes_w(const double* __restrict__ U, const double* __restrict__ V, uint32_t c,
                             double* __restrict__ W) {
  const uint64_t t = blockIdx.x * (uint64_t)kET + threadIdx.x;
  if (t >= (uint64_t)c * c) return;
  const uint64_t p = t / c, q = t % c;
  double s = 0.0;
  for (uint32_t k = 0; k < c; ++k) s = fma(U[p * c + k], V[q * c + k], s);
  W[t] = s;
}

// out[:, lo:lo+c] = hat[:, lo:lo+c] W
__global__ void cluster_apply(const double* __restrict__ hat, const double* __restrict__ W, uint64_t rows,
                              uint64_t cols, uint64_t lo, uint32_t c, double* __restrict__ out) {
  const uint64_t total = rows * c;
  for (uint64_t t = blockIdx.x * (uint64_t)kET + threadIdx.x; t < total; t += (uint64_t)gridDim.x * kET) {
    const uint64_t i = t / c, q = t % c;
    double s = 0.0;
    for (uint32_t k = 0; k < c; ++k) s = fma(hat[i * cols + lo + k], W[(uint64_t)k * c + q], s);
    out[i * cols + lo + q] = s;
  }
}

unsigned grid_of(uint64_t n, unsigned cap = 4096) {
  return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(ceil_div(n ? n : 1, kET), cap));
}

}  // namespace

double sigma_error_device(const double* a, uint64_t na, const double* b, uint64_t nb, cudaStream_t s) {
  const uint64_t n = std::max(na, nb);
  const unsigned g = grid_of(n, 256);
  DBuf<double> part(g + 1, s);
  absdiff_partial<<<g, kET, 0, s>>>(a, na, b, nb, n, part.get());
  RK_LAUNCH_CHECK();
  sum_in_order<<<1, 32, 0, s>>>(part.get(), g, part.get() + g);
  RK_LAUNCH_CHECK();
  double r = 0.0;
  RK_CUDA_CHECK(cudaMemcpyAsync(&r, part.get() + g, sizeof r, cudaMemcpyDeviceToHost, s));
  RK_CUDA_CHECK(cudaStreamSynchronize(s));
  return r;
}

void align_signs_device(Ctx& c, const double* hat, const double* ref, uint64_t rows, uint64_t cols,
                        const double* sigma_ref, uint64_t n_sigma, double* out) {
  cudaStream_t s = c.stream;
  if (n_sigma && n_sigma != cols) fail(RK_INVALID_ARGUMENT, "align_signs: sigma length mismatch");
  if (!rows || !cols) return;
  DBuf<double> dots(cols, s);
  column_dots<<<grid_of(cols, 1u << 20), kET, 0, s>>>(hat, ref, rows, cols, dots.get());
  RK_LAUNCH_CHECK();
  apply_flips<<<grid_of(rows * cols), kET, 0, s>>>(hat, dots.get(), rows, cols, out);
  RK_LAUNCH_CHECK();
  if (!n_sigma) return;
  // clusters from sigma_ref on the host (n_sigma doubles), as metrics.cpp:59-70
  std::vector<double> sg(n_sigma);
  RK_CUDA_CHECK(cudaMemcpyAsync(sg.data(), sigma_ref, n_sigma * sizeof(double), cudaMemcpyDeviceToHost, s));
  RK_CUDA_CHECK(cudaStreamSynchronize(s));
  double smax = 0.0;
  for (double x : sg) smax = std::max(smax, x);
  const double gap_tol = 1e-9 * smax;  // kClusterTol, metrics.cpp:15
  uint64_t lo = 0;
  while (lo < cols) {
    uint64_t hi = lo + 1;
    while (hi < cols && std::fabs(sg[hi - 1] - sg[hi]) <= gap_tol) ++hi;
    if (hi - lo > 1) {
      const uint32_t cn = (uint32_t)(hi - lo);
      DBuf<double> C((uint64_t)cn * cn, s), W((uint64_t)cn * cn, s);
      cluster_cross<<<grid_of((uint64_t)cn * cn, 1u << 20), kET, 0, s>>>(hat, ref, rows, cols, lo, cn, C.get());
      RK_LAUNCH_CHECK();
      DenseSvdOut sv;
      dense_svd_dev(c, C.get(), cn, cn, sv);
      procrustes_w<<<grid_of((uint64_t)cn * cn, 1u << 20), kET, 0, s>>>(sv.u.get(), sv.v.get(), cn, W.get());
      RK_LAUNCH_CHECK();
      cluster_apply<<<grid_of(rows * cn), kET, 0, s>>>(hat, W.get(), rows, cols, lo, cn, out);
      RK_LAUNCH_CHECK();
    }
    lo = hi;
  }
}

double left_vector_error_device(Ctx& c, const double* hat, const double* ref, uint64_t rows, uint64_t cols,
                                const double* sigma_ref, uint64_t n_sigma) {
  cudaStream_t s = c.stream;
  DBuf<double> al(rows * cols ? rows * cols : 1, s);
  align_signs_device(c, hat, ref, rows, cols, sigma_ref, n_sigma, al.get());
  return sigma_error_device(al.get(), rows * cols, ref, rows * cols, s);
}

uint64_t numerical_rank_device(Ctx& c, const double* a, uint64_t rows, uint64_t cols, double tol) {
  if (rows > 0xffffffffull || cols > 0xffffffffull) fail(RK_INVALID_ARGUMENT, "numerical_rank: matrix too large");
  DenseSvdOut sv;
  dense_svd_dev(c, a, (uint32_t)rows, (uint32_t)cols, sv);
  if (sv.k == 0) return 0;
  std::vector<double> sg(sv.k);
  RK_CUDA_CHECK(cudaMemcpyAsync(sg.data(), sv.sigma.get(), sv.k * sizeof(double), cudaMemcpyDeviceToHost, c.stream));
  RK_CUDA_CHECK(cudaStreamSynchronize(c.stream));
  const double threshold = tol * sg.front();
  uint64_t rank = 0;
  for (double x : sg)
    if (x > threshold && x > 0.0) ++rank;
  return rank;
}

}  // namespace rk
