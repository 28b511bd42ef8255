// rk_dense.cu -- batched dense FP64 factorizations on sm_100a.
//
//  qr_cluster_kernel   blocked Householder QR (reference: householder_qr,
//                      proj/src/svd.cpp:77-107) of a tall column-major matrix,
//                      one thread-block cluster per matrix. Compact-WY panels of
//                      NB reflectors (LAPACK dlarft form); rank 0 factors each
//                      panel, every CTA of the cluster updates its share of the
//                      trailing column tiles; cluster barriers separate phases.
//  jacobi_cluster_kernel
//                      one-sided (Hestenes) Jacobi (reference: jacobi_svd,
//                      proj/src/svd.cpp:214-306) with the same rotation formulas,
//                      thresholds (kJacobiTol=1e-14, freeze at tol^2*alpha_max),
//                      alpha bookkeeping and convergence rule (a sweep with no
//                      rotation; 60-sweep cap -> ConvergenceError). The cyclic
//                      pair order is replaced by a parallel block ordering: the
//                      columns form G groups of g; a round-robin tournament pairs
//                      groups, each CTA stages a group pair in shared memory and
//                      sweeps all its column pairs in g disjoint-pair rounds,
//                      one warp per pair with warp-shuffle dot products.
//  finalize_kernel     sigma = column norms, stable descending order, u = w/sigma,
//                      sign convention (svd.cpp:336-354), block-record payload u*sigma
//                      (block_record.cpp:69-84).
//  complete_kernel     orthonormal completion of deficient columns (svd.cpp:150-201).
//  apply_q_kernel      Q [x; 0] from stored reflectors (svd.cpp:111-132).
#include <cooperative_groups.h>

#include <algorithm>

#include "rk_internal.cuh"

namespace cg = cooperative_groups;

namespace rk {
namespace {

constexpr double kJacobiTol = 1e-14;
constexpr int kMaxSweeps = 60;
constexpr double kRankTol = 1e-10;

__device__ __forceinline__ double warp_sum(double x) {
#pragma unroll
  for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

// ===========================================================================
// QR
// ===========================================================================

constexpr int kQrThreads = 256;
constexpr int kQrWarps = kQrThreads / 32;
constexpr int NB = 16;      // reflectors per panel
constexpr int kTileCols = 4;

struct QrArgs {
  const QrJob* jobs;
};

// CTA-wide sum of up to NB values held per thread; result broadcast via smem
__device__ __forceinline__ void block_sum_vec(double* vals, int n, double* s_part, double* s_out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < NB; ++q) {
    if (q < n) {
      double x = warp_sum(vals[q]);
      if (lane == 0) s_part[warp * NB + q] = x;
    }
  }
  __syncthreads();
  if (threadIdx.x < n) {
    double t = 0.0;
    for (int w = 0; w < kQrWarps; ++w) t += s_part[w * NB + threadIdx.x];
    s_out[threadIdx.x] = t;
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kQrThreads) qr_cluster_kernel(QrArgs args) {
  cg::cluster_group cluster = cg::this_cluster();
  const unsigned rank = cluster.block_rank(), csize = cluster.num_blocks();
  const QrJob job = args.jobs[blockIdx.x / csize];
  double* __restrict__ A = job.a;
  const uint64_t lda = job.lda;
  const int m = (int)job.m, n = (int)job.n;
  const int K = m < n ? m : n;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  __shared__ double s_part[kQrWarps * NB];
  __shared__ double s_red[NB];
  __shared__ double s_T[NB * NB];  // T(r, c) at [r * NB + c], upper triangular
  __shared__ double s_beta;

  for (int k0 = 0; k0 < K; k0 += NB) {
    const int nbk = min(NB, K - k0);
    double* tglob = job.tmat + (uint64_t)(k0 / NB) * NB * NB;
    if (rank == 0) {
      // ---- panel factorization (unblocked, columns k0 .. k0+nbk-1) ----
      for (int t = tid; t < NB * NB; t += kQrThreads) s_T[t] = 0.0;
      for (int jj = 0; jj < nbk; ++jj) {
        const int kk = k0 + jj;
        double* ak = A + (uint64_t)kk * lda;
        double part[NB];
        part[0] = 0.0;
        for (int i = kk + tid; i < m; i += kQrThreads) {
          double x = __ldcg(ak + i);
          part[0] += x * x;
        }
        block_sum_vec(part, 1, s_part, s_red);
        if (tid == 0) {
          const double norm2 = s_red[0];
          double beta = 0.0, alpha = 0.0;
          if (norm2 > 0.0) {
            const double norm = sqrt(norm2);
            const double x0 = __ldcg(ak + kk);
            alpha = x0 >= 0.0 ? -norm : norm;
            const double v0 = x0 - alpha;
            const double vsq = 2.0 * norm * (norm + fabs(x0));  // = ||x - alpha e1||^2
            beta = 2.0 / vsq;
            ak[kk] = v0;  // v stored in place, v0 on the diagonal
          }
          job.diag[kk] = alpha;  // R(kk, kk); 0 for a zero column
          job.beta[kk] = beta;
          s_beta = beta;
        }
        __syncthreads();
        const double beta = s_beta;
        if (beta != 0.0) {
          // one reduction: dots with the remaining panel columns (kk+1 ..) and
          // with the earlier reflectors of this panel (for T)
          const int n_after = nbk - 1 - jj;
          const int n_vals = n_after + jj;
          double acc[NB];
#pragma unroll
          for (int q = 0; q < NB; ++q) acc[q] = 0.0;
          for (int i = kk + tid; i < m; i += kQrThreads) {
            const double vi = __ldcg(ak + i);
#pragma unroll
            for (int q = 0; q < NB; ++q) {
              if (q < n_after) acc[q] += vi * __ldcg(A + (uint64_t)(kk + 1 + q) * lda + i);
              else if (q < n_vals) acc[q] += vi * __ldcg(A + (uint64_t)(k0 + q - n_after) * lda + i);
            }
          }
          block_sum_vec(acc, n_vals, s_part, s_red);
          // apply H to the remaining panel columns
          for (int i = kk + tid; i < m; i += kQrThreads) {
            const double vi = __ldcg(ak + i);
            for (int q = 0; q < n_after; ++q) {
              double* aj = A + (uint64_t)(kk + 1 + q) * lda;
              aj[i] = __ldcg(aj + i) - beta * s_red[q] * vi;
            }
          }
          // T(0:jj, jj) = -beta T(0:jj,0:jj) z,  T(jj,jj) = beta  (dlarft, forward columnwise)
          if (tid < jj) {
            double t = 0.0;
            for (int s = tid; s < jj; ++s) t += s_T[tid * NB + s] * s_red[n_after + s];
            s_part[tid] = -beta * t;  // reuse scratch (after the reduction consumed it)
          }
          __syncthreads();
          if (tid < jj) s_T[tid * NB + jj] = s_part[tid];
          if (tid == 0) s_T[jj * NB + jj] = beta;
          __syncthreads();
        } else {
          // identity reflector: v = 0 (the column below the diagonal is zero)
          if (tid == 0) ak[kk] = 0.0;
          __syncthreads();
        }
      }
      for (int t = tid; t < NB * NB; t += kQrThreads) tglob[t] = s_T[t];
    }
    cluster.sync();
    if (rank != 0) {
      for (int t = tid; t < NB * NB; t += kQrThreads) s_T[t] = __ldcg(tglob + t);
      __syncthreads();
    }
    // ---- trailing update: C = (I - V T V^T)^T C for columns >= k0 + nbk ----
    const int c0 = k0 + nbk;
    const int ntiles = (n - c0 + kTileCols - 1) / kTileCols;
    for (int tile = rank * kQrWarps + warp; tile < ntiles; tile += csize * kQrWarps) {
      const int j0 = c0 + tile * kTileCols;
      double acc[NB][kTileCols];
#pragma unroll
      for (int r = 0; r < NB; ++r)
#pragma unroll
        for (int q = 0; q < kTileCols; ++q) acc[r][q] = 0.0;
      for (int i = k0 + lane; i < m; i += 32) {
        double vr[NB];
#pragma unroll
        for (int r = 0; r < NB; ++r)
          vr[r] = (r < nbk && i >= k0 + r) ? __ldcg(A + (uint64_t)(k0 + r) * lda + i) : 0.0;
#pragma unroll
        for (int q = 0; q < kTileCols; ++q) {
          const double c = (j0 + q < n) ? __ldcg(A + (uint64_t)(j0 + q) * lda + i) : 0.0;
#pragma unroll
          for (int r = 0; r < NB; ++r) acc[r][q] += vr[r] * c;
        }
      }
#pragma unroll
      for (int r = 0; r < NB; ++r)
#pragma unroll
        for (int q = 0; q < kTileCols; ++q) acc[r][q] = warp_sum(acc[r][q]);
      // W' = T^T W, in place from the bottom row up
#pragma unroll
      for (int r = NB - 1; r >= 0; --r) {
#pragma unroll
        for (int q = 0; q < kTileCols; ++q) {
          double t = 0.0;
#pragma unroll
          for (int s = 0; s <= r; ++s) t += s_T[s * NB + r] * acc[s][q];
          acc[r][q] = t;
        }
      }
      for (int i = k0 + lane; i < m; i += 32) {
        double vr[NB];
#pragma unroll
        for (int r = 0; r < NB; ++r)
          vr[r] = (r < nbk && i >= k0 + r) ? __ldcg(A + (uint64_t)(k0 + r) * lda + i) : 0.0;
#pragma unroll
        for (int q = 0; q < kTileCols; ++q) {
          if (j0 + q < n) {
            double* cp = A + (uint64_t)(j0 + q) * lda + i;
            double c = __ldcg(cp);
#pragma unroll
            for (int r = 0; r < NB; ++r) c -= vr[r] * acc[r][q];
            *cp = c;
          }
        }
      }
    }
    cluster.sync();
  }
}

// R (rows < K) from a factored job into W (n x n col-major): transpose ? R^T : R
__global__ void r_extract_kernel(const RJob* jobs, bool transpose) {
  const RJob j = jobs[blockIdx.y];
  const uint32_t n = j.n, K = j.m < j.n ? j.m : j.n;
  const uint64_t total = (uint64_t)n * n;
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < total;
       t += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t i = (uint32_t)(t % n), c = (uint32_t)(t / n);  // W(i, c)
    const uint32_t r = transpose ? c : i, col = transpose ? i : c;  // R(r, col)
    double x = 0.0;
    if (r < K) {
      if (col > r) x = j.a[r + (uint64_t)col * j.lda];
      else if (col == r) x = j.diag[r];
    }
    j.w[i + c * j.ldw] = x;
  }
}

// ===========================================================================
// Jacobi
// ===========================================================================

constexpr int kJThreads = 256;
constexpr int kJWarps = kJThreads / 32;

struct JacobiParams {
  const JacobiJob* jobs;
  uint32_t g;       // columns per group (even)
  uint32_t G;       // groups (even), G * g = cols_pad
  int with_v;
};

__device__ __forceinline__ uint32_t rr_slot(uint32_t pos, uint32_t step, uint32_t n) {
  // round-robin tournament: position 0 fixed, the rest rotate
  return pos == 0 ? 0 : 1 + (pos - 1 + step) % (n - 1);
}

// rotate one pair (p, q) of staged columns; returns 1 when rotated
__device__ __forceinline__ int rotate_pair(double* __restrict__ wp, double* __restrict__ wq, double* vp, double* vq,
                                           uint32_t rows, uint32_t vrows, double* alpha, int p, int q,
                                           double freeze, double& max_ratio) {
  const int lane = threadIdx.x & 31;
  const double ap = alpha[p], aq = alpha[q];
  if (ap <= freeze || aq <= freeze) return 0;
  double g = 0.0;
  for (uint32_t i = lane; i < rows; i += 32) g += wp[i] * wq[i];
  const double gamma = warp_sum(g);
  const double ratio = fabs(gamma) / sqrt(ap * aq);
  max_ratio = fmax(max_ratio, ratio);
  if (ratio <= kJacobiTol) return 0;
  const double zeta = (aq - ap) / (2.0 * gamma);
  const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
  const double c = 1.0 / sqrt(1.0 + t * t);
  const double s = c * t;
  for (uint32_t i = lane; i < rows; i += 32) {
    const double xp = wp[i], xq = wq[i];
    wp[i] = c * xp - s * xq;
    wq[i] = s * xp + c * xq;
  }
  if (vp) {
    for (uint32_t i = lane; i < vrows; i += 32) {
      const double xp = vp[i], xq = vq[i];
      vp[i] = c * xp - s * xq;
      vq[i] = s * xp + c * xq;
    }
  }
  __syncwarp();
  if (lane == 0) {
    const double na = c * c * ap - 2.0 * c * s * gamma + s * s * aq;
    const double nq = s * s * ap + 2.0 * c * s * gamma + c * c * aq;
    alpha[p] = na > 0.0 ? na : 0.0;
    alpha[q] = nq > 0.0 ? nq : 0.0;
  }
  __syncwarp();
  return 1;
}

__global__ void __launch_bounds__(kJThreads) jacobi_cluster_kernel(JacobiParams P) {
  extern __shared__ __align__(16) double smem[];
  cg::cluster_group cluster = cg::this_cluster();
  const unsigned rank = cluster.block_rank(), csize = cluster.num_blocks();
  const JacobiJob job = P.jobs[blockIdx.x / csize];
  const uint32_t rows = job.rows, cols_pad = job.cols_pad;
  const uint32_t g = P.g, G = P.G;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool with_v = P.with_v && job.v;
  const uint32_t vrows = cols_pad;

  double* sW = smem;                                    // 2g columns x rows
  double* sV = sW + (uint64_t)2 * g * rows;             // 2g columns x vrows (optional)
  double* sAlpha = sV + (with_v ? (uint64_t)2 * g * vrows : 0);  // 2g
  __shared__ double s_red[kJWarps];
  __shared__ double s_amax;
  __shared__ unsigned long long s_rot;
  __shared__ double s_maxratio;

  unsigned long long* counters = reinterpret_cast<unsigned long long*>(job.stats + 4);  // [3] rotations per sweep mod 3
  double* W = job.w;
  double* V = job.v;
  double* alpha_g = job.alpha;

  unsigned long long total_rot = 0;
  double last_max_ratio = 0.0;
  int converged = (job.cols < 2);
  int sweep = 0;
  for (; sweep < kMaxSweeps && !converged; ++sweep) {
    // ---- column norms (fresh each sweep, svd.cpp:222-226) ----
    for (uint32_t j = rank * kJWarps + warp; j < cols_pad; j += csize * kJWarps) {
      const double* wj = W + (uint64_t)j * rows;
      double a = 0.0;
      for (uint32_t i = lane; i < rows; i += 32) {
        const double x = __ldcg(wj + i);
        a += x * x;
      }
      a = warp_sum(a);
      if (lane == 0) alpha_g[j] = a;
    }
    if (rank == 0 && tid == 0) counters[(sweep + 1) % 3] = 0ull;
    cluster.sync();
    double amax = 0.0;
    for (uint32_t j = tid; j < cols_pad; j += kJThreads) amax = fmax(amax, __ldcg(alpha_g + j));
    for (int o = 16; o; o >>= 1) amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    if (lane == 0) s_red[warp] = amax;
    if (tid == 0) { s_rot = 0ull; s_maxratio = 0.0; }
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
      for (int w = 0; w < kJWarps; ++w) t = fmax(t, s_red[w]);
      s_amax = t;
    }
    __syncthreads();
    const double freeze = kJacobiTol * kJacobiTol * s_amax;
    unsigned long long my_rot = 0;
    double my_ratio = 0.0;

    for (uint32_t step = 0; step + 1 < G; ++step) {
      for (uint32_t pi = rank; pi < G / 2; pi += csize) {
        const uint32_t gA = rr_slot(pi, step, G), gB = rr_slot(G - 1 - pi, step, G);
        // stage the two groups: slots 0..g-1 = group A, g..2g-1 = group B
        for (uint32_t c = warp; c < 2 * g; c += kJWarps) {
          const uint32_t col = (c < g ? gA * g + c : gB * g + (c - g));
          const double* src = W + (uint64_t)col * rows;
          double* dst = sW + (uint64_t)c * rows;
          for (uint32_t i = lane; i < rows; i += 32) dst[i] = __ldcg(src + i);
          if (with_v) {
            const double* vs = V + (uint64_t)col * vrows;
            double* vd = sV + (uint64_t)c * vrows;
            for (uint32_t i = lane; i < vrows; i += 32) vd[i] = __ldcg(vs + i);
          }
          if (lane == 0) sAlpha[c] = __ldcg(alpha_g + col);
        }
        __syncthreads();
        // intra-group rounds (first step only: every group appears once)
        if (step == 0) {
          for (uint32_t r = 0; r + 1 < g; ++r) {
            for (uint32_t t = warp; t < g; t += kJWarps) {
              const uint32_t half = g / 2;
              const uint32_t grp = t / half, i = t % half;
              const uint32_t p = grp * g + rr_slot(i, r, g), q = grp * g + rr_slot(g - 1 - i, r, g);
              double* vp = with_v ? sV + (uint64_t)p * vrows : nullptr;
              double* vq = with_v ? sV + (uint64_t)q * vrows : nullptr;
              int rot = rotate_pair(sW + (uint64_t)p * rows, sW + (uint64_t)q * rows, vp, vq, rows, vrows, sAlpha,
                                    p, q, freeze, my_ratio);
              my_rot += (lane == 0) ? rot : 0;
            }
            __syncthreads();
          }
        }
        // cross rounds: (A_i, B_{(i + r) mod g})
        for (uint32_t r = 0; r < g; ++r) {
          for (uint32_t i = warp; i < g; i += kJWarps) {
            const uint32_t p = i, q = g + (i + r) % g;
            double* vp = with_v ? sV + (uint64_t)p * vrows : nullptr;
            double* vq = with_v ? sV + (uint64_t)q * vrows : nullptr;
            int rot = rotate_pair(sW + (uint64_t)p * rows, sW + (uint64_t)q * rows, vp, vq, rows, vrows, sAlpha, p,
                                  q, freeze, my_ratio);
            my_rot += (lane == 0) ? rot : 0;
          }
          __syncthreads();
        }
        // write back
        for (uint32_t c = warp; c < 2 * g; c += kJWarps) {
          const uint32_t col = (c < g ? gA * g + c : gB * g + (c - g));
          double* dst = W + (uint64_t)col * rows;
          const double* src = sW + (uint64_t)c * rows;
          for (uint32_t i = lane; i < rows; i += 32) dst[i] = src[i];
          if (with_v) {
            double* vd = V + (uint64_t)col * vrows;
            const double* vs = sV + (uint64_t)c * vrows;
            for (uint32_t i = lane; i < vrows; i += 32) vd[i] = vs[i];
          }
          if (lane == 0) alpha_g[col] = sAlpha[c];
        }
        __syncthreads();
      }
      if (step + 2 == G) {
        // last step of the sweep: publish this CTA's rotation count and max ratio
        if (lane == 0 && my_rot) atomicAdd(&s_rot, my_rot);
        for (int o = 16; o; o >>= 1) my_ratio = fmax(my_ratio, __shfl_xor_sync(0xffffffffu, my_ratio, o));
        if (lane == 0) s_red[warp] = my_ratio;
        __syncthreads();
        if (tid == 0) {
          double t = 0.0;
          for (int w = 0; w < kJWarps; ++w) t = fmax(t, s_red[w]);
          if (s_rot) atomicAdd(&counters[sweep % 3], s_rot);
          // max ratio across the cluster: doubles >= 0 order like their bit patterns
          atomicMax(reinterpret_cast<unsigned long long*>(job.stats + 3), __double_as_longlong(t));
        }
      }
      cluster.sync();
    }
    const unsigned long long rot = __ldcg(&counters[sweep % 3]);
    total_rot += rot;
    last_max_ratio = __longlong_as_double(__ldcg(reinterpret_cast<long long*>(job.stats + 3)));
    cluster.sync();  // everyone has read the counters before the next sweep reuses the ratio slot
    if (rank == 0 && tid == 0) job.stats[3] = 0ull;
    if (rot == 0) converged = 1;
    cluster.sync();
  }
  if (rank == 0 && tid == 0) {
    job.stats[0] = (uint64_t)sweep;
    job.stats[1] = total_rot;
    job.stats[2] = converged ? 0ull : 1ull;
    job.stats[3] = (uint64_t)__double_as_longlong(last_max_ratio);
  }
}

// ===========================================================================
// finalize
// ===========================================================================

constexpr int kFThreads = 512;

__global__ void __launch_bounds__(kFThreads) finalize_kernel(const FinalJob* jobs) {
  const FinalJob J = jobs[blockIdx.x];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int nw = kFThreads / 32;
  const uint32_t rows = J.rows, cols = J.cols;
  double* sig = J.scratch;
  // column norms (svd.cpp:271-272)
  for (uint32_t j = warp; j < cols; j += nw) {
    const double* wj = J.w + (uint64_t)j * rows;
    double a = 0.0;
    for (uint32_t i = lane; i < rows; i += 32) a += wj[i] * wj[i];
    a = warp_sum(a);
    if (lane == 0) sig[j] = sqrt(a);
  }
  __syncthreads();
  // stable descending order: rank = #greater + #equal before (svd.cpp:274-277)
  for (uint32_t j = tid; j < cols; j += kFThreads) {
    const double s = sig[j];
    uint32_t rnk = 0;
    for (uint32_t i = 0; i < cols; ++i) {
      const double t = sig[i];
      rnk += (t > s) || (t == s && i < j);
    }
    J.order[rnk] = j;
  }
  __syncthreads();
  const double smax = cols ? sig[J.order[0]] : 0.0;
  const double thr = kRankTol * smax;
  if (J.sigma_all)
    for (uint32_t j = tid; j < cols; j += kFThreads) J.sigma_all[j] = sig[J.order[j]];
  for (uint32_t j = warp; j < J.k; j += nw) {
    const uint32_t src = J.order[j];
    const double s = sig[src];
    const bool deficient = !(s > thr && s > 0.0);
    const double* wj = J.w + (uint64_t)src * rows;
    // sign convention on u = w / s: first index of the largest |u|
    double best = -1.0;
    uint32_t arg = 0;
    if (!deficient) {
      for (uint32_t i = lane; i < rows; i += 32) {
        const double mag = fabs(wj[i] / s);
        if (mag > best) { best = mag; arg = i; }
      }
      for (int o = 16; o; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const uint32_t oa = __shfl_xor_sync(0xffffffffu, arg, o);
        if (ob > best || (ob == best && oa < arg)) { best = ob; arg = oa; }
      }
    }
    const double flip = (!deficient && (wj[arg] / s) < 0.0) ? -1.0 : 1.0;
    if (J.sigma && lane == 0) J.sigma[j] = s;
    if (J.deficient && lane == 0) J.deficient[j] = deficient ? 1 : 0;
    for (uint32_t i = lane; i < rows; i += 32) {
      const double u = deficient ? 0.0 : flip * (wj[i] / s);
      if (J.u) J.u[(uint64_t)i * J.k + j] = u;
      if (J.payload) J.payload[(uint64_t)i * J.k + j] = deficient ? (s > 0.0 ? wj[i] : 0.0) : u * s;
    }
    if (J.v_out) {
      const double* vs = J.v_in + (uint64_t)src * J.ldv;
      for (uint32_t i = lane; i < cols; i += 32) J.v_out[(uint64_t)i * J.k + j] = flip * vs[i];
    }
  }
}

// ===========================================================================
// orthonormal completion (single warp, deterministic) -- svd.cpp:150-201
// u is row-major rows x cols
// ===========================================================================

__global__ void complete_kernel(double* u, uint32_t rows, uint32_t cols, const uint8_t* deficient, int* fail) {
  extern __shared__ double cw[];
  double* w = cw;
  double* best = cw + rows;
  const int lane = threadIdx.x;
  for (uint32_t j = 0; j < cols; ++j) {
    if (!deficient[j]) continue;
    double best_norm = -1.0;
    for (uint32_t cand = 0; cand < rows; ++cand) {
      for (uint32_t i = lane; i < rows; i += 32) w[i] = (i == cand) ? 1.0 : 0.0;
      __syncwarp();
      for (int pass = 0; pass < 2; ++pass) {
        for (uint32_t c = 0; c < cols; ++c) {
          if (deficient[c] && c >= j) continue;
          double d = 0.0;
          for (uint32_t i = lane; i < rows; i += 32) d += u[(uint64_t)i * cols + c] * w[i];
          d = warp_sum(d);
          for (uint32_t i = lane; i < rows; i += 32) w[i] -= d * u[(uint64_t)i * cols + c];
          __syncwarp();
        }
      }
      double nn = 0.0;
      for (uint32_t i = lane; i < rows; i += 32) nn += w[i] * w[i];
      const double wn = sqrt(warp_sum(nn));
      const bool take = wn > 0.5;
      if (take || wn > best_norm) {
        best_norm = wn;
        for (uint32_t i = lane; i < rows; i += 32) best[i] = w[i];
        __syncwarp();
      }
      if (take) break;
    }
    if (!(best_norm > 0.0)) {
      // no independent direction (svd.cpp:183-186)
      if (lane == 0) *fail = 1;
      return;
    }
    for (uint32_t i = lane; i < rows; i += 32) u[(uint64_t)i * cols + j] = best[i] / best_norm;
    __syncwarp();
    if (best_norm <= 0.5) {
      for (uint32_t c = 0; c < cols; ++c) {
        if (deficient[c] && c >= j) continue;
        double d = 0.0;
        for (uint32_t i = lane; i < rows; i += 32) d += u[(uint64_t)i * cols + c] * u[(uint64_t)i * cols + j];
        d = warp_sum(d);
        for (uint32_t i = lane; i < rows; i += 32) u[(uint64_t)i * cols + j] -= d * u[(uint64_t)i * cols + c];
        __syncwarp();
      }
      double nn = 0.0;
      for (uint32_t i = lane; i < rows; i += 32) nn += u[(uint64_t)i * cols + j] * u[(uint64_t)i * cols + j];
      const double wn = sqrt(warp_sum(nn));
      for (uint32_t i = lane; i < rows; i += 32) u[(uint64_t)i * cols + j] /= wn;
      __syncwarp();
    }
  }
}

// ===========================================================================
// apply_q: out(:, c) = H_0 ... H_{K-1} [x(:, c); 0] -- warp per column
// ===========================================================================

__global__ void apply_q_kernel(QrJob qr, const double* x, uint32_t x_rows, uint32_t ncols, double* out) {
  const int lane = threadIdx.x & 31;
  const uint32_t m = qr.m, K = qr.m < qr.n ? qr.m : qr.n;
  for (uint32_t c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; c < ncols;
       c += (gridDim.x * blockDim.x) >> 5) {
    double* o = out + (uint64_t)c * m;
    for (uint32_t i = lane; i < m; i += 32) o[i] = i < x_rows ? x[(uint64_t)c * x_rows + i] : 0.0;
    __syncwarp();
    for (int kk = (int)K - 1; kk >= 0; --kk) {
      const double beta = qr.beta[kk];
      if (beta == 0.0) continue;
      const double* v = qr.a + (uint64_t)kk * qr.lda;  // v0 on the diagonal, then below
      double d = 0.0;
      for (uint32_t i = kk + lane; i < m; i += 32) d += v[i] * o[i];
      d = warp_sum(d);
      const double bw = beta * d;
      for (uint32_t i = kk + lane; i < m; i += 32) o[i] -= bw * v[i];
      __syncwarp();
    }
  }
}

template <class K>
void launch_cluster(K kernel, unsigned grid, unsigned cluster, unsigned threads, size_t smem, cudaStream_t s,
                    void** args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid, 1, 1);
  cfg.blockDim = dim3(threads, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cluster;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  RK_CUDA_CHECK(cudaLaunchKernelExC(&cfg, (const void*)kernel, args));
  RK_LAUNCH_CHECK();
}

}  // namespace

void qr_batched(const std::vector<QrJob>& jobs, cudaStream_t s, int sms) {
  if (jobs.empty()) return;
  static bool configured = false;
  if (!configured) {
    RK_CUDA_CHECK(cudaFuncSetAttribute(qr_cluster_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    configured = true;
  }
  // cluster size: spread the batch over the SMs, at most 8 CTAs per matrix
  unsigned cl = (unsigned)std::max<uint64_t>(1, (uint64_t)(2 * sms) / jobs.size());
  unsigned widest = 0;
  for (const QrJob& j : jobs) widest = std::max(widest, j.n);
  const unsigned useful = std::max(1u, (widest / kTileCols + kQrWarps - 1) / kQrWarps);
  cl = std::min({cl, 8u, useful});
  unsigned p2 = 1;
  while (p2 * 2 <= cl) p2 *= 2;
  cl = p2;
  DBuf<QrJob> dj(jobs.size(), s);
  to_device(dj.get(), jobs.data(), jobs.size(), s);
  QrArgs args{dj.get()};
  void* kargs[] = {&args};
  launch_cluster(qr_cluster_kernel, (unsigned)jobs.size() * cl, cl, kQrThreads, 0, s, kargs);
}

void r_extract_batched(const std::vector<RJob>& jobs, bool transpose, cudaStream_t s) {
  if (jobs.empty()) return;
  DBuf<RJob> dj(jobs.size(), s);
  to_device(dj.get(), jobs.data(), jobs.size(), s);
  uint32_t nmax = 0;
  for (const RJob& j : jobs) nmax = std::max(nmax, j.n);
  unsigned gx = (unsigned)std::min<uint64_t>(ceil_div((uint64_t)nmax * nmax, 256), 4096);
  r_extract_kernel<<<dim3(std::max(gx, 1u), (unsigned)jobs.size()), 256, 0, s>>>(dj.get(), transpose);
  RK_LAUNCH_CHECK();
}

size_t jacobi_smem(uint32_t rows, uint32_t g, uint32_t cols_pad, bool with_v);

void jacobi_plan(uint32_t rows, uint32_t cols, bool with_v, size_t smem_budget, uint32_t& g, uint32_t& G) {
  // largest even group size (<= 32) whose two staged groups fit the shared-memory budget
  for (uint32_t gmax = 32; gmax >= 2; gmax -= 2) {
    G = (uint32_t)ceil_div(cols ? cols : 1, gmax);
    if (G < 2) G = 2;
    if (G & 1) ++G;
    g = (uint32_t)ceil_div(cols ? cols : 1, G);
    if (g & 1) ++g;
    if (g < 2) g = 2;
    if (jacobi_smem(rows, g, g * G, with_v) <= smem_budget) return;
  }
  fail(RK_INVALID_ARGUMENT, "Jacobi: a " + std::to_string(rows) + "-row matrix does not fit shared memory");
}

size_t jacobi_smem(uint32_t rows, uint32_t g, uint32_t cols_pad, bool with_v) {
  return (size_t)2 * g * rows * 8 + (with_v ? (size_t)2 * g * cols_pad * 8 : 0) + (size_t)2 * g * 8;
}

void jacobi_batched(std::vector<JacobiJob>& jobs, cudaStream_t s, int sms, size_t smem_optin) {
  if (jobs.empty()) return;
  // jobs in one launch share rows / cols_pad / with_v (the caller groups them);
  // the group layout is a function of (rows, cols_pad) only
  const uint32_t rows = jobs[0].rows, cols_pad = jobs[0].cols_pad;
  const bool with_v = jobs[0].v != nullptr;
  uint32_t g, G;
  const size_t budget = std::min<size_t>(smem_optin, 200 * 1024);
  jacobi_plan(rows, cols_pad, with_v, budget, g, G);
  for (JacobiJob& j : jobs) {
    if (j.rows != rows || j.cols_pad != cols_pad || (j.v != nullptr) != with_v)
      fail(RK_RUNTIME, "jacobi_batched: heterogeneous batch");
    if (j.cols > cols_pad) fail(RK_RUNTIME, "jacobi_batched: cols > cols_pad");
  }
  if (g * G != cols_pad) fail(RK_RUNTIME, "jacobi_batched: cols_pad is not a planned width");
  const size_t smem = jacobi_smem(rows, g, g * G, with_v);
  RK_CUDA_CHECK(cudaFuncSetAttribute(jacobi_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  RK_CUDA_CHECK(cudaFuncSetAttribute(jacobi_cluster_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  unsigned cl = (unsigned)std::max<uint64_t>(1, (uint64_t)sms / jobs.size());
  cl = std::min<unsigned>({cl, G / 2, 8u});
  unsigned p2 = 1;
  while (p2 * 2 <= cl) p2 *= 2;
  cl = p2;
  DBuf<JacobiJob> dj(jobs.size(), s);
  to_device(dj.get(), jobs.data(), jobs.size(), s);
  JacobiParams P{dj.get(), g, G, with_v ? 1 : 0};
  void* kargs[] = {&P};
  launch_cluster(jacobi_cluster_kernel, (unsigned)jobs.size() * cl, cl, kJThreads, smem, s, kargs);
}

uint32_t jacobi_cols_pad(uint32_t rows, uint32_t cols, bool with_v, size_t smem_optin) {
  // a width that re-plans to itself, so jacobi_batched can recover (g, G) from it
  uint32_t g, G, cp = cols;
  for (int it = 0; it < 16; ++it) {
    jacobi_plan(rows, cp, with_v, std::min<size_t>(smem_optin, 200 * 1024), g, G);
    if (g * G == cp) return cp;
    cp = g * G;
  }
  fail(RK_RUNTIME, "jacobi_cols_pad: no stable padded width");
}

void finalize_batched(const std::vector<FinalJob>& jobs, cudaStream_t s) {
  if (jobs.empty()) return;
  DBuf<FinalJob> dj(jobs.size(), s);
  to_device(dj.get(), jobs.data(), jobs.size(), s);
  finalize_kernel<<<(unsigned)jobs.size(), kFThreads, 0, s>>>(dj.get());
  RK_LAUNCH_CHECK();
}

void complete_columns_device(double* u, uint32_t rows, uint32_t cols, const uint8_t* deficient, int* d_fail,
                             cudaStream_t s) {
  const size_t smem = (size_t)2 * rows * 8;
  if (smem > 48 * 1024)
    RK_CUDA_CHECK(cudaFuncSetAttribute(complete_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  complete_kernel<<<1, 32, smem, s>>>(u, rows, cols, deficient, d_fail);
  RK_LAUNCH_CHECK();
}

void apply_q_device(const QrJob& qr, const double* x, uint32_t x_rows, uint32_t ncols, double* out, cudaStream_t s) {
  if (!ncols) return;
  unsigned grid = (unsigned)std::min<uint64_t>(ceil_div((uint64_t)ncols * 32, 256), 4096);
  apply_q_kernel<<<grid, 256, 0, s>>>(qr, x, x_rows, ncols, out);
  RK_LAUNCH_CHECK();
}

}  // namespace rk
