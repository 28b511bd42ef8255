// rk_qr.cu -- batched blocked Householder QR of tall column-major FP64 matrices
// (reference: householder_qr, proj/src/svd.cpp:77-107).
//
// One thread-block cluster per matrix (cluster size 1 when the batch alone
// fills the GPU). For every panel of NB columns:
//   * rank 0 stages the panel (rows k0..m-1) in shared memory, factors it with
//     unblocked Householder steps (one CTA reduction for the norm, one for all
//     dots of the step) and builds the compact-WY factor T (LAPACK dlarft,
//     forward/columnwise), then writes the reflectors back in place (v0 on the
//     diagonal, R's diagonal to job.diag);
//   * every CTA of the cluster loads V and T into its own shared memory and
//     updates its share of the trailing column tiles, C -= V (T^T (V^T C)), one
//     warp per tile of 4 columns with register accumulators and V read from
//     shared memory.
// The reflector convention is the reference's: alpha = -sign(x0) ||x||,
// v = x - alpha e1, beta = 2 / ||v||^2, beta = 0 for a zero column. NB is a
// template parameter chosen from the matrix height so the panel fits in smem.
#include <cooperative_groups.h>

#include <algorithm>

#include "rk_internal.cuh"

namespace cg = cooperative_groups;

namespace rk {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kTile = 4;

__device__ __forceinline__ double wsum(double x) {
#pragma unroll
  for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

// CTA-wide sums of the first n of N per-thread values -> s_out[0..n)
template <int N>
__device__ __forceinline__ void block_sums(const double (&v)[N], int n, double* s_part, double* s_out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < N; ++q) {
    if (q < n) {
      const double x = wsum(v[q]);
      if (lane == 0) s_part[warp * N + q] = x;
    }
  }
  __syncthreads();
  if (threadIdx.x < n) {
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) t += s_part[w * N + threadIdx.x];
    s_out[threadIdx.x] = t;
  }
  __syncthreads();
}

template <int NB>
__global__ void __launch_bounds__(kThreads, 1) qr_kernel(const QrJob* __restrict__ jobs) {
  extern __shared__ __align__(16) double sm[];
  cg::cluster_group cluster = cg::this_cluster();
  const unsigned rank = cluster.block_rank(), csize = cluster.num_blocks();
  const QrJob job = jobs[blockIdx.x / csize];
  double* __restrict__ A = job.a;
  const uint64_t lda = job.lda;
  const int m = (int)job.m, n = (int)job.n;
  const int K = m < n ? m : n;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  double* P = sm;                        // NB x m, column-major (ld m); local row i = global row k0+i
  double* sT = P + (size_t)NB * m;       // NB x NB, T(r, c) at r * NB + c
  double* s_part = sT + NB * NB;         // kWarps x NB
  double* s_red = s_part + kWarps * NB;  // NB
  __shared__ double s_beta;

  auto csync = [&]() {
    if (csize > 1) cluster.sync();
    else __syncthreads();
  };

  for (int k0 = 0; k0 < K; k0 += NB) {
    const int nbk = min(NB, K - k0);
    const int h = m - k0;
    double* tglob = job.tmat + (uint64_t)(k0 / NB) * NB * NB;
    if (rank == 0) {
      for (int q = 0; q < nbk; ++q) {
        const double* src = A + (uint64_t)(k0 + q) * lda + k0;
        for (int i = tid; i < h; i += kThreads) P[q * m + i] = __ldcg(src + i);
      }
      for (int t = tid; t < NB * NB; t += kThreads) sT[t] = 0.0;
      __syncthreads();
      for (int jj = 0; jj < nbk; ++jj) {
        double* pj = P + jj * m;
        double nrm[1] = {0.0};
        for (int i = jj + tid; i < h; i += kThreads) nrm[0] += pj[i] * pj[i];
        block_sums<1>(nrm, 1, s_part, s_red);
        if (tid == 0) {
          const double norm2 = s_red[0];
          double beta = 0.0, alpha = 0.0;
          if (norm2 > 0.0) {
            const double norm = sqrt(norm2);
            const double x0 = pj[jj];
            alpha = x0 >= 0.0 ? -norm : norm;
            beta = 2.0 / (2.0 * norm * (norm + fabs(x0)));  // ||x - alpha e1||^2 = 2 norm (norm + |x0|)
            pj[jj] = x0 - alpha;
          } else {
            pj[jj] = 0.0;  // identity reflector
          }
          job.diag[k0 + jj] = alpha;
          job.beta[k0 + jj] = beta;
          s_beta = beta;
        }
        __syncthreads();
        const double beta = s_beta;
        if (beta == 0.0) continue;
        // dots with the panel columns to the right and with the earlier reflectors (for T)
        const int n_after = nbk - 1 - jj, n_vals = nbk - 1;
        double acc[NB];
#pragma unroll
        for (int q = 0; q < NB; ++q) acc[q] = 0.0;
        for (int i = jj + tid; i < h; i += kThreads) {
          const double vi = pj[i];
#pragma unroll
          for (int q = 0; q < NB; ++q) {
            if (q < n_after) acc[q] += vi * P[(jj + 1 + q) * m + i];
            else if (q < n_vals) acc[q] += vi * P[(q - n_after) * m + i];
          }
        }
        block_sums<NB>(acc, n_vals, s_part, s_red);
        for (int i = jj + tid; i < h; i += kThreads) {
          const double vi = pj[i];
          for (int q = 0; q < n_after; ++q) P[(jj + 1 + q) * m + i] -= beta * s_red[q] * vi;
        }
        // T(0:jj, jj) = -beta T(0:jj, 0:jj) z, T(jj, jj) = beta
        if (tid < jj) {
          double t = 0.0;
          for (int s = tid; s < jj; ++s) t += sT[tid * NB + s] * s_red[n_after + s];
          s_part[tid] = -beta * t;
        }
        __syncthreads();
        if (tid < jj) sT[tid * NB + jj] = s_part[tid];
        if (tid == 0) sT[jj * NB + jj] = beta;
        __syncthreads();
      }
      for (int q = 0; q < nbk; ++q) {
        double* dst = A + (uint64_t)(k0 + q) * lda + k0;
        for (int i = tid; i < h; i += kThreads) dst[i] = P[q * m + i];
      }
      if (csize > 1)
        for (int t = tid; t < NB * NB; t += kThreads) tglob[t] = sT[t];
    }
    csync();
    if (rank != 0) {
      for (int q = 0; q < nbk; ++q) {
        const double* src = A + (uint64_t)(k0 + q) * lda + k0;
        for (int i = tid; i < h; i += kThreads) P[q * m + i] = __ldcg(src + i);
      }
      for (int t = tid; t < NB * NB; t += kThreads) sT[t] = __ldcg(tglob + t);
      __syncthreads();
    }
    // ---- trailing update: C = C - V (T^T (V^T C)) on columns >= k0 + nbk ----
    const int c0 = k0 + nbk;
    const int ntiles = (n - c0 + kTile - 1) / kTile;
    for (int tile = rank * kWarps + warp; tile < ntiles; tile += csize * kWarps) {
      const int j0 = c0 + tile * kTile;
      double acc[NB][kTile];
#pragma unroll
      for (int r = 0; r < NB; ++r)
#pragma unroll
        for (int q = 0; q < kTile; ++q) acc[r][q] = 0.0;
      double* cb[kTile];
#pragma unroll
      for (int q = 0; q < kTile; ++q) cb[q] = A + (uint64_t)min(j0 + q, n - 1) * lda + k0;
      for (int i = lane; i < h; i += 32) {
        double c[kTile];
#pragma unroll
        for (int q = 0; q < kTile; ++q) c[q] = (j0 + q < n) ? __ldcg(cb[q] + i) : 0.0;
#pragma unroll
        for (int r = 0; r < NB; ++r) {
          const double vr = (r < nbk && i >= r) ? P[r * m + i] : 0.0;
#pragma unroll
          for (int q = 0; q < kTile; ++q) acc[r][q] += vr * c[q];
        }
      }
#pragma unroll
      for (int r = 0; r < NB; ++r)
#pragma unroll
        for (int q = 0; q < kTile; ++q) acc[r][q] = wsum(acc[r][q]);
#pragma unroll
      for (int r = NB - 1; r >= 0; --r) {
#pragma unroll
        for (int q = 0; q < kTile; ++q) {
          double t = 0.0;
#pragma unroll
          for (int s = 0; s <= r; ++s) t += sT[s * NB + r] * acc[s][q];
          acc[r][q] = t;
        }
      }
      for (int i = lane; i < h; i += 32) {
        double c[kTile];
#pragma unroll
        for (int q = 0; q < kTile; ++q) c[q] = (j0 + q < n) ? __ldcg(cb[q] + i) : 0.0;
#pragma unroll
        for (int r = 0; r < NB; ++r) {
          const double vr = (r < nbk && i >= r) ? P[r * m + i] : 0.0;
#pragma unroll
          for (int q = 0; q < kTile; ++q) c[q] -= vr * acc[r][q];
        }
#pragma unroll
        for (int q = 0; q < kTile; ++q)
          if (j0 + q < n) cb[q][i] = c[q];
      }
    }
    csync();
  }
}

template <int NB>
size_t qr_smem(uint32_t m) {
  return ((size_t)NB * m + NB * NB + kWarps * NB + NB) * sizeof(double);
}

template <int NB>
void launch_qr(const std::vector<QrJob>& jobs, const QrJob* d_jobs, unsigned cl, uint32_t m_max, cudaStream_t s) {
  const size_t smem = qr_smem<NB>(m_max);
  RK_CUDA_CHECK(cudaFuncSetAttribute(qr_kernel<NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  RK_CUDA_CHECK(cudaFuncSetAttribute(qr_kernel<NB>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  const void* args[] = {&d_jobs};
  launch_cluster_kernel((const void*)qr_kernel<NB>, (unsigned)jobs.size() * cl, cl, kThreads, smem, s,
                        const_cast<void**>(args));
}

}  // namespace

uint32_t qr_max_rows() { return 5120; }

void qr_batched(const std::vector<QrJob>& jobs, cudaStream_t s, int sms) {
  if (jobs.empty()) return;
  uint32_t m_max = 0, widest = 0;
  for (const QrJob& j : jobs) {
    m_max = std::max(m_max, j.m);
    widest = std::max(widest, j.n);
  }
  if (m_max > qr_max_rows()) fail(RK_RUNTIME, "qr_batched: matrix taller than a panel can stage");
  unsigned cl = (unsigned)std::max<uint64_t>(1, (uint64_t)(2 * sms) / jobs.size());
  const unsigned useful = std::max(1u, (widest / kTile + kWarps - 1) / kWarps);
  cl = std::min({cl, 8u, useful});
  unsigned p2 = 1;
  while (p2 * 2 <= cl) p2 *= 2;
  cl = p2;
  DBuf<QrJob> dj(jobs.size(), s);
  to_device(dj.get(), jobs.data(), jobs.size(), s);
  const QrJob* d = dj.get();
  const size_t budget = 200 * 1024;
  if (qr_smem<16>(m_max) <= budget) launch_qr<16>(jobs, d, cl, m_max, s);
  else if (qr_smem<8>(m_max) <= budget) launch_qr<8>(jobs, d, cl, m_max, s);
  else launch_qr<4>(jobs, d, cl, m_max, s);
}

}  // namespace rk
