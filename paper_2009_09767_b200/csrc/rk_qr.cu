// rk_qr.cu -- batched blocked Householder QR of tall column-major FP64 matrices
// (reference: householder_qr, proj/src/svd.cpp:77-107).
//
// One CTA per matrix (a thread-block cluster per matrix when the batch is too
// small to fill the GPU). For every panel of NB columns:
//   * rank 0 stages the panel's active rows in shared memory and factors it with
//     unblocked Householder steps. Each step needs ONE CTA reduction: the norm of
//     x, the dots x^T a_j with the panel columns to the right and x^T V with the
//     earlier reflectors are reduced together, and the v-dots follow from
//     v^T y = x^T y - alpha y[0]. The compact-WY factor T (LAPACK dlarft,
//     forward/columnwise) is built on the fly;
//   * every CTA of the cluster updates its share of the trailing columns,
//     C -= V (T^T (V^T C)), one warp per 8-column tile with FP64 tensor-core
//     MMAs (mma.sync m8n8k4 f64 -> DMMA): V^T C accumulates in the MMA (no
//     shuffle reductions), T^T W goes through a warp-private smem tile, and
//     C - V W' is a second MMA pass with C as the accumulator.
//
// Row sets: a dense job factors rows k0..m-1 at panel k0. A "stacked" job
// (split > 0) is [R_a; R_b] with R_a an n x n upper triangle in rows [0, split)
// and R_b upper trapezoidal in rows [split, m): the reflector of column k only
// involves top row k and bottom rows 0..k, so panel k0 works on the top rows
// [k0, k0+nb) plus bottom rows [0, k0+nb) -- the TSQR combine costs ~2/3 n^3
// instead of 10/3 n^3 flops, with the same arithmetic as the dense kernel on
// the rows that are not identically zero.
//
// Reflector convention as the reference: alpha = -sign(x0) ||x||, v = x - alpha e1,
// beta = 2/||v||^2 (= 1/(||x|| (||x|| + |x0|))), beta = 0 for a zero column.
#include <cooperative_groups.h>

#include <algorithm>

#include "rk_internal.cuh"

namespace cg = cooperative_groups;

namespace rk {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kTileN = 8;  // columns per warp tile (MMA n)
constexpr int kKB = 8;     // k-steps (4 rows each) whose loads are issued together
constexpr int kRBq = 4;    // 8-row blocks whose loads are issued together

__device__ __forceinline__ double wsum(double x) {
#pragma unroll
  for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

// d (8x8 f64 accumulator fragment: 2 per lane) += a (8x4, 1 per lane) * b (4x8, 1 per lane)
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
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

struct Rows {  // local row i of the panel at k0 -> global row
  uint32_t top_cnt, top_base, bot_base;
  __device__ __forceinline__ uint32_t operator()(uint32_t i) const {
    return i < top_cnt ? top_base + i : bot_base + (i - top_cnt);
  }
};

template <int NB>
__global__ void __launch_bounds__(kThreads, 2) qr_kernel(const QrJob* __restrict__ jobs, uint32_t ldp) {
  extern __shared__ __align__(16) double sm[];
  cg::cluster_group cluster = cg::this_cluster();
  const unsigned rank = cluster.block_rank(), csize = cluster.num_blocks();
  const QrJob job = jobs[blockIdx.x / csize];
  double* __restrict__ A = job.a;
  const uint64_t lda = job.lda;
  const int m = (int)job.m, n = (int)job.n;
  const int split = (int)job.split;
  const int K = split ? n : (m < n ? m : n);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  double* P = sm;                        // NB x ldp, column-major: local row i of panel column q at q * ldp + i
  double* sT = P + (size_t)NB * ldp;     // NB x NB, T(r, c) at r * NB + c
  double* s_part = sT + NB * NB;         // kWarps x NB
  double* s_red = s_part + kWarps * NB;  // NB
  double* s_w = s_red + NB;              // kWarps x (NB x 8): per-warp W' tiles
  __shared__ double s_alpha, s_beta;

  auto csync = [&]() {
    if (csize > 1) cluster.sync();
    else __syncthreads();
  };

  for (int k0 = 0; k0 < K; k0 += NB) {
    const int nbk = min(NB, K - k0);
    Rows R;
    int h;
    if (split) {
      const int hb = min(k0 + nbk, m - split);
      R = {(uint32_t)nbk, (uint32_t)k0, (uint32_t)split};
      h = nbk + hb;
    } else {
      R = {(uint32_t)(m - k0), (uint32_t)k0, 0u};
      h = m - k0;
    }
    double* tglob = job.tmat + (uint64_t)(k0 / NB) * NB * NB;
    if (rank == 0) {
      for (int q = 0; q < nbk; ++q) {
        const double* src = A + (uint64_t)(k0 + q) * lda;
        for (int i = tid; i < h; i += kThreads) P[q * ldp + i] = __ldcg(src + R(i));
      }
      for (int t = tid; t < NB * NB; t += kThreads) sT[t] = 0.0;
      __syncthreads();
      for (int jj = 0; jj < nbk; ++jj) {
        double* pj = P + jj * ldp;
        const int n_after = nbk - 1 - jj;
        // x^T x, x^T a_{jj+1..}, x^T v_{0..jj-1} over local rows >= jj
        double acc[NB];
#pragma unroll
        for (int q = 0; q < NB; ++q) acc[q] = 0.0;
        for (int i = jj + tid; i < h; i += kThreads) {
          const double xi = pj[i];
          acc[0] += xi * xi;
#pragma unroll
          for (int q = 1; q < NB; ++q) {
            if (q <= n_after) acc[q] += xi * P[(jj + q) * ldp + i];
            else if (q < nbk) acc[q] += xi * P[(q - 1 - n_after) * ldp + i];
          }
        }
        block_sums<NB>(acc, nbk, s_part, s_red);
        if (tid == 0) {
          const double norm2 = s_red[0];
          double beta = 0.0, alpha = 0.0;
          const double x0 = pj[jj];
          if (norm2 > 0.0) {
            const double norm = sqrt(norm2);
            alpha = x0 >= 0.0 ? -norm : norm;
            beta = 1.0 / (norm * (norm + fabs(x0)));
            pj[jj] = x0 - alpha;
          }
          job.diag[k0 + jj] = alpha;
          job.beta[k0 + jj] = beta;
          s_alpha = alpha;
          s_beta = beta;
        }
        __syncthreads();
        const double beta = s_beta, alpha = s_alpha;
        if (beta == 0.0) continue;  // identity reflector, v = 0 (the column is zero from row jj)
        // w_q = v^T a = x^T a - alpha a[jj]; z_r = v^T v_r = x^T v_r - alpha v_r[jj]
        if (tid < n_after) s_part[tid] = s_red[1 + tid] - alpha * P[(jj + 1 + tid) * ldp + jj];
        if (tid >= NB && tid < NB + jj) {
          const int r = tid - NB;
          s_part[NB + r] = s_red[1 + n_after + r] - alpha * P[r * ldp + jj];
        }
        __syncthreads();
        for (int i = jj + tid; i < h; i += kThreads) {
          const double vi = pj[i];
          for (int q = 0; q < n_after; ++q) P[(jj + 1 + q) * ldp + i] -= beta * s_part[q] * vi;
        }
        // T(0:jj, jj) = -beta T(0:jj, 0:jj) z, T(jj, jj) = beta
        if (tid < jj) {
          double t = 0.0;
          for (int s = tid; s < jj; ++s) t += sT[tid * NB + s] * s_part[NB + s];
          s_red[tid] = -beta * t;
        }
        __syncthreads();
        if (tid < jj) sT[tid * NB + jj] = s_red[tid];
        if (tid == 0) sT[jj * NB + jj] = beta;
        __syncthreads();
      }
      for (int q = 0; q < nbk; ++q) {
        double* dst = A + (uint64_t)(k0 + q) * lda;
        for (int i = tid; i < h; i += kThreads) dst[R(i)] = P[q * ldp + i];
      }
      for (int t = tid; t < NB * NB; t += kThreads) tglob[t] = sT[t];  // kept: apply_q_wy reads it
    }
    csync();
    if (rank != 0) {
      for (int q = 0; q < nbk; ++q) {
        const double* src = A + (uint64_t)(k0 + q) * lda;
        for (int i = tid; i < h; i += kThreads) P[q * ldp + i] = __ldcg(src + R(i));
      }
      for (int t = tid; t < NB * NB; t += kThreads) sT[t] = __ldcg(tglob + t);
      __syncthreads();
    }
    // ---- trailing update on columns >= k0 + nbk, one warp per 8-column tile ----
    const int c0 = k0 + nbk;
    const int ntiles = (n - c0 + kTileN - 1) / kTileN;
    double* wt = s_w + warp * (NB * 8);
    const int lr = lane >> 2, lc = lane & 3;  // fragment coordinates
    for (int tile = rank * kWarps + warp; tile < ntiles; tile += csize * kWarps) {
      const int j0 = c0 + tile * kTileN;
      // pass 1: W = V^T C (NB x 8), k = rows
      const int jb = j0 + lr;  // B fragment column
      const bool jb_ok = jb < n;
      const double* cb = A + (uint64_t)(jb_ok ? jb : n - 1) * lda;
      double w[(NB + 7) / 8][2];
#pragma unroll
      for (int hh = 0; hh < (NB + 7) / 8; ++hh) w[hh][0] = w[hh][1] = 0.0;
      // 8 k-steps per batch: the batch's loads are in flight together (one L2 round
      // trip per 32 rows instead of one per 4)
      for (int i0 = 0; i0 < h; i0 += 4 * kKB) {
        double bv[kKB];
#pragma unroll
        for (int u = 0; u < kKB; ++u) {
          const int i = i0 + 4 * u + lc;
          bv[u] = (jb_ok && i < h) ? __ldcg(cb + R(i)) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < kKB; ++u) {
          const int i = i0 + 4 * u + lc;
#pragma unroll
          for (int hh = 0; hh < (NB + 7) / 8; ++hh) {
            const int r = hh * 8 + lr;
            const double av = (r < nbk && i >= r && i < h) ? P[r * ldp + i] : 0.0;
            dmma(w[hh][0], w[hh][1], av, bv[u]);
          }
        }
      }
      // W -> smem (row r = hh*8 + lr, cols 2lc, 2lc+1), then W' = -(T^T W) in place
#pragma unroll
      for (int hh = 0; hh < (NB + 7) / 8; ++hh) {
        const int r = hh * 8 + lr;
        if (r < NB) {
          wt[r * 8 + 2 * lc] = w[hh][0];
          wt[r * 8 + 2 * lc + 1] = w[hh][1];
        }
      }
      __syncwarp();
      double wn[(NB * 8 + 31) / 32];
#pragma unroll
      for (int e = 0; e < (NB * 8 + 31) / 32; ++e) {
        const int idx = e * 32 + lane;
        double t = 0.0;
        if (idx < NB * 8) {
          const int r = idx >> 3, q = idx & 7;
          for (int s = 0; s <= r; ++s) t += sT[s * NB + r] * wt[s * 8 + q];
        }
        wn[e] = -t;
      }
      __syncwarp();
#pragma unroll
      for (int e = 0; e < (NB * 8 + 31) / 32; ++e) {
        const int idx = e * 32 + lane;
        if (idx < NB * 8) wt[idx] = wn[e];
      }
      __syncwarp();
      // pass 2: C(8 rows x 8 cols) += V(8 x NB) * (-W'), accumulator = C
      const int ja = j0 + 2 * lc;
      double* ca0 = A + (uint64_t)min(ja, n - 1) * lda;
      double* ca1 = A + (uint64_t)min(ja + 1, n - 1) * lda;
      double bw[(NB + 3) / 4];
#pragma unroll
      for (int kk = 0; kk < NB; kk += 4) bw[kk / 4] = (kk + lc < NB) ? wt[(kk + lc) * 8 + lr] : 0.0;
      for (int i0 = 0; i0 < h; i0 += 8 * kRBq) {
        double d0[kRBq], d1[kRBq];
        uint32_t gi[kRBq];
#pragma unroll
        for (int u = 0; u < kRBq; ++u) {
          const int i = i0 + 8 * u + lr;
          const bool row_ok = i < h;
          gi[u] = row_ok ? R(i) : 0u;
          d0[u] = (row_ok && ja < n) ? __ldcg(ca0 + gi[u]) : 0.0;
          d1[u] = (row_ok && ja + 1 < n) ? __ldcg(ca1 + gi[u]) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < kRBq; ++u) {
          const int i = i0 + 8 * u + lr;
          const bool row_ok = i < h;
#pragma unroll
          for (int kk = 0; kk < NB; kk += 4) {
            const int r = kk + lc;
            const double av = (r < nbk && row_ok && i >= r) ? P[r * ldp + i] : 0.0;
            dmma(d0[u], d1[u], av, bw[kk / 4]);
          }
          if (row_ok) {
            if (ja < n) ca0[gi[u]] = d0[u];
            if (ja + 1 < n) ca1[gi[u]] = d1[u];
          }
        }
      }
      __syncwarp();
    }
    csync();
  }
}


// out (m x ncols, ld m) = Q [x; 0] for a job factored by qr_kernel<NB> (dense, not
// stacked), through the compact-WY panels the factorisation left in tmat:
// Q = Q_1 Q_2 ... Q_P, Q_p = I - V_p T_p V_p^T, applied last panel first. One CTA per
// job, one warp per 8-column tile of out (the tile stays with its warp for all
// panels); per panel W = V^T O and O += V (-(T W)) run on the FP64 tensor cores
// exactly as the factorisation's trailing update does (svd.cpp:111-132 applies the
// same reflectors one at a time).
template <int NB>
__global__ void __launch_bounds__(kThreads, 2) apply_q_wy_kernel(const ApplyQJob* __restrict__ jobs, uint32_t ldp) {
  extern __shared__ __align__(16) double sm[];
  const ApplyQJob aj = jobs[blockIdx.x];
  const int wslot = blockIdx.y * kWarps + (threadIdx.x >> 5), wstride = gridDim.y * kWarps;  // tiles over the job's CTAs
  const QrJob& job = aj.qr;
  const int m = (int)job.m, K = (int)(job.m < job.n ? job.m : job.n), ncols = (int)aj.ncols;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int lr = lane >> 2, lc = lane & 3;
  double* P = sm;                     // NB x ldp
  double* sT = P + (size_t)NB * ldp;  // NB x NB, T(r, c) at r * NB + c
  double* wt = sT + NB * NB + warp * (NB * 8);
  double* O = aj.out;
  const int ntiles = (ncols + kTileN - 1) / kTileN;
  // O = [x; 0]
  for (int tile = wslot; tile < ntiles; tile += wstride)
    for (int cc = 0; cc < kTileN; ++cc) {
      const int c = tile * kTileN + cc;
      if (c >= ncols) break;
      for (int i = lane; i < m; i += 32)
        O[(uint64_t)c * m + i] = i < (int)aj.x_rows ? __ldcg(aj.x + (uint64_t)c * aj.x_rows + i) : 0.0;
    }
  __syncwarp();
  const int npanels = (K + NB - 1) / NB;
  for (int pi = npanels - 1; pi >= 0; --pi) {
    const int k0 = pi * NB, nbk = min(NB, K - k0), h = m - k0;
    __syncthreads();  // the previous panel is consumed
    for (int q = 0; q < nbk; ++q) {
      const double* src = job.a + (uint64_t)(k0 + q) * job.lda + k0;
      for (int i = tid; i < h; i += kThreads) P[q * ldp + i] = __ldcg(src + i);
    }
    const double* tglob = job.tmat + (uint64_t)pi * NB * NB;
    for (int t = tid; t < NB * NB; t += kThreads) sT[t] = __ldcg(tglob + t);
    __syncthreads();
    for (int tile = wslot; tile < ntiles; tile += wstride) {
      const int j0 = tile * kTileN;
      // pass 1: W = V^T O (NB x 8), k = rows k0..m-1
      const int jb = j0 + lr;
      const bool jb_ok = jb < ncols;
      const double* cb = O + (uint64_t)(jb_ok ? jb : ncols - 1) * m + k0;
      double w[(NB + 7) / 8][2];
#pragma unroll
      for (int hh = 0; hh < (NB + 7) / 8; ++hh) w[hh][0] = w[hh][1] = 0.0;
      for (int i0 = 0; i0 < h; i0 += 4 * kKB) {
        double bv[kKB];
#pragma unroll
        for (int u = 0; u < kKB; ++u) {
          const int i = i0 + 4 * u + lc;
          bv[u] = (jb_ok && i < h) ? cb[i] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < kKB; ++u) {
          const int i = i0 + 4 * u + lc;
#pragma unroll
          for (int hh = 0; hh < (NB + 7) / 8; ++hh) {
            const int r = hh * 8 + lr;
            const double av = (r < nbk && i >= r && i < h) ? P[r * ldp + i] : 0.0;
            dmma(w[hh][0], w[hh][1], av, bv[u]);
          }
        }
      }
#pragma unroll
      for (int hh = 0; hh < (NB + 7) / 8; ++hh) {
        const int r = hh * 8 + lr;
        if (r < NB) {
          wt[r * 8 + 2 * lc] = w[hh][0];
          wt[r * 8 + 2 * lc + 1] = w[hh][1];
        }
      }
      __syncwarp();
      // W' = -(T W): T upper triangular
      double wn[(NB * 8 + 31) / 32];
#pragma unroll
      for (int e = 0; e < (NB * 8 + 31) / 32; ++e) {
        const int idx = e * 32 + lane;
        double t = 0.0;
        if (idx < NB * 8) {
          const int r = idx >> 3, q = idx & 7;
          for (int s2 = r; s2 < NB; ++s2) t += sT[r * NB + s2] * wt[s2 * 8 + q];
        }
        wn[e] = -t;
      }
      __syncwarp();
#pragma unroll
      for (int e = 0; e < (NB * 8 + 31) / 32; ++e) {
        const int idx = e * 32 + lane;
        if (idx < NB * 8) wt[idx] = wn[e];
      }
      __syncwarp();
      // pass 2: O(8 rows x 8 cols) += V(8 x NB) W'
      const int ja = j0 + 2 * lc;
      double* ca0 = O + (uint64_t)min(ja, ncols - 1) * m + k0;
      double* ca1 = O + (uint64_t)min(ja + 1, ncols - 1) * m + k0;
      double bw[NB / 4];
#pragma unroll
      for (int kk = 0; kk < NB; kk += 4) bw[kk / 4] = wt[(kk + lc) * 8 + lr];
      for (int i0 = 0; i0 < h; i0 += 8 * kRBq) {
        double d0[kRBq], d1[kRBq];
#pragma unroll
        for (int u = 0; u < kRBq; ++u) {
          const int i = i0 + 8 * u + lr;
          d0[u] = (i < h && ja < ncols) ? ca0[i] : 0.0;
          d1[u] = (i < h && ja + 1 < ncols) ? ca1[i] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < kRBq; ++u) {
          const int i = i0 + 8 * u + lr;
          const bool row_ok = i < h;
#pragma unroll
          for (int kk = 0; kk < NB; kk += 4) {
            const int r = kk + lc;
            const double av = (r < nbk && row_ok && i >= r) ? P[r * ldp + i] : 0.0;
            dmma(d0[u], d1[u], av, bw[kk / 4]);
          }
          if (row_ok) {
            if (ja < ncols) ca0[i] = d0[u];
            if (ja + 1 < ncols) ca1[i] = d1[u];
          }
        }
      }
      __syncwarp();
    }
  }
}

uint32_t panel_ld(uint32_t h) {
  // >= h, == 4 mod 16: the 8 reflectors x 4 rows of an MMA A fragment hit distinct bank pairs
  uint32_t ld = (h + 15) / 16 * 16 + 4;
  return ld;
}

template <int NB>
size_t qr_smem(uint32_t h_max) {
  return ((size_t)NB * panel_ld(h_max) + NB * NB + kWarps * NB + NB + kWarps * NB * 8) * sizeof(double);
}

template <int NB>
void launch_qr(const std::vector<QrJob>& jobs, const QrJob* d_jobs, unsigned cl, uint32_t h_max, cudaStream_t s) {
  const size_t smem = qr_smem<NB>(h_max);
  uint32_t ldp = panel_ld(h_max);
  RK_CUDA_CHECK(cudaFuncSetAttribute(qr_kernel<NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  RK_CUDA_CHECK(cudaFuncSetAttribute(qr_kernel<NB>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  RK_CUDA_CHECK(cudaFuncSetAttribute(qr_kernel<NB>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
  void* args[] = {(void*)&d_jobs, (void*)&ldp};
  launch_cluster_kernel((const void*)qr_kernel<NB>, (unsigned)jobs.size() * cl, cl, kThreads, smem, s, args);
}

}  // namespace

uint32_t qr_max_rows() { return 24000; }

static int qr_nb_for(uint32_t h_max) {
  const size_t budget = 224 * 1024;
  int nb = 16;
  while (nb > 1 && (nb == 16 ? qr_smem<16>(h_max) : nb == 8 ? qr_smem<8>(h_max) : nb == 4 ? qr_smem<4>(h_max)
                                                                                          : qr_smem<2>(h_max)) > budget)
    nb /= 2;
  return nb;
}

uint32_t qr_panel_nb(uint32_t h_max) { return (uint32_t)qr_nb_for(h_max); }

bool apply_q_wy_batched(const ApplyQJob* d_jobs, size_t n_jobs, uint32_t m_max, uint32_t c_max, uint32_t nb,
                        cudaStream_t s) {
  if (nb != 16 || !n_jobs) return false;  // the panel width every m <= ~1700 factors with
  const uint32_t ldp = panel_ld(m_max);
  const size_t smem = ((size_t)16 * ldp + 16 * 16 + kWarps * 16 * 8) * sizeof(double);
  if (smem > 224 * 1024) return false;
  RK_CUDA_CHECK(cudaFuncSetAttribute(apply_q_wy_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  // a warp per 8-column tile: enough CTAs per job that no warp takes a second tile
  const unsigned gy = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(8, ceil_div(ceil_div(c_max, kTileN), kWarps)));
  apply_q_wy_kernel<16><<<dim3((unsigned)n_jobs, gy), kThreads, smem, s>>>(d_jobs, ldp);
  RK_LAUNCH_CHECK();
  return true;
}

void qr_batched(const std::vector<QrJob>& jobs, cudaStream_t s, int sms) {
  if (jobs.empty()) return;
  uint32_t h_max = 0, widest = 0;
  for (const QrJob& j : jobs) {
    // active panel rows: dense m - k0 <= m; stacked <= nb + (m - split)
    const uint32_t h = j.split ? std::min<uint32_t>(j.m, (j.m - j.split) + 16) : j.m;
    h_max = std::max(h_max, h);
    widest = std::max(widest, j.n);
  }
  if (h_max > qr_max_rows()) fail(RK_RUNTIME, "qr_batched: matrix taller than a panel can stage");
  const size_t budget = 224 * 1024;  // sm_100a opt-in limit is 227 KB
  int nb = 16;
  while (nb > 1 && (nb == 16 ? qr_smem<16>(h_max) : nb == 8 ? qr_smem<8>(h_max) : nb == 4 ? qr_smem<4>(h_max)
                                                                                          : qr_smem<2>(h_max)) > budget)
    nb /= 2;
  const size_t smem = nb == 16 ? qr_smem<16>(h_max)
                      : nb == 8 ? qr_smem<8>(h_max)
                      : nb == 4 ? qr_smem<4>(h_max)
                      : nb == 2 ? qr_smem<2>(h_max)
                                : qr_smem<1>(h_max);
  if (smem > budget) fail(RK_RUNTIME, "qr_batched: matrix taller than a panel can stage");
  // one CTA per matrix while the batch fills the GPU (other CTAs on the SM hide the
  // panel latency); clusters split the trailing update of small batches
  const unsigned per_sm = (unsigned)std::max<size_t>(1, std::min<size_t>(2, (228 * 1024) / (smem + 2048)));
  unsigned cl = (unsigned)std::max<uint64_t>(1, (uint64_t)sms * per_sm / jobs.size());
  const unsigned useful = std::max(1u, (widest / kTileN + kWarps - 1) / kWarps);
  cl = std::min({cl, 8u, useful});
  unsigned p2 = 1;
  while (p2 * 2 <= cl) p2 *= 2;
  cl = p2;
  DBuf<QrJob> dj(jobs.size(), s);
  to_device(dj.get(), jobs.data(), jobs.size(), s);
  const QrJob* d = dj.get();
  if (nb == 16) launch_qr<16>(jobs, d, cl, h_max, s);
  else if (nb == 8) launch_qr<8>(jobs, d, cl, h_max, s);
  else if (nb == 4) launch_qr<4>(jobs, d, cl, h_max, s);
  else if (nb == 2) launch_qr<2>(jobs, d, cl, h_max, s);
  else launch_qr<1>(jobs, d, cl, h_max, s);
}

}  // namespace rk
