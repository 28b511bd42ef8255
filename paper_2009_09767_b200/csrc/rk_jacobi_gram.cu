// rk_jacobi_gram.cu -- Gram-assisted blocked one-sided Jacobi for
// well-conditioned matrices (the Gram/Cholesky-route blocks and merge, whose
// kappa is bounded by kappa_max(M); see rk_gram.cu).
//
// Same sweep/tournament structure, thresholds and convergence rule as the
// direct kernel (rk_dense.cu, after proj/src/svd.cpp:214-306), but for each
// staged group pair X = [W_A W_B] (M x 2g):
//   1. H = X^T X on the FP64 tensor cores (mma.sync m8n8k4 f64 -> DMMA): fresh
//      dot products and column norms for every pair of the step;
//   2. the step's rounds (intra-group rounds in step 0, then g cross rounds) run
//      on H instead of on the M-long columns: a rotation of columns (p, q) is the
//      two-sided update H <- J^T H J (rows, then columns, of a 2g x 2g matrix),
//      accumulated into Z = J_1 J_2 ...;
//   3. X <- X Z on the tensor cores (one GEMM per step instead of g rounds of
//      M-long axpys), written back.
// The first decision of every pair in a step uses a fresh dot; later decisions
// in the same step read H as updated by the step's rotations (the reference
// likewise tests updated alpha values). A sweep with no rotation is therefore
// an exact convergence check. Restricted to matrices whose kappa keeps the
// two-sided updates' rounding far below the 1e-14 rotation threshold.
#include <cooperative_groups.h>

#include <algorithm>

#include "rk_internal.cuh"

namespace cg = cooperative_groups;

namespace rk {

namespace {

constexpr double kJacobiTol = 1e-14;
constexpr int kMaxSweeps = 60;
constexpr int kT = 256;
constexpr int kW = kT / 32;

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ double wsum(double x) {
#pragma unroll
  for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

__device__ __forceinline__ uint32_t rr_slot(uint32_t pos, uint32_t step, uint32_t n) {
  return pos == 0 ? 0 : 1 + (pos - 1 + step) % (n - 1);
}

// FP32-steered, exactly renormalized rotation (same as rk_dense.cu)
__device__ __forceinline__ void rot_cs(double ap, double aq, double gamma, double& c, double& s) {
  const double d = aq - ap, e = 2.0 * gamma;
  const double m = fmax(fabs(d), fabs(e));
  const int ex = ((__double2hiint(m) >> 20) & 0x7ff) - 1023;
  const double f = __hiloint2double((1023 - ex) << 20, 0);
  const float df = (float)(d * f), ef = (float)(e * f);
  const float r = sqrtf(fmaf(df, df, ef * ef));
  const float sgn = (df == 0.0f || ((df > 0.0f) == (ef > 0.0f))) ? 1.0f : -1.0f;
  const float t = sgn * fabsf(ef) / (fabsf(df) + r);
  const float c32 = rsqrtf(fmaf(t, t, 1.0f));
  double cc = (double)c32, ss = (double)(c32 * t);
  const double n = cc * cc + ss * ss;
  double r1 = 1.5 - 0.5 * n;
  r1 = r1 * (1.5 - 0.5 * n * r1 * r1);
  c = cc * r1;
  s = ss * r1;
}

struct GramParams {
  const JacobiJob* jobs;
  uint32_t g, G;
};

// One round on H: lane group `grp` (Q lanes) owns pair (p, q).
template <int Q>
__device__ __forceinline__ void h_round(double* H, double* Z, uint32_t ldH, uint32_t n2, bool has_pair, uint32_t p,
                                        uint32_t q, double freeze, double& max_r2, unsigned long long& my_rot) {
  const int lq = threadIdx.x & (Q - 1);
  double c = 1.0, s = 0.0;
  bool rot = false;
  if (has_pair) {
    const double ap = H[p + p * ldH], aq = H[q + q * ldH], gm = H[p + q * ldH];
    const bool live = !(ap <= freeze || aq <= freeze);
    const double prod = ap * aq, g2 = gm * gm;
    if (live && g2 > max_r2 * prod) max_r2 = g2 / prod;
    rot = live && (g2 > kJacobiTol * kJacobiTol * prod);
    if (rot) {
      rot_cs(ap, aq, gm, c, s);
      // rows p, q: H(p, j), H(q, j)
      for (uint32_t j = lq; j < n2; j += Q) {
        const double hp = H[p + j * ldH], hq = H[q + j * ldH];
        H[p + j * ldH] = c * hp - s * hq;
        H[q + j * ldH] = s * hp + c * hq;
      }
      if (lq == 0) ++my_rot;
    }
  }
  __syncthreads();
  if (rot) {
    // columns p, q of H and Z
    double* hp = H + p * ldH;
    double* hq = H + q * ldH;
    double* zp = Z + p * ldH;
    double* zq = Z + q * ldH;
    for (uint32_t i = lq; i < n2; i += Q) {
      const double a = hp[i], b = hq[i];
      hp[i] = c * a - s * b;
      hq[i] = s * a + c * b;
      const double za = zp[i], zb = zq[i];
      zp[i] = c * za - s * zb;
      zq[i] = s * za + c * zb;
    }
  }
  __syncthreads();
}

template <int Q>
__global__ void __launch_bounds__(kT, 2) jacobi_gram_kernel(GramParams P) {
  extern __shared__ __align__(16) double smem[];
  cg::cluster_group cluster = cg::this_cluster();
  const unsigned rank = cluster.block_rank(), csize = cluster.num_blocks();
  const JacobiJob job = P.jobs[blockIdx.x / csize];
  const uint32_t rows = job.rows, cols_pad = job.cols_pad;
  const uint32_t g = P.g, G = P.G, n2 = 2 * g;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int lr = lane >> 2, lc = lane & 3;
  const uint32_t ldS = (rows + 3) / 4 * 4 + 4;   // == 4 mod 8 doubles: conflict-free MMA fragments
  const uint32_t ldH = n2 + 4;
  const uint32_t rows4 = (rows + 3) / 4 * 4;

  double* X = smem;                      // n2 columns, stride ldS (rows..rows4 zero)
  double* H = X + (uint64_t)n2 * ldS;    // n2 x n2, column-major, ld ldH
  double* Z = H + (uint64_t)n2 * ldH;    // n2 x n2
  __shared__ double s_red[kW];
  __shared__ double s_amax;
  __shared__ unsigned long long s_rot;

  unsigned long long* counters = reinterpret_cast<unsigned long long*>(job.stats + 4);
  double* W = job.w;
  double* alpha_g = job.alpha;
  constexpr int kGroups = kT / Q;
  const int grp = tid / Q;

  unsigned long long total_rot = 0;
  double last_max_ratio = 0.0;
  int converged = (job.cols < 2);
  int sweep = 0;
  for (; sweep < kMaxSweeps && !converged; ++sweep) {
    for (uint32_t j = rank * kW + warp; j < cols_pad; j += csize * kW) {
      const double* wj = W + (uint64_t)j * rows;
      double a = 0.0;
      for (uint32_t i = lane; i < rows; i += 32) {
        const double x = __ldcg(wj + i);
        a += x * x;
      }
      a = wsum(a);
      if (lane == 0) alpha_g[j] = a;
    }
    if (rank == 0 && tid == 0) counters[(sweep + 1) % 3] = 0ull;
    cluster.sync();
    double amax = 0.0;
    for (uint32_t j = tid; j < cols_pad; j += kT) amax = fmax(amax, __ldcg(alpha_g + j));
    for (int o = 16; o; o >>= 1) amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    if (lane == 0) s_red[warp] = amax;
    if (tid == 0) s_rot = 0ull;
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
      for (int w = 0; w < kW; ++w) t = fmax(t, s_red[w]);
      s_amax = t;
    }
    __syncthreads();
    const double freeze = kJacobiTol * kJacobiTol * s_amax;
    unsigned long long my_rot = 0;
    double my_ratio = 0.0;

    for (uint32_t step = 0; step + 1 < G; ++step) {
      for (uint32_t pi = rank; pi < G / 2; pi += csize) {
        const uint32_t gA = rr_slot(pi, step, G), gB = rr_slot(G - 1 - pi, step, G);
        // ---- stage X ----
        for (uint32_t c = warp; c < n2; c += kW) {
          const uint32_t col = (c < g ? gA * g + c : gB * g + (c - g));
          const double* src = W + (uint64_t)col * rows;
          double* dst = X + (uint64_t)c * ldS;
          for (uint32_t i = lane; i < rows4; i += 32) dst[i] = i < rows ? __ldcg(src + i) : 0.0;
        }
        for (uint32_t t = tid; t < n2 * n2; t += kT) {
          const uint32_t i = t % n2, j = t / n2;
          Z[i + j * ldH] = (i == j) ? 1.0 : 0.0;
        }
        __syncthreads();
        // ---- H = X^T X (lower 8x8 tiles, DMMA), mirrored ----
        const uint32_t nt = n2 / 8;
        for (uint32_t tt = warp; tt < nt * (nt + 1) / 2; tt += kW) {
          uint32_t ti = 0;
          while ((ti + 1) * (ti + 2) / 2 <= tt) ++ti;
          const uint32_t tj = tt - ti * (ti + 1) / 2;
          const double* xa = X + (uint64_t)(ti * 8 + lr) * ldS + lc;
          const double* xb = X + (uint64_t)(tj * 8 + lr) * ldS + lc;
          double d0 = 0.0, d1 = 0.0;
#pragma unroll 8
          for (uint32_t k0 = 0; k0 < rows4; k0 += 4) dmma(d0, d1, xa[k0], xb[k0]);
          const uint32_t i = ti * 8 + lr, j0 = tj * 8 + 2 * lc;
          H[i + j0 * ldH] = d0;
          H[i + (j0 + 1) * ldH] = d1;
          H[j0 + i * ldH] = d0;
          H[(j0 + 1) + i * ldH] = d1;
        }
        __syncthreads();
        // ---- the step's rounds on H ----
        if (step == 0) {
          for (uint32_t r = 0; r + 1 < g; ++r) {
            const bool has = (uint32_t)grp < g;
            uint32_t p = 0, q = 0;
            if (has) {
              const uint32_t half = g / 2, gi = grp / half, i = grp % half;
              p = gi * g + rr_slot(i, r, g);
              q = gi * g + rr_slot(g - 1 - i, r, g);
            }
            h_round<Q>(H, Z, ldH, n2, has, p, q, freeze, my_ratio, my_rot);
          }
        }
        for (uint32_t r = 0; r < g; ++r) {
          const bool has = (uint32_t)grp < g;
          const uint32_t p = has ? grp : 0, q = has ? g + (grp + r) % g : 0;
          h_round<Q>(H, Z, ldH, n2, has, p, q, freeze, my_ratio, my_rot);
        }
        // ---- X <- X Z (DMMA), row blocks of 8 owned by one warp ----
        for (uint32_t rb = warp; rb * 8 < rows4; rb += kW) {
          const uint32_t r0 = rb * 8;
          double av[16];  // n2 / 4 <= 16 (g <= 32)
#pragma unroll
          for (int kk = 0; kk < 16; ++kk)
            av[kk] = ((uint32_t)kk * 4 < n2 && r0 + lr < rows4) ? X[(uint64_t)(kk * 4 + lc) * ldS + r0 + lr] : 0.0;
          __syncwarp();
          for (uint32_t ntile = 0; ntile < nt; ++ntile) {
            double d0 = 0.0, d1 = 0.0;
#pragma unroll
            for (int kk = 0; kk < 16; ++kk)
              if ((uint32_t)kk * 4 < n2) dmma(d0, d1, av[kk], Z[(kk * 4 + lc) + (ntile * 8 + lr) * ldH]);
            const uint32_t i = r0 + lr, j0 = ntile * 8 + 2 * lc;
            if (i < rows4) {
              X[(uint64_t)j0 * ldS + i] = d0;
              X[(uint64_t)(j0 + 1) * ldS + i] = d1;
            }
          }
        }
        __syncthreads();
        // ---- write back ----
        for (uint32_t c = warp; c < n2; c += kW) {
          const uint32_t col = (c < g ? gA * g + c : gB * g + (c - g));
          double* dst = W + (uint64_t)col * rows;
          const double* src = X + (uint64_t)c * ldS;
          for (uint32_t i = lane; i < rows; i += 32) dst[i] = src[i];
        }
        __syncthreads();
      }
      if (step + 2 == G) {
        if (my_rot) atomicAdd(&s_rot, my_rot);
        for (int o = 16; o; o >>= 1) my_ratio = fmax(my_ratio, __shfl_xor_sync(0xffffffffu, my_ratio, o));
        if (lane == 0) s_red[warp] = my_ratio;
        __syncthreads();
        if (tid == 0) {
          double t = 0.0;
          for (int w = 0; w < kW; ++w) t = fmax(t, s_red[w]);
          if (s_rot) atomicAdd(&counters[sweep % 3], s_rot);
          atomicMax(reinterpret_cast<unsigned long long*>(job.stats + 3), __double_as_longlong(sqrt(t)));
        }
      }
      cluster.sync();
    }
    const unsigned long long rot = __ldcg(&counters[sweep % 3]);
    total_rot += rot;
    last_max_ratio = __longlong_as_double(__ldcg(reinterpret_cast<long long*>(job.stats + 3)));
    cluster.sync();
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

}  // namespace

size_t jacobi_gram_smem(uint32_t rows, uint32_t g) {
  const uint32_t n2 = 2 * g;
  const uint32_t ldS = (rows + 3) / 4 * 4 + 4, ldH = n2 + 4;
  return ((size_t)n2 * ldS + 2 * (size_t)n2 * ldH) * sizeof(double);
}

bool jacobi_gram_supported(uint32_t rows, uint32_t g, size_t smem_optin) {
  return g % 4 == 0 && g <= 32 && jacobi_gram_smem(rows, g) <= std::min<size_t>(smem_optin, 200 * 1024);
}

void jacobi_gram_batched(std::vector<JacobiJob>& jobs, uint32_t g, uint32_t G, cudaStream_t s, int sms) {
  const size_t smem = jacobi_gram_smem(jobs[0].rows, g);
  const unsigned per_sm = (unsigned)std::max<size_t>(1, std::min<size_t>(2, (228 * 1024) / (smem + 2048)));
  unsigned cl = (unsigned)std::max<uint64_t>(1, (uint64_t)sms * per_sm / jobs.size());
  cl = std::min<unsigned>({cl, G / 2, 8u});
  unsigned p2 = 1;
  while (p2 * 2 <= cl) p2 *= 2;
  cl = p2;
  DBuf<JacobiJob> dj(jobs.size(), s);
  to_device(dj.get(), jobs.data(), jobs.size(), s);
  GramParams P{dj.get(), g, G};
  void* kargs[] = {&P};
  int Q = 32;
  while (Q > 8 && (kT / Q) < (int)g) Q /= 2;
  auto launch = [&](auto kern) {
    RK_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    RK_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    RK_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    launch_cluster_kernel((const void*)kern, (unsigned)jobs.size() * cl, cl, kT, smem, s, kargs);
  };
  if (Q == 8) launch(jacobi_gram_kernel<8>);
  else if (Q == 16) launch(jacobi_gram_kernel<16>);
  else launch(jacobi_gram_kernel<32>);
}

}  // namespace rk
