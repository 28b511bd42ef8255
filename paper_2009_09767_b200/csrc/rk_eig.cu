// rk_eig.cu -- the merge's Gram route by a symmetric eigensolver.
//
// On the Gram route the merge holds G = P P^T (M x M, SPD) and, after the kappa
// guard, needs sigma and U of P: the eigen-decomposition G = U diag(sigma^2) U^T.
// Round 1 took the Cholesky factor and ran the one-sided Jacobi on it: one M x M
// matrix, a dependent chain of M-1 rounds per sweep on at most 16 SMs (c3, M=512:
// 12 sweeps, 13 ms). Here:
//   1. Householder tridiagonalisation G = Q T Q^T in ONE thread-block cluster of 16
//      CTAs with G resident in the cluster's shared memory (column-cyclic: CTA r
//      owns columns j = r (mod 16)); per step the owner forms the reflector, every
//      CTA reads it over DSMEM, computes its share of p = G v, the shares are summed
//      over DSMEM, and each CTA applies the rank-2 update to its own columns: two
//      cluster barriers per step, no global-memory round trip (LAPACK dsytd2's
//      algorithm, lower);
//   2. the eigenvalues of T by multisection (a warp per eigenvalue: 32 Sturm counts
//      per round narrow the interval 33x; ~11 rounds to full precision);
//   3. the eigenvectors of T by inverse iteration (a thread per eigenvalue, LU with
//      partial pivoting of the tridiagonal), then U = Q Z by the reflectors
//      (apply_q_batched).
// Accuracy: the tridiagonalisation is backward stable (|E| <= c M eps |G|) and
// bisection is accurate to eps |T|, so sigma_i moves by ~ c M eps kappa_i^2 / 2
// relative -- the same class as the Cholesky route it replaces, under the same
// kappa guard (kappa_max(M), rk_gram.cu). Inverse iteration without
// reorthogonalisation gives vectors to ~eps |T| / gap; the route declines (false:
// the caller runs the Cholesky + Jacobi route) when two eigenvalues are closer
// than 1e-8 |T| or adjacent vectors are not orthogonal to 1e-10.
#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>

#include "rk_pipeline.cuh"

namespace cg = cooperative_groups;

namespace rk {
namespace {

constexpr int kTC = 16;    // CTAs per cluster
constexpr int kTT = 512;   // threads per CTA
constexpr uint32_t kEigMaxM = 576;

__device__ __forceinline__ double block_reduce_sum(double x, double* red) {
#pragma unroll
  for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();  // red reused across calls
  if (lane == 0) red[warp] = x;
  __syncthreads();
  double t = 0.0;
  if (warp == 0) {
    t = lane < (kTT / 32) ? red[lane] : 0.0;
#pragma unroll
    for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (lane == 0) red[0] = t;
  }
  __syncthreads();
  return red[0];
}

// smem layout per CTA: A_loc [M x w] | vbuf [2][M + 2] | pbuf [2][M] | vloc [M] | wloc [M] | red [32]
__global__ void __cluster_dims__(kTC, 1, 1) __launch_bounds__(kTT, 1)
    tridiag_cluster_kernel(const double* __restrict__ G, uint32_t M, double* __restrict__ d, double* __restrict__ e,
                           double* __restrict__ V, double* __restrict__ tau) {
  cg::cluster_group cluster = cg::this_cluster();
  const int r = (int)cluster.block_rank();
  const uint32_t w = (M + kTC - 1) / kTC;  // local columns
  extern __shared__ __align__(16) double sm[];
  double* A = sm;                              // A[i + jl * M], global column j = jl * kTC + r
  double* vbuf = A + (uint64_t)M * w;          // 2 x (M + 2): v (index t <-> row k+1+t), [M] = tau
  double* pbuf = vbuf + 2 * (M + 2);           // 2 x M: this CTA's share of p (row index)
  double* vloc = pbuf + 2 * M;                 // v by row index (rows k+1..M-1)
  double* wloc = vloc + M;                     // w by row index
  double* red = wloc + M;
  const int tid = threadIdx.x;
  // load own columns
  for (uint32_t jl = 0; jl < w; ++jl) {
    const uint32_t j = jl * kTC + r;
    for (uint32_t i = tid; i < M; i += kTT) A[i + (uint64_t)jl * M] = j < M ? G[i + (uint64_t)j * M] : 0.0;
  }
  __syncthreads();
  cluster.sync();
  for (uint32_t k = 0; k + 1 < M; ++k) {
    const int owner = (int)(k % kTC);
    const uint32_t kl = k / kTC;
    const uint32_t n = M - k - 1;  // reflector length (rows k+1 .. M-1)
    const int buf = k & 1;
    double* vb = vbuf + buf * (M + 2);
    if (r == owner) {
      // (a) dlarfg on x = A[k+1 .. M-1, k]
      const double* x = A + (uint64_t)kl * M + k + 1;
      double s2 = 0.0;
      for (uint32_t t = 1 + tid; t < n; t += kTT) s2 = fma(x[t], x[t], s2);
      const double xnorm2 = block_reduce_sum(s2, red);
      const double alpha = x[0];
      double beta, tk, scale;
      if (xnorm2 == 0.0) {
        beta = alpha;
        tk = 0.0;
        scale = 0.0;
      } else {
        beta = -copysign(sqrt(fma(alpha, alpha, xnorm2)), alpha);
        tk = (beta - alpha) / beta;
        scale = 1.0 / (alpha - beta);
      }
      for (uint32_t t = tid; t < n; t += kTT) vb[t] = t == 0 ? 1.0 : x[t] * scale;
      if (tid == 0) {
        vb[M] = tk;
        d[k] = A[(uint64_t)kl * M + k];
        e[k] = beta;
        tau[k + 1] = tk;  // apply_q convention: reflector k lives in column k+1 (v0 on its diagonal)
      }
      for (uint32_t t = tid; t < n; t += kTT) V[(uint64_t)(k + 1) * M + k + 1 + t] = t == 0 ? 1.0 : x[t] * scale;
    }
    cluster.sync();  // (b) the reflector is published
    const double* ov = cluster.map_shared_rank(vb, owner);
    const double tk = ov[M];
    for (uint32_t t = tid; t < n; t += kTT) vloc[k + 1 + t] = ov[t];
    __syncthreads();
    // (d) this CTA's share of p = A v over its columns j > k
    double* pb = pbuf + buf * M;
    const uint32_t jl0 = (k + 1 + (kTC - 1) - r) / kTC;  // first local column with j > k
    for (uint32_t i = k + 1 + tid; i < M; i += kTT) {
      double acc = 0.0;
      for (uint32_t jl = jl0; jl < w; ++jl) {
        const uint32_t j = jl * kTC + r;
        if (j >= M) break;
        acc = fma(A[i + (uint64_t)jl * M], vloc[j], acc);
      }
      pb[i] = acc;
    }
    cluster.sync();  // (e) every share written
    // (f) p = sum of the shares (DSMEM), w = tau p - (tau^2 / 2)(p.v) v
    double pv = 0.0;
    for (uint32_t i = k + 1 + tid; i < M; i += kTT) {
      double p = 0.0;
      for (int q = 0; q < kTC; ++q) p += cluster.map_shared_rank(pb, q)[i];
      p *= tk;
      wloc[i] = p;
      pv = fma(p, vloc[i], pv);
    }
    const double K = -0.5 * tk * block_reduce_sum(pv, red);
    for (uint32_t i = k + 1 + tid; i < M; i += kTT) wloc[i] = fma(K, vloc[i], wloc[i]);
    __syncthreads();
    // (g) A -= v w^T + w v^T on this CTA's columns j > k (rows > k)
    for (uint32_t jl = jl0; jl < w; ++jl) {
      const uint32_t j = jl * kTC + r;
      if (j >= M) break;
      const double vj = vloc[j], wj = wloc[j];
      double* col = A + (uint64_t)jl * M;
      for (uint32_t i = k + 1 + tid; i < M; i += kTT) col[i] = fma(-vloc[i], wj, fma(-wloc[i], vj, col[i]));
    }
    __syncthreads();
  }
  if (r == (int)((M - 1) % kTC) && tid == 0) d[M - 1] = A[(uint64_t)((M - 1) / kTC) * M + M - 1];
  cluster.sync();  // no CTA leaves while others may still read its shared memory
}

// Sturm count: eigenvalues of T below x
__device__ __forceinline__ uint32_t sturm_count(const double* d, const double* e2, uint32_t M, double x,
                                                double pivmin) {
  uint32_t cnt = 0;
  double q = d[0] - x;
  if (fabs(q) < pivmin) q = -pivmin;
  cnt += q < 0.0;
  for (uint32_t i = 1; i < M; ++i) {
    q = d[i] - x - e2[i - 1] / q;
    if (fabs(q) < pivmin) q = -pivmin;
    cnt += q < 0.0;
  }
  return cnt;
}

// a warp per eigenvalue index j (ascending): multisection on [lo, hi] with 31 interior
// points per round until the interval is at the rounding level
__global__ void bisect_kernel(const double* __restrict__ d, const double* __restrict__ e, uint32_t M, double glo,
                              double ghi, double* __restrict__ lam) {
  extern __shared__ double e2s[];
  for (uint32_t i = threadIdx.x; i + 1 < M; i += blockDim.x) e2s[i] = e[i] * e[i];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const uint32_t j = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (j >= M) return;
  const double tnorm = fmax(fabs(glo), fabs(ghi));
  const double pivmin = 1e-300 + 4.9e-324;
  double lo = glo, hi = ghi;
  for (int round = 0; round < 40; ++round) {
    if (hi - lo <= 2.3e-16 * fmax(fabs(lo), fabs(hi)) + 1e-300 || hi - lo <= 1e-17 * tnorm) break;
    const double x = lo + (hi - lo) * (double)(lane + 1) / 33.0;
    const uint32_t c = sturm_count(d, e2s, M, x, pivmin);
    // the smallest point with count > j bounds lambda_j from above
    const unsigned above = __ballot_sync(0xffffffffu, c > j);
    const int first = above ? __ffs(above) - 1 : 32;  // lanes are ordered by x
    const double nhi = first < 32 ? __shfl_sync(0xffffffffu, x, first) : hi;
    const double nlo = first > 0 ? __shfl_sync(0xffffffffu, x, first > 0 ? first - 1 : 0) : lo;
    lo = nlo;
    hi = nhi;
  }
  if (lane == 0) lam[j] = 0.5 * (lo + hi);
}

// Inverse iteration, a thread per eigenvalue: the LU of T - lambda I with partial
// pivoting (dgttrf), then three solves with it (dgttrs), start vector all ones. The
// per-thread arrays are interleaved (element i of thread j at [i M + j]) so a warp's
// accesses coalesce, and the solves are a separate kernel so their read-only factors
// go through the non-coherent path with loads hoisted across unrolled iterations.
// The vectors land in Zt (row-major: z_j[i] at [i M + j]).
__global__ void inverse_lu_kernel(const double* __restrict__ d, const double* __restrict__ e, uint32_t M,
                                  const double* __restrict__ lam, double tnorm, double* __restrict__ work,
                                  uint8_t* __restrict__ pivw) {
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= M) return;
  const uint64_t MM = (uint64_t)M * M;
  double* __restrict__ dl = work;
  double* __restrict__ u0 = work + MM;
  double* __restrict__ u1 = work + 2 * MM;
  double* __restrict__ u2 = work + 3 * MM;
  const double x = lam[j];
  const double eps_t = 2.2e-16 * tnorm;
  double a = d[0] - x, b = M > 1 ? e[0] : 0.0;
  for (uint32_t i = 0; i + 1 < M; ++i) {
    const uint64_t at = (uint64_t)i * M + j;
    const double sub = e[i], dn = d[i + 1] - x, en = i + 2 < M ? e[i + 1] : 0.0;
    double p0, p1, p2;
    if (fabs(a) >= fabs(sub)) {
      pivw[at] = 0;
      const double m = a != 0.0 ? sub / a : 0.0;
      dl[at] = m;
      p0 = a; p1 = b; p2 = 0.0;
      a = dn - m * b;
      b = en;
    } else {
      pivw[at] = 1;
      const double m = a / sub;
      dl[at] = m;
      p0 = sub; p1 = dn; p2 = en;
      a = b - m * dn;
      b = -m * en;
    }
    u0[at] = fabs(p0) < eps_t ? copysign(eps_t, p0 == 0.0 ? 1.0 : p0) : p0;
    u1[at] = p1;
    u2[at] = p2;
  }
  const uint64_t at = (uint64_t)(M - 1) * M + j;
  u0[at] = fabs(a) < eps_t ? copysign(eps_t, a == 0.0 ? 1.0 : a) : a;
}

__global__ void inverse_solve_kernel(uint32_t M, const double* __restrict__ work, const uint8_t* __restrict__ pivw,
                                     double* __restrict__ Zt) {
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= M) return;
  const uint64_t MM = (uint64_t)M * M;
  const double* __restrict__ dl = work;
  const double* __restrict__ u0 = work + MM;
  const double* __restrict__ u1 = work + 2 * MM;
  const double* __restrict__ u2 = work + 3 * MM;
  double scale = 1.0;  // z = scale * y, y kept unnormalised between passes
  for (int it = 0; it < 3; ++it) {
    // forward: L^{-1} with the row interchanges
    // the recurrences read Zt one element ahead of (forward) or at (backward) the one they
    // write; eight elements are loaded before the eight dependent steps that use and
    // overwrite them, so the chain waits for one L2 round trip per eight steps, not per step
    constexpr uint32_t kB = 8;
    double zi = it == 0 ? 1.0 : Zt[j] * scale;
    for (uint32_t i0 = 0; i0 + 1 < M; i0 += kB) {
      double zn[kB], mm[kB];
      uint8_t pv[kB];
#pragma unroll
      for (uint32_t u = 0; u < kB; ++u) {
        const uint32_t i = i0 + u;
        if (i + 1 < M) {
          const uint64_t at = (uint64_t)i * M + j;
          zn[u] = it == 0 ? 1.0 : Zt[at + M] * scale;
          mm[u] = __ldg(dl + at);
          pv[u] = __ldg(pivw + at);
        }
      }
#pragma unroll
      for (uint32_t u = 0; u < kB; ++u) {
        const uint32_t i = i0 + u;
        if (i + 1 < M) {
          const uint64_t at = (uint64_t)i * M + j;
          if (pv[u]) {
            Zt[at] = zn[u];
            zi = fma(-mm[u], zn[u], zi);
          } else {
            Zt[at] = zi;
            zi = fma(-mm[u], zi, zn[u]);
          }
        }
      }
    }
    Zt[(uint64_t)(M - 1) * M + j] = zi;
    // backward: U z = y
    double z1 = 0.0, z2 = 0.0, nrm = 0.0;
    for (int i0 = (int)M - 1; i0 >= 0; i0 -= (int)kB) {
      double y[kB], a0[kB], a1[kB], a2[kB];
#pragma unroll
      for (int u = 0; u < (int)kB; ++u) {
        const int i = i0 - u;
        if (i >= 0) {
          const uint64_t at = (uint64_t)i * M + j;
          y[u] = Zt[at];
          a0[u] = __ldg(u0 + at);
          a1[u] = __ldg(u1 + at);
          a2[u] = __ldg(u2 + at);
        }
      }
#pragma unroll
      for (int u = 0; u < (int)kB; ++u) {
        const int i = i0 - u;
        if (i >= 0) {
          const double zz = (y[u] - a1[u] * z1 - a2[u] * z2) / a0[u];
          Zt[(uint64_t)i * M + j] = zz;
          z2 = z1;
          z1 = zz;
          nrm = fma(zz, zz, nrm);
        }
      }
    }
    scale = 1.0 / sqrt(nrm);
  }
#pragma unroll 8
  for (uint32_t i = 0; i < M; ++i) Zt[(uint64_t)i * M + j] *= scale;
}

// Z (column-major, z_j in column j) from Zt (row-major), 32 x 32 tiles
__global__ void transpose_sq_kernel(const double* __restrict__ in, uint32_t M, double* __restrict__ out) {
  __shared__ double t[32][33];
  const uint32_t x0 = blockIdx.x * 32, y0 = blockIdx.y * 32;
  for (uint32_t k = threadIdx.y; k < 32; k += blockDim.y) {
    const uint32_t r = y0 + k, c = x0 + threadIdx.x;
    if (r < M && c < M) t[k][threadIdx.x] = in[(uint64_t)r * M + c];
  }
  __syncthreads();
  for (uint32_t k = threadIdx.y; k < 32; k += blockDim.y) {
    const uint32_t r = x0 + k, c = y0 + threadIdx.x;
    if (r < M && c < M) out[(uint64_t)r * M + c] = t[threadIdx.x][k];
  }
}

// max |z_j . z_{j+1}| over adjacent eigenvalues (the closest pairs)
__global__ void adjacent_dots(const double* __restrict__ Z, uint32_t M, double* __restrict__ out) {
  __shared__ double red[32];
  const uint32_t j = blockIdx.x;
  if (j + 1 >= M) return;
  double s = 0.0;
  for (uint32_t i = threadIdx.x; i < M; i += blockDim.x) s = fma(Z[(uint64_t)j * M + i], Z[(uint64_t)(j + 1) * M + i], s);
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (uint32_t w2 = 0; w2 < blockDim.x / 32; ++w2) t += red[w2];
    out[j] = fabs(t);
  }
}

// U (M x M row-major, descending sigma) from the back-transformed eigenvectors
// (ascending, column-major), with the sign convention (first index of the largest |u|)
__global__ void eig_finalize(const double* __restrict__ U_asc, const double* __restrict__ lam, uint32_t M,
                             double* __restrict__ u, double* __restrict__ sigma) {
  const uint32_t c = blockIdx.x;  // output column (descending)
  const uint32_t src = M - 1 - c;
  const double* col = U_asc + (uint64_t)src * M;
  __shared__ double s_best[32];
  __shared__ uint32_t s_arg[32];
  double best = -1.0;
  uint32_t arg = 0;
  for (uint32_t i = threadIdx.x; i < M; i += blockDim.x) {
    const double a = fabs(col[i]);
    if (a > best) { best = a; arg = i; }
  }
  for (int o = 16; o; o >>= 1) {
    const double ob = __shfl_xor_sync(0xffffffffu, best, o);
    const uint32_t oa = __shfl_xor_sync(0xffffffffu, arg, o);
    if (ob > best || (ob == best && oa < arg)) { best = ob; arg = oa; }
  }
  if ((threadIdx.x & 31) == 0) { s_best[threadIdx.x >> 5] = best; s_arg[threadIdx.x >> 5] = arg; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (uint32_t w2 = 1; w2 < blockDim.x / 32; ++w2)
      if (s_best[w2] > s_best[0] || (s_best[w2] == s_best[0] && s_arg[w2] < s_arg[0])) {
        s_best[0] = s_best[w2];
        s_arg[0] = s_arg[w2];
      }
    sigma[c] = sqrt(fmax(lam[src], 0.0));
  }
  __syncthreads();
  const double sgn = col[s_arg[0]] < 0.0 ? -1.0 : 1.0;
  for (uint32_t i = threadIdx.x; i < M; i += blockDim.x) u[(uint64_t)i * M + c] = sgn * col[i];
}

}  // namespace

// measured: at M = 512 (c3) 7.0 ms against the Jacobi's 13 ms; at M = 256 (c2) the
// Jacobi's 1.7 ms wins (255 tridiagonalisation steps of ~6 us each)
constexpr uint32_t kEigMinM = 384;
bool eig_merge_eligible(uint32_t M) { return tuning().eig_merge && M >= kEigMinM && M <= kEigMaxM; }

bool gram_merge_eig(Ctx& c, const double* G, uint32_t M, MergeOut& out) {
  if (!eig_merge_eligible(M)) return false;
  RK_NVTX("rk.merge.eig");
  cudaStream_t s = c.stream;
  const uint32_t w = (M + kTC - 1) / kTC;
  const size_t smem = ((size_t)M * w + 2 * (M + 2) + 2 * (size_t)M + 2 * (size_t)M + 32) * sizeof(double);
  if (smem > c.smem_optin) return false;
  DBuf<double> d(M, s), e(M, s), tau(M + 1, s), V((uint64_t)M * M, s);
  V.zero();
  tau.zero();
  RK_CUDA_CHECK(cudaFuncSetAttribute(tridiag_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  RK_CUDA_CHECK(cudaFuncSetAttribute(tridiag_cluster_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(kTC, 1, 1);
    cfg.blockDim = dim3(kTT, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    double* dp = d.get();
    double* ep = e.get();
    double* vp = V.get();
    double* tp = tau.get();
    void* args[] = {(void*)&G, (void*)&M, (void*)&dp, (void*)&ep, (void*)&vp, (void*)&tp};
    RK_CUDA_CHECK(cudaLaunchKernelExC(&cfg, (const void*)tridiag_cluster_kernel, args));
    RK_LAUNCH_CHECK();
  }
  prof_mark(s, "mrg eig: tridiag");
  // Gershgorin bounds of T (host: 2 M doubles)
  std::vector<double> hd, he;
  to_host(hd, d.get(), M, s);
  to_host(he, e.get(), M, s);
  sync(s);
  double glo = INFINITY, ghi = -INFINITY;
  for (uint32_t i = 0; i < M; ++i) {
    const double r = (i ? fabs(he[i - 1]) : 0.0) + (i + 1 < M ? fabs(he[i]) : 0.0);
    glo = std::min(glo, hd[i] - r);
    ghi = std::max(ghi, hd[i] + r);
  }
  const double tnorm = std::max(fabs(glo), fabs(ghi));
  glo -= 4e-16 * tnorm * M;
  ghi += 4e-16 * tnorm * M;
  DBuf<double> lam(M, s);
  bisect_kernel<<<(unsigned)ceil_div(M, 8), 256, (size_t)M * sizeof(double), s>>>(d.get(), e.get(), M, glo, ghi,
                                                                                  lam.get());
  RK_LAUNCH_CHECK();
  std::vector<double> hl;
  to_host(hl, lam.get(), M, s);
  sync(s);
  prof_mark(s, "mrg eig: bisection");
  // kappa guard (lambda = sigma^2) and the separation the inverse iteration needs
  const double lmax = hl[M - 1], lmin = hl[0];
  if (!(lmin > 0.0) || std::sqrt(lmax / lmin) > kappa_max(M)) return false;
  for (uint32_t i = 0; i + 1 < M; ++i)
    if (hl[i + 1] - hl[i] <= 1e-8 * tnorm) return false;
  DBuf<double> Z((uint64_t)M * M, s), Zt((uint64_t)M * M, s), work((uint64_t)M * 4 * M, s);
  DBuf<uint8_t> pivw((uint64_t)M * M, s);
  inverse_lu_kernel<<<(unsigned)ceil_div(M, 32), 32, 0, s>>>(d.get(), e.get(), M, lam.get(), tnorm, work.get(),
                                                             pivw.get());
  RK_LAUNCH_CHECK();
  inverse_solve_kernel<<<(unsigned)ceil_div(M, 32), 32, 0, s>>>(M, work.get(), pivw.get(), Zt.get());
  RK_LAUNCH_CHECK();
  transpose_sq_kernel<<<dim3((unsigned)ceil_div(M, 32), (unsigned)ceil_div(M, 32)), dim3(32, 8), 0, s>>>(
      Zt.get(), M, Z.get());
  RK_LAUNCH_CHECK();
  work.release();
  Zt.release();
  {
    DBuf<double> dots(M, s);
    dots.zero();
    adjacent_dots<<<M, 256, 0, s>>>(Z.get(), M, dots.get());
    RK_LAUNCH_CHECK();
    std::vector<double> hdots;
    to_host(hdots, dots.get(), M, s);
    sync(s);
    for (uint32_t i = 0; i + 1 < M; ++i)
      if (!(hdots[i] <= 1e-10)) return false;
  }
  // U = Q Z: the reflectors of the tridiagonalisation (reflector k in column k+1)
  DBuf<double> Uc((uint64_t)M * M, s);
  QrJob q;
  q.a = V.get(); q.lda = M; q.m = M; q.n = M; q.diag = nullptr; q.beta = tau.get(); q.tmat = nullptr;
  apply_q_batched({ApplyQJob{q, Z.get(), M, M, Uc.get()}}, s);
  out.k = M;
  out.sigma.alloc(M, s);
  out.u.alloc((uint64_t)M * M, s);
  eig_finalize<<<M, 256, 0, s>>>(Uc.get(), lam.get(), M, out.u.get(), out.sigma.get());
  RK_LAUNCH_CHECK();
  out.sweeps = 0;
  out.rotations = 0;
  const double Md = M;
  out.flops = 4.0 / 3.0 * Md * Md * Md + 2.0 * Md * Md * Md;  // tridiagonalisation + back-transformation
  prof_mark(s, "mrg eig: vectors");
  return true;
}

}  // namespace rk
