// rk_dense.cu -- batched dense FP64 factorizations on sm_100a.
//
//  (the blocked Householder QR lives in rk_qr.cu)
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
#include <cstdlib>

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
  double check_ratio;  // Gram convergence check after a sweep whose max ratio is below this (0: off)
  int check_first;     // start with the tail check (W comes from jacobi_warp_kernel)
  int debug;           // RK_JACOBI_DEBUG=1: print the hand-over of job 0
};

__device__ __forceinline__ uint32_t rr_slot(uint32_t pos, uint32_t step, uint32_t n) {
  // round-robin tournament: position 0 fixed, the rest rotate
  return pos == 0 ? 0 : 1 + (pos - 1 + step) % (n - 1);
}

// Rotation (c, s) for a pair with norms^2 ap, aq and inner product gamma, the
// reference's angle (svd.cpp:238-242: tan(theta) = t = sign(zeta) / (|zeta| +
// sqrt(1 + zeta^2)), zeta = (aq - ap) / (2 gamma), the root with |theta| <= pi/4),
// evaluated for latency -- this is on every round's dependent chain, and on the
// B200 an FP64 op costs 23 cycles, rsqrt 78, a conversion ~26:
//   * d = aq - ap and e = 2 gamma are scaled by an exact power of two so that
//     max(|d|, |e|) is in [1, 2), then rounded to FP32;
//   * with cos(2 theta) = |d| / r, sin(2 theta) = |e| / r (r = |(d, e)|):
//     c = sqrt((1 + cos 2theta) / 2), s = sign(d e) sin(2 theta) / (2 c), two
//     MUFU rsqrts and a few FP32 multiplies (the angle only steers convergence);
//   * (c, s) is rounded to FP64 and renormalized: with delta = c^2 + s^2 - 1
//     (~1e-7, formed with FMAs), 1 / sqrt(1 + delta) = 1 - delta/2 + 3 delta^2/8
//     + O(delta^3), so the applied rotation is orthogonal to FP64 rounding.
// The rotation decision itself uses the FP64 gamma, so the stopping rule is the
// reference's. (The previous form -- t in FP32, then two Newton steps for
// 1/sqrt(c^2 + s^2) in FP64 -- had a ~480-cycle chain; this one ~300.)
__device__ __forceinline__ void rotation_cs(double ap, double aq, double gamma, double& c, double& s) {
  const double d = aq - ap, e = 2.0 * gamma;
  const double m = fmax(fabs(d), fabs(e));
  // 2^-floor(log2 m) built from the exponent bits (exact scaling, m > 0 here)
  const int ex = ((__double2hiint(m) >> 20) & 0x7ff) - 1023;
  const double f = __hiloint2double((1023 - ex) << 20, 0);
  const float df = (float)(d * f), ef = (float)(e * f);
  const float rr = rsqrtf(fmaf(df, df, ef * ef));    // 1 / r
  const float x = fmaf(0.5f * fabsf(df), rr, 0.5f);  // (1 + cos 2theta) / 2, in [1/2, 1]
  const float rx = rsqrtf(x);                        // 1 / c
  const float sgn = (df == 0.0f || ((df > 0.0f) == (ef > 0.0f))) ? 1.0f : -1.0f;
  const double cc = (double)(x * rx), ss = (double)(sgn * 0.5f * fabsf(ef) * rr * rx);
  const double dl = fma(cc, cc, fma(ss, ss, -1.0));
  const double r = fma(dl, fma(dl, 0.375, -0.5), 1.0);
  c = cc * r;
  s = ss * r;
}

// Rotate one pair (p, q) of staged columns with a group of Q lanes (Q | 32);
// returns 1 when rotated. Same decision rule as the reference (svd.cpp:232-260):
// frozen columns are skipped before the dot; the pair rotates when
// |gamma| > tol * sqrt(alpha_p alpha_q) (tested squared); t, c, s follow
// zeta = (alpha_q - alpha_p) / (2 gamma), written without the division by gamma:
// t = sign(zeta) |2 gamma| / (|d| + sqrt(d^2 + 4 gamma^2)), c = rsqrt(1 + t^2).
// Each group starts its sweep over the rows at a different offset so the
// lane groups of a warp hit different shared-memory banks.
template <int Q>
__device__ __forceinline__ int rotate_pair_q(double* __restrict__ wp, double* __restrict__ wq, double* vp,
                                             double* vq, uint32_t rows, uint32_t vrows, double* alpha, int p,
                                             int q, double freeze, double& max_r2, uint32_t stagger) {
  const int lq = threadIdx.x & (Q - 1);
  // the Q lanes of one pair synchronize among themselves only: other groups of
  // the warp may take different branches or have no pair this round
  const unsigned gmask = (Q == 32) ? 0xffffffffu : (((1u << Q) - 1u) << ((threadIdx.x & 31) & ~(Q - 1)));
  const double ap = alpha[p], aq = alpha[q];
  if (ap <= freeze || aq <= freeze) return 0;
  const uint32_t off = stagger % rows;
  double g0 = 0.0, g1 = 0.0;
  uint32_t i = lq + off;
  uint32_t k = lq;
  for (; k + Q < rows; k += 2 * Q) {
    uint32_t i0 = i >= rows ? i - rows : i;
    uint32_t i1 = i0 + Q >= rows ? i0 + Q - rows : i0 + Q;
    g0 += wp[i0] * wq[i0];
    g1 += wp[i1] * wq[i1];
    i += 2 * Q;
    if (i >= 2 * rows) i -= rows;
  }
  if (k < rows) {
    uint32_t i0 = i >= rows ? i - rows : i;
    g0 += wp[i0] * wq[i0];
  }
  double gamma = g0 + g1;
#pragma unroll
  for (int o = Q / 2; o; o >>= 1) gamma += __shfl_xor_sync(gmask, gamma, o);
  const double prod = ap * aq, g2 = gamma * gamma;
  if (g2 > max_r2 * prod) max_r2 = g2 / prod;
  if (!(g2 > kJacobiTol * kJacobiTol * prod)) return 0;
  double c, s;
  rotation_cs(ap, aq, gamma, c, s);
  i = lq + off;
  for (k = lq; k < rows; k += Q) {
    const uint32_t ii = i >= rows ? i - rows : i;
    const double xp = wp[ii], xq = wq[ii];
    wp[ii] = c * xp - s * xq;
    wq[ii] = s * xp + c * xq;
    i += Q;
  }
  if (vp) {
    for (uint32_t j = lq; j < vrows; j += Q) {
      const double xp = vp[j], xq = vq[j];
      vp[j] = c * xp - s * xq;
      vq[j] = s * xp + c * xq;
    }
  }
  __syncwarp(gmask);
  if (lq == 0) {
    const double na = c * c * ap - 2.0 * c * s * gamma + s * s * aq;
    const double nq = s * s * ap + 2.0 * c * s * gamma + c * c * aq;
    alpha[p] = na > 0.0 ? na : 0.0;
    alpha[q] = nq > 0.0 ? nq : 0.0;
  }
  __syncwarp(gmask);
  return 1;
}

// Cross round r pairs A_t with B_{(t+r) mod g}. Group t keeps A_t (and its alpha)
// in registers for all g rounds of the step and streams the B columns through
// shared memory: per element-pair one 8-byte shared load and one store (the
// B value), instead of re-reading and re-writing both columns. Control flow is
// warp-uniform (the two or four lane groups of a warp may disagree on whether
// their pair is frozen or rotates; that is handled with predication), so the
// group reductions use full-warp shuffles that stay inside the group (xor < Q).
// GT > 0: the group size g is the compile-time constant GT (with EXACT rows the
// whole round loop unrolls: the B column of round r is a constant offset from the
// group's own, wrapped with a mask)
template <int Q, int E, bool EXACT, int GT = 0>
__device__ __forceinline__ void cross_rounds_reg(double* sW, uint32_t ldS_rt, uint32_t rows_rt, uint32_t g_rt,
                                                 double* sAlpha, double freeze, double& max_r2,
                                                 unsigned long long& my_rot) {
  const uint32_t rows = EXACT ? (uint32_t)(Q * E) : rows_rt;
  const uint32_t g = GT > 0 ? (uint32_t)GT : g_rt;
  const uint32_t ldS = (EXACT && GT > 0) ? (uint32_t)(Q * E + 8) : ldS_rt;
  const int tid = threadIdx.x;
  const int grp = tid / Q, lq = tid & (Q - 1);
  const bool active = (uint32_t)grp < g;
  double a[E];
  double aA = 0.0;
  {
    const double* pa = sW + (uint64_t)(active ? grp : 0) * ldS + lq;
#pragma unroll
    for (int k = 0; k < E; ++k) a[k] = (active && (EXACT || lq + Q * k < (int)rows)) ? pa[Q * k] : 0.0;
    aA = active ? sAlpha[grp] : 0.0;
  }
  uint32_t jl = active ? (uint32_t)grp : 0u;  // (grp + r) mod g, advanced incrementally
  double* const bbase = sW + (uint64_t)g * ldS + lq;
  constexpr bool kWide = (Q == 32 && GT == 8);  // the latency plan's instantiation (1 CTA / SM)
  double best_g2 = 0.0, best_prod = 1.0;
#pragma unroll(GT > 0 ? 4 : 1)
  for (uint32_t r = 0; r < g; ++r) {
    if (GT > 0 && (GT & (GT - 1)) == 0) jl = (uint32_t)(grp + r) & (uint32_t)(GT - 1);
    double* pb = bbase + (uint64_t)jl * ldS;
    const double aB = sAlpha[g + jl];
    const bool live = active && !(aA <= freeze || aB <= freeze);
    double b[E];
    double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0, acc3 = 0.0;
#pragma unroll
    for (int k = 0; k < E; ++k) {
      b[k] = (EXACT || lq + Q * k < (int)rows) ? pb[Q * k] : 0.0;  // frozen pairs: gamma unused
      const double pr = a[k] * b[k];
      if ((k & 3) == 0) acc0 += pr;
      else if ((k & 3) == 1) acc1 += pr;
      else if ((k & 3) == 2) acc2 += pr;
      else acc3 += pr;
    }
    double gamma = (acc0 + acc1) + (acc2 + acc3);
#pragma unroll
    for (int o = Q / 2; o; o >>= 1) gamma += __shfl_xor_sync(0xffffffffu, gamma, o);
    const double prod = aA * aB, g2 = gamma * gamma;
    if constexpr (kWide) {
      // the largest ratio as a (g2, prod) pair compared by cross multiplication: no
      // division on the round's chain (one per call, below). Only where registers
      // allow (the one-CTA-per-SM instantiation): at the 128-register cap the two
      // extra live values spill
      if (live && g2 * best_prod > best_g2 * prod) {
        best_g2 = g2;
        best_prod = prod;
      }
    } else {
      if (live && g2 > max_r2 * prod) max_r2 = g2 / prod;
    }
    const bool rot = live && (g2 > kJacobiTol * kJacobiTol * prod);
    if (__any_sync(0xffffffffu, rot)) {
      double c = 1.0, sn = 0.0;
      if (rot) rotation_cs(aA, aB, gamma, c, sn);
#pragma unroll
      for (int k = 0; k < E; ++k) {
        const double xp = a[k], xq = b[k];
        a[k] = c * xp - sn * xq;
        if (rot && (EXACT || lq + Q * k < (int)rows)) pb[Q * k] = sn * xp + c * xq;
      }
      if (rot) {
        const double na = c * c * aA - 2.0 * c * sn * gamma + sn * sn * aB;
        const double nq = sn * sn * aA + 2.0 * c * sn * gamma + c * c * aB;
        aA = na > 0.0 ? na : 0.0;
        if (lq == 0) {
          sAlpha[g + jl] = nq > 0.0 ? nq : 0.0;
          ++my_rot;
        }
      }
    }
    if (!(GT > 0 && (GT & (GT - 1)) == 0)) jl = (jl + 1 == g) ? 0u : jl + 1;
    __syncthreads();
  }
  if (kWide && best_g2 > max_r2 * best_prod) max_r2 = best_g2 / best_prod;
  if (active) {
    double* pa = sW + (uint64_t)grp * ldS + lq;
#pragma unroll
    for (int k = 0; k < E; ++k)
      if (EXACT || lq + Q * k < (int)rows) pa[Q * k] = a[k];
    if (lq == 0) sAlpha[grp] = aA;
  }
  __syncthreads();
}

// ---- convergence tail -------------------------------------------------------
// Once the sweeps are in the quadratic regime, what is left is the rounding-noise
// floor: a handful of pairs whose |gamma| / sqrt(alpha_p alpha_q) sits at the
// 1e-14 threshold, rotated by tiny angles sweep after sweep until, by chance, none
// exceeds it (the reference stops after a sweep with no rotation, svd.cpp:265). A
// full sweep re-tests all n(n-1)/2 pairs in n-1 latency-bound rounds to rotate
// those few. The tail instead
//   1. tests every pair at once: W^T W by DMMA (one 32x32 block per warp across
//      the cluster), with fresh norms and the reference's freeze and rotation
//      rule; the violating pairs go to a list in CTA 0's shared memory (DSMEM);
//   2. no violation: the check IS the reference's rotation-free last sweep -> done;
//   3. a few violations: CTA 0 sorts them (deterministic order) and rotates
//      exactly those pairs, sequentially, with fresh dots -- a sweep in which
//      every other pair was tested and left alone -- then checks again;
//   4. many violations: back to full sweeps.
// Each check computes all the sweep's dot products, so it counts as a sweep.
#ifndef RK_VIOL_CAP
#define RK_VIOL_CAP 64
#endif
constexpr int kViolCap = RK_VIOL_CAP;
constexpr int kTailIters = 8;  // then back to full sweeps

__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

struct TailShared {
  uint32_t count;
  uint32_t list[kViolCap];  // (q << 16) | p, p < q
};

// Step 1; returns the number of violating pairs (may exceed kViolCap). All
// threads of the cluster call it; *freeze_out gets the fresh freeze level.
__device__ uint32_t tail_check(cg::cluster_group& cluster, const JacobiJob& job, unsigned rank, unsigned csize,
                               double* s_red, double* s_amax, TailShared* ts, double* worst_out) {
  const uint32_t rows = job.rows, n = job.cols_pad;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const double* W = job.w;
  double* alpha_g = job.alpha;
  for (uint32_t j = rank * kJWarps + warp; j < n; j += csize * kJWarps) {
    const double* wj = W + (uint64_t)j * rows;
    double a = 0.0;
    for (uint32_t i = lane; i < rows; i += 32) {
      const double x = __ldcg(wj + i);
      a += x * x;
    }
    a = warp_sum(a);
    if (lane == 0) alpha_g[j] = a;
  }
  if (rank == 0 && tid == 0) {
    ts->count = 0;
    job.stats[7] = 0ull;
  }
  cluster.sync();
  double amax = 0.0;
  for (uint32_t j = tid; j < n; j += kJThreads) amax = fmax(amax, __ldcg(alpha_g + j));
  for (int o = 16; o; o >>= 1) amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
  if (lane == 0) s_red[warp] = amax;
  __syncthreads();
  if (tid == 0) {
    double t = 0.0;
    for (int w = 0; w < kJWarps; ++w) t = fmax(t, s_red[w]);
    *s_amax = t;
  }
  __syncthreads();
  const double freeze = kJacobiTol * kJacobiTol * (*s_amax);
  TailShared* ts0 = cluster.map_shared_rank(ts, 0);
  // 32 x 32 blocks of the lower triangle (4 x 4 DMMA tiles per warp)
  constexpr int kTB = 4;
  const uint32_t nb = (n + 8 * kTB - 1) / (8 * kTB);
  const uint32_t T = nb * (nb + 1) / 2;
  const int lr = lane >> 2, lc = lane & 3;
  double worst = 0.0;
  for (uint32_t t = rank * kJWarps + warp; t < T; t += csize * kJWarps) {
    uint32_t bi = 0;
    while ((bi + 1) * (bi + 2) / 2 <= t) ++bi;
    const uint32_t bj = t - bi * (bi + 1) / 2;
    double acc[kTB][kTB][2];
#pragma unroll
    for (int i = 0; i < kTB; ++i)
#pragma unroll
      for (int j = 0; j < kTB; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    const double* pa[kTB];
    const double* pb[kTB];
    bool va[kTB], vb[kTB];
#pragma unroll
    for (int i = 0; i < kTB; ++i) {
      const uint32_t ca = bi * 8 * kTB + i * 8 + lr, cb = bj * 8 * kTB + i * 8 + lr;
      va[i] = ca < n;
      vb[i] = cb < n;
      pa[i] = W + (uint64_t)(va[i] ? ca : 0) * rows + lc;
      pb[i] = W + (uint64_t)(vb[i] ? cb : 0) * rows + lc;
    }
#pragma unroll 4
    for (uint32_t k0 = 0; k0 < rows; k0 += 4) {
      const bool ok = k0 + lc < rows;
      double a[kTB], b[kTB];
#pragma unroll
      for (int i = 0; i < kTB; ++i) {
        a[i] = (ok && va[i]) ? __ldcg(pa[i] + k0) : 0.0;
        b[i] = (ok && vb[i]) ? __ldcg(pb[i] + k0) : 0.0;
      }
#pragma unroll
      for (int i = 0; i < kTB; ++i)
#pragma unroll
        for (int j = 0; j < kTB; ++j) dmma884(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
#pragma unroll
    for (int i = 0; i < kTB; ++i)
#pragma unroll
      for (int j = 0; j < kTB; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const uint32_t r = bi * 8 * kTB + i * 8 + lr, c = bj * 8 * kTB + j * 8 + 2 * lc + e;
          if (r < n && c < n && r > c) {
            const double h = acc[i][j][e];
            const double ar = __ldcg(alpha_g + r), ac = __ldcg(alpha_g + c);
            if (ar > freeze && ac > freeze) {
              const double q = h * h / (ar * ac);
              worst = fmax(worst, q);
              if (h * h > kJacobiTol * kJacobiTol * (ar * ac)) {
                const uint32_t slot = atomicAdd(&ts0->count, 1u);
                if (slot < (uint32_t)kViolCap) ts0->list[slot] = (r << 16) | c;
              }
            }
          }
        }
  }
  for (int o = 16; o; o >>= 1) worst = fmax(worst, __shfl_xor_sync(0xffffffffu, worst, o));
  if (lane == 0 && worst > 0.0)
    atomicMax(reinterpret_cast<unsigned long long*>(job.stats + 7), __double_as_longlong(worst));
  cluster.sync();
  const uint32_t nv = ts0->count;
  *worst_out = sqrt(__longlong_as_double(__ldcg(reinterpret_cast<const long long*>(job.stats + 7))));
  cluster.sync();  // every CTA has read CTA 0's count before anyone moves on
  return nv;
}

// Step 3 (CTA 0, warp 0): rotate the listed pairs in sorted order, fresh dots.
__device__ uint32_t tail_rotate(const JacobiJob& job, TailShared* ts, uint32_t nv, double freeze, bool with_v) {
  const int lane = threadIdx.x & 31;
  const uint32_t rows = job.rows, vrows = job.cols_pad;
  double* W = job.w;
  double* V = job.v;
  // rank sort of the (distinct) keys: deterministic whatever the atomic order was
  uint32_t keys[(kViolCap + 31) / 32];
#pragma unroll
  for (int u = 0; u < (kViolCap + 31) / 32; ++u) {
    const uint32_t i = u * 32 + lane;
    keys[u] = i < nv ? ts->list[i] : 0u;
  }
  __syncwarp();
#pragma unroll
  for (int u = 0; u < (kViolCap + 31) / 32; ++u) {
    const uint32_t i = u * 32 + lane;
    if (i < nv) {
      uint32_t rnk = 0;
      for (uint32_t j = 0; j < nv; ++j) rnk += ts->list[j] < keys[u];
      keys[u] = rnk;  // reuse: rank of my key
    }
  }
  __syncwarp();
  uint32_t mine[(kViolCap + 31) / 32];
#pragma unroll
  for (int u = 0; u < (kViolCap + 31) / 32; ++u) {
    const uint32_t i = u * 32 + lane;
    mine[u] = i < nv ? ts->list[i] : 0u;
  }
  __syncwarp();
#pragma unroll
  for (int u = 0; u < (kViolCap + 31) / 32; ++u) {
    const uint32_t i = u * 32 + lane;
    if (i < nv) ts->list[keys[u]] = mine[u];
  }
  __syncwarp();
  uint32_t rotated = 0;
  for (uint32_t t = 0; t < nv; ++t) {
    const uint32_t key = ts->list[t];
    const uint32_t q = key >> 16, p = key & 0xffffu;  // p < q
    double* wp = W + (uint64_t)p * rows;
    double* wq = W + (uint64_t)q * rows;
    double ap = 0.0, aq = 0.0, gm = 0.0;
    for (uint32_t i = lane; i < rows; i += 32) {
      const double x = wp[i], y = wq[i];
      ap += x * x;
      aq += y * y;
      gm += x * y;
    }
    ap = warp_sum(ap);
    aq = warp_sum(aq);
    gm = warp_sum(gm);
    // the DMMA check flagged this pair; at the noise floor a sequential dot may land
    // just under the threshold -- rotate anyway (an angle of ~1e-14) so the pass
    // always makes progress
    if (ap <= freeze || aq <= freeze || gm == 0.0) continue;
    double c, sn;
    rotation_cs(ap, aq, gm, c, sn);
    for (uint32_t i = lane; i < rows; i += 32) {
      const double x = wp[i], y = wq[i];
      wp[i] = c * x - sn * y;
      wq[i] = sn * x + c * y;
    }
    if (with_v) {
      double* vp = V + (uint64_t)p * vrows;
      double* vq = V + (uint64_t)q * vrows;
      for (uint32_t i = lane; i < vrows; i += 32) {
        const double x = vp[i], y = vq[i];
        vp[i] = c * x - sn * y;
        vq[i] = sn * x + c * y;
      }
    }
    __syncwarp();
    ++rotated;
  }
  return rotated;
}

// The tail loop: each check counts as a sweep (`done` = completed sweeps).
// Returns true once a check finds no pair to rotate.
__device__ bool run_tail(cg::cluster_group& cluster, const JacobiJob& job, unsigned rank, unsigned csize,
                         double* s_red, double* s_amax, TailShared* s_tail, bool with_v, int& done,
                         unsigned long long& total_rot, double& last_max_ratio) {
  const int warp = threadIdx.x >> 5;
  for (int it = 0; it < kTailIters && done < kMaxSweeps; ++it) {
    double worst = 0.0;
    const uint32_t nv = tail_check(cluster, job, rank, csize, s_red, s_amax, s_tail, &worst);
    last_max_ratio = worst;
    ++done;
    if (nv == 0) return true;                    // the rotation-free sweep
    if (nv > (uint32_t)kViolCap) return false;   // back to full sweeps
    if (rank == 0 && warp == 0) total_rot += tail_rotate(job, s_tail, nv, kJacobiTol * kJacobiTol * (*s_amax), with_v);
    cluster.sync();
  }
  return false;
}

template <int Q, int E, bool EXACT, int GT = 0>
__global__ void __launch_bounds__(kJThreads, (E <= 16 && !(Q == 32 && GT == 8) ? 2 : 1)) jacobi_cluster_kernel(JacobiParams P) {
  extern __shared__ __align__(16) double smem[];
  cg::cluster_group cluster = cg::this_cluster();
  const unsigned rank = cluster.block_rank(), csize = cluster.num_blocks();
  const JacobiJob job = P.jobs[blockIdx.x / csize];
  const uint32_t rows = job.rows, cols_pad = job.cols_pad;
  const uint32_t g = P.g, G = P.G;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool with_v = P.with_v && job.v;
  const uint32_t vrows = cols_pad;
  const uint32_t ldS = rows + 8, ldV = vrows + 8;  // padded: consecutive columns start in alternate bank halves

  double* sW = smem;                                          // 2g columns, stride ldS
  double* sV = sW + (uint64_t)2 * g * ldS;                    // 2g columns, stride ldV (optional)
  double* sAlpha = sV + (with_v ? (uint64_t)2 * g * ldV : 0);  // 2g
  __shared__ double s_red[kJWarps];
  __shared__ double s_amax;
  __shared__ unsigned long long s_rot;
  __shared__ TailShared s_tail;

  unsigned long long* counters = reinterpret_cast<unsigned long long*>(job.stats + 4);  // rotations per sweep, mod 3
  double* W = job.w;
  double* V = job.v;
  double* alpha_g = job.alpha;
  constexpr int kGroups = kJThreads / Q;
  const int grp_id = tid / Q;

  unsigned long long total_rot = 0;
  double last_max_ratio = 0.0;
  int converged = (job.cols < 2);
  int sweep = 0;
  if (P.check_first && !converged) {
    // continuing after the Gram-assisted warp kernel: certify on W first
    sweep = (int)job.stats[0];
    total_rot = job.stats[1];
    int done = sweep;
    converged = run_tail(cluster, job, rank, csize, s_red, &s_amax, &s_tail, with_v, done, total_rot,
                         last_max_ratio);
    sweep = done;
    if (P.debug && rank == 0 && tid == 0 && blockIdx.x == 0)
      printf("[jacobi] job 0: warp kernel %d sweeps, tail -> converged %d after %d\n", (int)job.stats[0], converged,
             sweep);
    cluster.sync();
  }
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
    if (tid == 0) s_rot = 0ull;
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
        if constexpr (EXACT && GT > 0) {
          // compile-time shape: every load of the step is issued before the first
          // store (one L2 round trip per step instead of one per column chunk)
          constexpr uint32_t kR = (uint32_t)(Q * E), kC = 2 * GT / kJWarps, kI = kR / 32;
          double v[kC * kI];
#pragma unroll
          for (uint32_t cc = 0; cc < kC; ++cc) {
            const uint32_t c = warp + cc * kJWarps;
            const uint32_t col = (c < GT ? gA * GT + c : gB * GT + (c - GT));
            const double* src = W + (uint64_t)col * kR + lane;
#pragma unroll
            for (uint32_t i = 0; i < kI; ++i) v[cc * kI + i] = __ldcg(src + 32 * i);
          }
#pragma unroll
          for (uint32_t cc = 0; cc < kC; ++cc) {
            const uint32_t c = warp + cc * kJWarps;
            double* dst = sW + (uint64_t)c * (kR + 8) + lane;
#pragma unroll
            for (uint32_t i = 0; i < kI; ++i) dst[32 * i] = v[cc * kI + i];
            if (lane == 0) sAlpha[c] = __ldcg(alpha_g + (c < GT ? gA * GT + c : gB * GT + (c - GT)));
          }
        } else
        for (uint32_t c = warp; c < 2 * g; c += kJWarps) {
          const uint32_t col = (c < g ? gA * g + c : gB * g + (c - g));
          const double* src = W + (uint64_t)col * rows;
          double* dst = sW + (uint64_t)c * ldS;
          for (uint32_t i = lane; i < rows; i += 32) dst[i] = __ldcg(src + i);
          if (with_v) {
            const double* vs = V + (uint64_t)col * vrows;
            double* vd = sV + (uint64_t)c * ldV;
            for (uint32_t i = lane; i < vrows; i += 32) vd[i] = __ldcg(vs + i);
          }
          if (lane == 0) sAlpha[c] = __ldcg(alpha_g + col);
        }
        __syncthreads();
        // intra-group rounds (first step only: every group appears once)
        if (step == 0) {
          for (uint32_t r = 0; r + 1 < g; ++r) {
            for (uint32_t t = grp_id; t < g; t += kGroups) {
              const uint32_t half = g / 2;
              const uint32_t grp = t / half, i = t % half;
              const uint32_t p = grp * g + rr_slot(i, r, g), q = grp * g + rr_slot(g - 1 - i, r, g);
              double* vp = with_v ? sV + (uint64_t)p * ldV : nullptr;
              double* vq = with_v ? sV + (uint64_t)q * ldV : nullptr;
              int rot = rotate_pair_q<Q>(sW + (uint64_t)p * ldS, sW + (uint64_t)q * ldS, vp, vq, rows, vrows,
                                         sAlpha, p, q, freeze, my_ratio, 0);
              my_rot += ((tid & (Q - 1)) == 0) ? rot : 0;
            }
            __syncthreads();
          }
        }
        // cross rounds: (A_i, B_{(i + r) mod g})
        if constexpr (E > 0) {
          cross_rounds_reg<Q, E, EXACT, GT>(sW, ldS, rows, g, sAlpha, freeze, my_ratio, my_rot);
        } else {
          for (uint32_t r = 0; r < g; ++r) {
            for (uint32_t t = grp_id; t < g; t += kGroups) {
              const uint32_t p = t, q = g + (t + r) % g;
              double* vp = with_v ? sV + (uint64_t)p * ldV : nullptr;
              double* vq = with_v ? sV + (uint64_t)q * ldV : nullptr;
              int rot = rotate_pair_q<Q>(sW + (uint64_t)p * ldS, sW + (uint64_t)q * ldS, vp, vq, rows, vrows,
                                         sAlpha, p, q, freeze, my_ratio, 0);
              my_rot += ((tid & (Q - 1)) == 0) ? rot : 0;
            }
            __syncthreads();
          }
        }
        // write back
        if constexpr (EXACT && Q == 32 && GT == 8) {
          // the one-CTA-per-SM instantiation has the registers: all shared-memory
          // loads of the warp first, then the global stores
          constexpr uint32_t kR = (uint32_t)(Q * E), kC = 2 * GT / kJWarps, kI = kR / 32;
          double v[kC * kI];
#pragma unroll
          for (uint32_t cc = 0; cc < kC; ++cc) {
            const double* src = sW + (uint64_t)(warp + cc * kJWarps) * (kR + 8) + lane;
#pragma unroll
            for (uint32_t i = 0; i < kI; ++i) v[cc * kI + i] = src[32 * i];
          }
#pragma unroll
          for (uint32_t cc = 0; cc < kC; ++cc) {
            const uint32_t c = warp + cc * kJWarps;
            const uint32_t col = (c < GT ? gA * GT + c : gB * GT + (c - GT));
            double* dst = W + (uint64_t)col * kR + lane;
#pragma unroll
            for (uint32_t i = 0; i < kI; ++i) dst[32 * i] = v[cc * kI + i];
            if (lane == 0) alpha_g[col] = sAlpha[c];
          }
        } else
        for (uint32_t c = warp; c < 2 * g; c += kJWarps) {
          const uint32_t col = (c < g ? gA * g + c : gB * g + (c - g));
          double* dst = W + (uint64_t)col * rows;
          const double* src = sW + (uint64_t)c * ldS;
          for (uint32_t i = lane; i < rows; i += 32) dst[i] = src[i];
          if (with_v) {
            double* vd = V + (uint64_t)col * vrows;
            const double* vs = sV + (uint64_t)c * ldV;
            for (uint32_t i = lane; i < vrows; i += 32) vd[i] = vs[i];
          }
          if (lane == 0) alpha_g[col] = sAlpha[c];
        }
        __syncthreads();
      }
      if (step + 2 == G) {
        // last step of the sweep: publish this CTA's rotation count and max ratio
        if (my_rot) atomicAdd(&s_rot, my_rot);
        for (int o = 16; o; o >>= 1) my_ratio = fmax(my_ratio, __shfl_xor_sync(0xffffffffu, my_ratio, o));
        if (lane == 0) s_red[warp] = my_ratio;
        __syncthreads();
        if (tid == 0) {
          double t = 0.0;
          for (int w = 0; w < kJWarps; ++w) t = fmax(t, s_red[w]);
          if (s_rot) atomicAdd(&counters[sweep % 3], s_rot);
          // max ratio across the cluster (my_ratio holds ratio^2); doubles >= 0
          // order like their bit patterns
          atomicMax(reinterpret_cast<unsigned long long*>(job.stats + 3), __double_as_longlong(sqrt(t)));
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
    // quadratic regime: the convergence tail (see tail_check)
    if (!converged && last_max_ratio < P.check_ratio && sweep + 1 < kMaxSweeps) {
      int done = sweep + 1;
      converged = run_tail(cluster, job, rank, csize, s_red, &s_amax, &s_tail, with_v, done, total_rot,
                           last_max_ratio);
      sweep = done - 1;  // the loop increment counts it
    }
  }
  if (rank == 0 && tid == 0) {
    job.stats[0] = (uint64_t)sweep;
    job.stats[1] = total_rot;
    job.stats[2] = converged ? 0ull : 1ull;
    job.stats[3] = (uint64_t)__double_as_longlong(last_max_ratio);
    if (P.debug && blockIdx.x == 0) printf("[jacobi] job 0: %d sweeps in all, converged %d\n", sweep, converged);
  }
}

// ===========================================================================
// Gram-assisted warp Jacobi (matrices accepted on the Gram route, kappa bounded)
// ===========================================================================
// The same tournament over groups of kWG = 8 columns, but one WARP owns a group
// pair for a whole step:
//   1. H = X^T X (16 x 16, X = the pair's 16 columns) by DMMA straight from W;
//   2. the step's rounds (intra-group rounds in step 0, then 8 cross rounds) on H
//      in the warp's shared memory -- a rotation of columns (p, q) is the two-sided
//      update H <- J^T H J (rows, then columns) -- with the reference's decision
//      rule and formulas on H's entries, accumulating Z = J_1 J_2 ... in registers;
//   3. X <- X Z by DMMA, back into W.
// The only barrier is one per step among the matrix's warps (a cluster of G/16
// CTAs), and the M-long work runs on the tensor cores. H is formed afresh every
// step and only the step's rotations are applied to it, so for the kappa the Gram
// route admits its rounding stays far below the 1e-14 rotation threshold. Once a
// sweep's largest |gamma| / sqrt(alpha_p alpha_q) is in the quadratic regime the
// kernel hands over to jacobi_cluster_kernel, which certifies convergence on W
// itself (tail_check) -- the reference's stopping rule. Convergence is measured on
// the fresh H of every step (fresh_scan), so the within-step rounding of H on graded
// columns neither stalls nor fakes it: any conditioning may run here.
constexpr int kWG = 8, kWN = 16, kWS = 17;

struct WarpParams {
  const JacobiJob* jobs;
  uint32_t G;         // groups of kWG columns (even), G * kWG = cols_pad
  double stop_ratio;  // hand over once a sweep's max ratio is below this
};

template <int KIND, int R>  // KIND 0: cross round R; 1: intra-group round R
__device__ __forceinline__ void round_pair(int i, int& p, int& q) {
  if (KIND == 0) {
    p = i;
    q = 8 + ((i + R) & 7);
  } else {
    const int grp = i >> 2, t = i & 3;
    const int a = t, b = 7 - t;
    p = grp * 8 + (a == 0 ? 0 : 1 + (a - 1 + R) % 7);
    q = grp * 8 + (b == 0 ? 0 : 1 + (b - 1 + R) % 7);
  }
}

template <int KIND, int R>
__device__ __forceinline__ void warp_round(double* sH, double* sCS, double (&z)[kWN], double freeze, double& max_r2,
                                           uint32_t& nrot) {
  const int lane = threadIdx.x & 31;
  if (lane < 8) {
    int p, q;
    round_pair<KIND, R>(lane, p, q);
    const double ap = sH[p * kWS + p], aq = sH[q * kWS + q], gm = sH[p * kWS + q];
    double c = 1.0, sn = 0.0;
    const bool live = !(ap <= freeze || aq <= freeze);
    const double prod = ap * aq, g2 = gm * gm;
    if (live && g2 > max_r2 * prod) max_r2 = g2 / prod;
    if (live && g2 > kJacobiTol * kJacobiTol * prod) {
      rotation_cs(ap, aq, gm, c, sn);
      ++nrot;
    }
    sCS[2 * lane] = c;
    sCS[2 * lane + 1] = sn;
  }
  __syncwarp();
  double cs[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) cs[i] = sCS[i];
  if (lane < kWN) {  // rows p, q of H; lane owns column `lane`
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      int p, q;
      round_pair<KIND, R>(i, p, q);
      const double x = sH[p * kWS + lane], y = sH[q * kWS + lane];
      sH[p * kWS + lane] = cs[2 * i] * x - cs[2 * i + 1] * y;
      sH[q * kWS + lane] = cs[2 * i + 1] * x + cs[2 * i] * y;
    }
  } else {  // Z <- Z J; lane owns row lane - 16
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      int p, q;
      round_pair<KIND, R>(i, p, q);
      const double x = z[p], y = z[q];
      z[p] = cs[2 * i] * x - cs[2 * i + 1] * y;
      z[q] = cs[2 * i + 1] * x + cs[2 * i] * y;
    }
  }
  __syncwarp();
  if (lane < kWN) {  // columns p, q of H; lane owns row `lane`
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      int p, q;
      round_pair<KIND, R>(i, p, q);
      const double x = sH[lane * kWS + p], y = sH[lane * kWS + q];
      sH[lane * kWS + p] = cs[2 * i] * x - cs[2 * i + 1] * y;
      sH[lane * kWS + q] = cs[2 * i + 1] * x + cs[2 * i] * y;
    }
  }
  __syncwarp();
}

// One round of the step on H (16 x 17 in the warp's shared memory), all 32 lanes
// on one instruction stream (no divergent halves):
//   1. lanes 0..7 take the angles of the round's 8 disjoint pairs (every lane runs
//      the arithmetic, selects instead of branches) -- and, in the same basic
//      block, every lane applies the PREVIOUS round's rotations to its row of Z in
//      registers, which hides under the angle's latency;
//   2. H <- J^T H J in one pass: the 64 2 x 2 blocks (row pair i, column pair j)
//      are independent (B' = J_i^T B J_j); a lane owns two of them.
template <int KIND, int R>
__device__ __forceinline__ void z_apply(double (&z)[kWN], const double (&cs)[16]) {
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    int p, q;
    round_pair<KIND, R>(i, p, q);
    const double x = z[p], y = z[q];
    z[p] = cs[2 * i] * x - cs[2 * i + 1] * y;
    z[q] = cs[2 * i + 1] * x + cs[2 * i] * y;
  }
}

// PK/PR: the previous round (its rotations are in cs and still have to reach Z); PK < 0: none
template <int KIND, int R, int PK, int PR>
__device__ __forceinline__ void smem_round2(double* sH, double (&z)[kWN], double (&cs)[16],
                                            double freeze, uint32_t& nrot) {
  const int lane = threadIdx.x & 31;
  {
    int p, q;
    round_pair<KIND, R>(lane & 7, p, q);
    const double ap = sH[p * kWS + p], aq = sH[q * kWS + q], gm = sH[p * kWS + q];
    if constexpr (PK >= 0) z_apply<PK, PR>(z, cs);  // independent of the angle: overlaps its latency
    const double prod = ap * aq, g2 = gm * gm;
    const bool rot = ap > freeze && aq > freeze && g2 > kJacobiTol * kJacobiTol * prod;
    double c, sn;
    rotation_cs(ap, aq, rot ? gm : 1.0, c, sn);
    if (lane < 8) {
      sH[(2 * lane) * kWS + kWN] = rot ? c : 1.0;
      sH[(2 * lane + 1) * kWS + kWN] = rot ? sn : 0.0;
      nrot += rot ? 1u : 0u;
    }
  }
  __syncwarp();
#pragma unroll
  for (int i = 0; i < 16; ++i) cs[i] = sH[i * kWS + kWN];
  {
    const int i = lane >> 2, j0 = 2 * (lane & 3);
    int pi, qi;
    round_pair<KIND, R>(i, pi, qi);
    const double ci = sH[(2 * i) * kWS + kWN], si = sH[(2 * i + 1) * kWS + kWN];
    double* rp = sH + pi * kWS;
    double* rq = sH + qi * kWS;
    double b[2][4];
    int pj[2], qj[2];
    double cj[2], sj[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      round_pair<KIND, R>(j0 + u, pj[u], qj[u]);
      cj[u] = sH[(2 * (j0 + u)) * kWS + kWN];
      sj[u] = sH[(2 * (j0 + u) + 1) * kWS + kWN];
      b[u][0] = rp[pj[u]];
      b[u][1] = rp[qj[u]];
      b[u][2] = rq[pj[u]];
      b[u][3] = rq[qj[u]];
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const double t00 = cj[u] * b[u][0] - sj[u] * b[u][1], t01 = sj[u] * b[u][0] + cj[u] * b[u][1];
      const double t10 = cj[u] * b[u][2] - sj[u] * b[u][3], t11 = sj[u] * b[u][2] + cj[u] * b[u][3];
      rp[pj[u]] = ci * t00 - si * t10;
      rp[qj[u]] = ci * t01 - si * t11;
      rq[pj[u]] = si * t00 + ci * t10;
      rq[qj[u]] = si * t01 + ci * t11;
    }
  }
  __syncwarp();
}

// The fresh H of a step (before any rotation touches it): the largest
// gamma^2 / (alpha_p alpha_q) over the 120 pairs of its 16 columns, kept as a
// fraction (best_g2 / best_prod), and whether any pair this step rotates (all of
// them in step 0, the cross pairs later) is over the rotation threshold. The pairs
// are folded into 8 rows of 15 (row fr, then row 15 - fr), 4 lanes a row.
__device__ __forceinline__ bool fresh_scan(const double* sH, double freeze, bool intra, double& best_g2,
                                           double& best_prod) {
  const int lane = threadIdx.x & 31, fr = lane >> 2, sub = lane & 3;
  bool need = false;
#pragma unroll
  for (int e0 = 0; e0 < 16; e0 += 4) {
    const int e = e0 + sub;
    if (e < 15) {
      const bool first = e < 15 - fr;
      const int i = first ? fr : 15 - fr, j = first ? fr + 1 + e : 1 + e;
      const double aii = sH[i * kWS + i], ajj = sH[j * kWS + j], gij = sH[i * kWS + j];
      const double prod = aii * ajj, g2 = gij * gij;
      const bool live = aii > freeze && ajj > freeze;
      if (live && g2 * best_prod > best_g2 * prod) {
        best_g2 = g2;
        best_prod = prod;
      }
      need = need || (live && g2 > kJacobiTol * kJacobiTol * prod && (intra || (i < kWG && j >= kWG)));
    }
  }
  return __any_sync(0xffffffffu, need);
}

// The rounds of one step on H; leaves Z (16 x 16 row-major, stride kWN) where H was.
__device__ __forceinline__ void step_rounds(double* sH, bool intra, double freeze, uint32_t& nrot,
                                            double* keepA = nullptr, double* keepB = nullptr) {
  const int lane = threadIdx.x & 31;
  double z[kWN], cs[16];
#pragma unroll
  for (int k = 0; k < kWN; ++k) z[k] = (k == (lane & 15)) ? 1.0 : 0.0;  // lanes 16..31 mirror 0..15
  if (intra) {
    smem_round2<1, 0, -1, 0>(sH, z, cs, freeze, nrot);
    smem_round2<1, 1, 1, 0>(sH, z, cs, freeze, nrot);
    smem_round2<1, 2, 1, 1>(sH, z, cs, freeze, nrot);
    smem_round2<1, 3, 1, 2>(sH, z, cs, freeze, nrot);
    smem_round2<1, 4, 1, 3>(sH, z, cs, freeze, nrot);
    smem_round2<1, 5, 1, 4>(sH, z, cs, freeze, nrot);
    smem_round2<1, 6, 1, 5>(sH, z, cs, freeze, nrot);
    smem_round2<0, 0, 1, 6>(sH, z, cs, freeze, nrot);
  } else {
    smem_round2<0, 0, -1, 0>(sH, z, cs, freeze, nrot);
  }
  smem_round2<0, 1, 0, 0>(sH, z, cs, freeze, nrot);
  smem_round2<0, 2, 0, 1>(sH, z, cs, freeze, nrot);
  smem_round2<0, 3, 0, 2>(sH, z, cs, freeze, nrot);
  smem_round2<0, 4, 0, 3>(sH, z, cs, freeze, nrot);
  smem_round2<0, 5, 0, 4>(sH, z, cs, freeze, nrot);
  smem_round2<0, 6, 0, 5>(sH, z, cs, freeze, nrot);
  smem_round2<0, 7, 0, 6>(sH, z, cs, freeze, nrot);
  z_apply<0, 7>(z, cs);
  if (keepA) {  // the rotated diagonal blocks (8 x 8 each) outlive the step: the groups carry them
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int t = lane + 32 * u, i = t >> 3, j = t & 7;
      __stcg(keepA + t, sH[i * kWS + j]);
      __stcg(keepB + t, sH[(kWG + i) * kWS + kWG + j]);
    }
    __syncwarp();
  }
  if (lane < kWN) {  // H is dead: Z takes its place
#pragma unroll
    for (int k = 0; k < kWN; ++k) sH[lane * kWN + k] = z[k];
  }
  __syncwarp();
}

// H = X^T X for the 16 columns cA..cA+7, cB..cB+7 of W (column-major, ld rows)
__device__ __forceinline__ void warp_gram(const double* __restrict__ W, uint32_t rows, uint32_t cA, uint32_t cB,
                                          double* sH) {
  const int lane = threadIdx.x & 31, lr = lane >> 2, lc = lane & 3;
  const double* pa = W + (uint64_t)(cA + lr) * rows + lc;
  const double* pb = W + (uint64_t)(cB + lr) * rows + lc;
  double h[12];
#pragma unroll
  for (int i = 0; i < 12; ++i) h[i] = 0.0;
  uint32_t k0 = 0;
  // 8 k-steps per batch: 16 loads in flight before the 24 DMMAs that use them
  for (; k0 + 32 <= rows; k0 += 32) {
    double a[8], b[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      a[u] = __ldcg(pa + k0 + 4 * u);
      b[u] = __ldcg(pb + k0 + 4 * u);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int o = (u & 1) * 6;
      dmma884(h[o], h[o + 1], a[u], a[u]);
      dmma884(h[o + 2], h[o + 3], b[u], a[u]);
      dmma884(h[o + 4], h[o + 5], b[u], b[u]);
    }
  }
  for (; k0 + 8 <= rows; k0 += 8) {
    const double a0 = __ldcg(pa + k0), b0 = __ldcg(pb + k0), a1 = __ldcg(pa + k0 + 4), b1 = __ldcg(pb + k0 + 4);
    dmma884(h[0], h[1], a0, a0);
    dmma884(h[2], h[3], b0, a0);
    dmma884(h[4], h[5], b0, b0);
    dmma884(h[6], h[7], a1, a1);
    dmma884(h[8], h[9], b1, a1);
    dmma884(h[10], h[11], b1, b1);
  }
  for (; k0 < rows; k0 += 4) {
    const bool ok = k0 + lc < rows;
    const double a0 = ok ? __ldcg(pa + k0) : 0.0, b0 = ok ? __ldcg(pb + k0) : 0.0;
    dmma884(h[0], h[1], a0, a0);
    dmma884(h[2], h[3], b0, a0);
    dmma884(h[4], h[5], b0, b0);
  }
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    const int j = 2 * lc + e;
    const double t00 = h[e] + h[6 + e], t10 = h[2 + e] + h[8 + e], t11 = h[4 + e] + h[10 + e];
    sH[lr * kWS + j] = t00;              // (A, A)
    sH[(8 + lr) * kWS + j] = t10;        // (B, A)
    sH[j * kWS + 8 + lr] = t10;          // (A, B) mirror
    sH[(8 + lr) * kWS + 8 + j] = t11;    // (B, B)
  }
  __syncwarp();
}

// X <- X Z (Z from the warp's shared memory, row-major 16 x 16)
__device__ __forceinline__ void warp_xz(double* __restrict__ W, uint32_t rows, uint32_t cA, uint32_t cB,
                                        const double* sZ) {
  const int lane = threadIdx.x & 31, lr = lane >> 2, lc = lane & 3;
  double bf[4][2];
#pragma unroll
  for (int kc = 0; kc < 4; ++kc)
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) bf[kc][nt] = sZ[(4 * kc + lc) * kWN + 8 * nt + lr];
  const double* src[4];
#pragma unroll
  for (int kc = 0; kc < 4; ++kc) {
    const int t = 4 * kc + lc;
    src[kc] = W + (uint64_t)(t < kWG ? cA + t : cB + t - kWG) * rows;
  }
  double* dst[2][2];
#pragma unroll
  for (int nt = 0; nt < 2; ++nt)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int t = 8 * nt + 2 * lc + e;
      dst[nt][e] = W + (uint64_t)(t < kWG ? cA + t : cB + t - kWG) * rows;
    }
  // 4 row blocks per batch: 16 loads in flight
  constexpr int kRB = 4;
  for (uint32_t r0 = 0; r0 < rows; r0 += 8 * kRB) {
    double af[kRB][4];
#pragma unroll
    for (int u = 0; u < kRB; ++u) {
      const uint32_t r = r0 + 8 * u + lr;
#pragma unroll
      for (int kc = 0; kc < 4; ++kc) af[u][kc] = r < rows ? __ldcg(src[kc] + r) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < kRB; ++u) {
      const uint32_t r = r0 + 8 * u + lr;
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
        double d0 = 0.0, d1 = 0.0;
#pragma unroll
        for (int kc = 0; kc < 4; ++kc) dmma884(d0, d1, af[u][kc], bf[kc][nt]);
        if (r < rows) {
          dst[nt][0][r] = d0;
          dst[nt][1][r] = d1;
        }
      }
    }
  }
}

__global__ void __launch_bounds__(kJThreads, 2) jacobi_warp_kernel(WarpParams P) {
  cg::cluster_group cluster = cg::this_cluster();
  const unsigned rank = cluster.block_rank(), csize = cluster.num_blocks();
  const JacobiJob job = P.jobs[blockIdx.x / csize];
  const uint32_t rows = job.rows, cols_pad = job.cols_pad, G = P.G, npairs = G / 2;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  __shared__ double sH[kJWarps][kWN * kWS];  // H, then Z (step_rounds)
  __shared__ double s_red[kJWarps];
  __shared__ double s_amax;
  __shared__ unsigned long long s_rot;
  unsigned long long* counters = reinterpret_cast<unsigned long long*>(job.stats + 4);
  double* W = job.w;
  double* alpha_g = job.alpha;
  const uint32_t w = rank * kJWarps + warp;  // this warp's first pair slot
  constexpr int kWarpMaxSweeps = 40;        // leave sweeps for the direct kernel
  double prev_ratio = INFINITY;

  unsigned long long total_rot = 0;
  double last_max_ratio = 0.0;
  int converged = (job.cols < 2);
  int sweep = 0;
  for (; sweep < kMaxSweeps && !converged; ++sweep) {
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
    if (tid == 0) s_rot = 0ull;
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
      for (int i = 0; i < kJWarps; ++i) t = fmax(t, s_red[i]);
      s_amax = t;
    }
    __syncthreads();
    const double freeze = kJacobiTol * kJacobiTol * s_amax;
    uint32_t nrot = 0;
    double best_g2 = 0.0, best_prod = 1.0;  // the sweep's largest fresh ratio^2, as a fraction
    for (uint32_t step = 0; step + 1 < G; ++step) {
      for (uint32_t pw = w; pw < npairs; pw += csize * kJWarps) {
        const uint32_t cA = rr_slot(pw, step, G) * kWG, cB = rr_slot(G - 1 - pw, step, G) * kWG;
        double* h = sH[warp];
        warp_gram(W, rows, cA, cB, h);
        // rotate only where the fresh H has a pair over the threshold (late sweeps: few)
        if (fresh_scan(h, freeze, step == 0, best_g2, best_prod)) {
          step_rounds(h, step == 0, freeze, nrot);
          warp_xz(W, rows, cA, cB, h);
        }
        __syncwarp();  // Z is consumed before the next pair's H lands on it
      }
      cluster.sync();
    }
    // rotations and the largest ratio of the sweep, over the cluster
    unsigned long long r64 = nrot;
    double max_r2 = best_g2 / best_prod;
    for (int o = 16; o; o >>= 1) {
      r64 += __shfl_xor_sync(0xffffffffu, r64, o);
      max_r2 = fmax(max_r2, __shfl_xor_sync(0xffffffffu, max_r2, o));
    }
    if (lane == 0) {
      if (r64) atomicAdd(&s_rot, r64);
      s_red[warp] = max_r2;
    }
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
      for (int i = 0; i < kJWarps; ++i) t = fmax(t, s_red[i]);
      if (s_rot) atomicAdd(&counters[sweep % 3], s_rot);
      atomicMax(reinterpret_cast<unsigned long long*>(job.stats + 3), __double_as_longlong(sqrt(t)));
    }
    cluster.sync();
    const unsigned long long rot = __ldcg(&counters[sweep % 3]);
    total_rot += rot;
    last_max_ratio = __longlong_as_double(__ldcg(reinterpret_cast<long long*>(job.stats + 3)));
    cluster.sync();
    if (rank == 0 && tid == 0) job.stats[3] = 0ull;
    // hand over: converged on H, in the quadratic regime, or stagnating (the
    // rounding of H-based decisions on a badly conditioned pair) -- the direct
    // kernel finishes on W either way
    const bool stagnant = sweep >= 3 && last_max_ratio < 1e-4 && last_max_ratio > 0.25 * prev_ratio;
    if (rot == 0 || last_max_ratio < P.stop_ratio || stagnant || sweep + 1 >= kWarpMaxSweeps) {
      ++sweep;
      break;
    }
    prev_ratio = last_max_ratio;
    cluster.sync();
  }
  cluster.sync();
  if (rank == 0 && tid == 0) {
    job.stats[0] = (uint64_t)sweep;
    job.stats[1] = total_rot;
    job.stats[2] = 0ull;
    job.stats[3] = (uint64_t)__double_as_longlong(last_max_ratio);
    job.stats[4] = job.stats[5] = job.stats[6] = 0ull;
  }
}

// ===========================================================================
// Shared-memory-resident Gram-assisted Jacobi (matrices that fit a cluster's
// shared memory: c3's reduced R factors, c2's 256 x 256 Cholesky factors)
// ===========================================================================
// The tournament and the step of jacobi_warp_kernel (H = X^T X by DMMA, the
// step's rounds on H in the warp's shared memory, X <- X Z by DMMA), but the
// matrix stays in shared memory for the whole run: a cluster of C CTAs holds it
// (CTA r owns the column groups [r Gc, (r+1) Gc)), a warp reaches both groups of
// its pair through (distributed) shared memory, and global memory is touched
// twice: the load and the write-back. Only the first rows_nz rows are staged
// (a reduced R is n_d x n_d in a taller zero-padded slot; zero rows stay zero).
// Convergence is measured on the FRESH H of every step (all 120 pairs of the 16
// columns, before any rotation touches H), so the within-step rounding of H on
// graded columns cannot stall or fake it. A group pair whose fresh H has no
// pair over the rotation threshold skips its rounds and its X Z. Hands over to
// jacobi_cluster_kernel (check_first) once a sweep's largest fresh ratio is in
// the quadratic regime; that kernel certifies on W with the reference's rule.
struct SmemParams {
  const JacobiJob* jobs;
  uint32_t ld;        // shared-memory column stride (doubles), = 4 mod 8
  uint32_t cap_cols;  // columns the layout holds per CTA (multiple of 8)
  uint32_t nw;        // warps per CTA
  double stop_ratio;
  double* keep;          // per job of the launch: its groups' carried diagonal blocks (null: full Grams every step)
  uint64_t keep_stride;  // doubles per job
};
constexpr int kSH = kWN * kWS;  // doubles per warp: H (16 x 17); its pad column holds the round's 8 (c, s)
constexpr int kSmemMaxWarps = 12;
constexpr int kSmemMisc = 32 + 4;    // s_red, s_pub


__device__ __forceinline__ void smem_gram(const double* pA, const double* pB, uint32_t ld, uint32_t rows,
                                          double* sH) {
  const int lane = threadIdx.x & 31, lr = lane >> 2, lc = lane & 3;
  const double* pa = pA + (uint32_t)lr * ld + lc;
  const double* pb = pB + (uint32_t)lr * ld + lc;
  double h[12];
#pragma unroll
  for (int i = 0; i < 12; ++i) h[i] = 0.0;
  uint32_t k0 = 0;
  for (; k0 + 16 <= rows; k0 += 16) {
    double a[4], b[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      a[u] = pa[k0 + 4 * u];
      b[u] = pb[k0 + 4 * u];
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int o = (u & 1) * 6;
      dmma884(h[o], h[o + 1], a[u], a[u]);
      dmma884(h[o + 2], h[o + 3], b[u], a[u]);
      dmma884(h[o + 4], h[o + 5], b[u], b[u]);
    }
  }
  for (; k0 < rows; k0 += 8) {  // rows is a multiple of 8
    const double a0 = pa[k0], b0 = pb[k0], a1 = pa[k0 + 4], b1 = pb[k0 + 4];
    dmma884(h[0], h[1], a0, a0);
    dmma884(h[2], h[3], b0, a0);
    dmma884(h[4], h[5], b0, b0);
    dmma884(h[6], h[7], a1, a1);
    dmma884(h[8], h[9], b1, a1);
    dmma884(h[10], h[11], b1, b1);
  }
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    const int j = 2 * lc + e;
    const double t00 = h[e] + h[6 + e], t10 = h[2 + e] + h[8 + e], t11 = h[4 + e] + h[10 + e];
    sH[lr * kWS + j] = t00;
    sH[(8 + lr) * kWS + j] = t10;
    sH[j * kWS + 8 + lr] = t10;
    sH[(8 + lr) * kWS + 8 + j] = t11;
  }
  __syncwarp();
}

// The cross block (B, A) only, by DMMA; the two diagonal blocks come from the
// groups' carried 8 x 8 blocks (kept by step_rounds after the groups' last step,
// seeded afresh by the full Gram of every sweep's step 0): a third of the Gram's
// DMMAs. The carried blocks are H entries that have been through the rotations of
// the steps since -- the same two-sided updates the rounds of one step apply.
__device__ __forceinline__ void smem_gram_cross(const double* pA, const double* pB, uint32_t ld, uint32_t rows,
                                                const double* keepA, const double* keepB, double* sH) {
  const int lane = threadIdx.x & 31, lr = lane >> 2, lc = lane & 3;
  double da[2], db[2];
#pragma unroll
  for (int u = 0; u < 2; ++u) {  // issued first: in flight during the DMMA loop
    da[u] = __ldcg(keepA + lane + 32 * u);
    db[u] = __ldcg(keepB + lane + 32 * u);
  }
  const double* pa = pA + (uint32_t)lr * ld + lc;
  const double* pb = pB + (uint32_t)lr * ld + lc;
  double h[4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i) h[i][0] = h[i][1] = 0.0;
  uint32_t k0 = 0;
  for (; k0 + 16 <= rows; k0 += 16) {
    double a[4], b[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      a[u] = pa[k0 + 4 * u];
      b[u] = pb[k0 + 4 * u];
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) dmma884(h[u][0], h[u][1], b[u], a[u]);
  }
  for (; k0 < rows; k0 += 8) {  // rows is a multiple of 8
    const double a0 = pa[k0], b0 = pb[k0], a1 = pa[k0 + 4], b1 = pb[k0 + 4];
    dmma884(h[0][0], h[0][1], b0, a0);
    dmma884(h[1][0], h[1][1], b1, a1);
  }
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    const int j = 2 * lc + e;
    const double t10 = (h[0][e] + h[1][e]) + (h[2][e] + h[3][e]);
    sH[(8 + lr) * kWS + j] = t10;
    sH[j * kWS + 8 + lr] = t10;
  }
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const int t = lane + 32 * u, i = t >> 3, j = t & 7;
    sH[i * kWS + j] = da[u];
    sH[(kWG + i) * kWS + kWG + j] = db[u];
  }
  __syncwarp();
}

__device__ __forceinline__ void smem_xz(double* pA, double* pB, uint32_t ld, uint32_t rows, const double* sZ) {
  const int lane = threadIdx.x & 31, lr = lane >> 2, lc = lane & 3;
  double bf[4][2];
#pragma unroll
  for (int kc = 0; kc < 4; ++kc)
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) bf[kc][nt] = sZ[(4 * kc + lc) * kWN + 8 * nt + lr];
  const double* src[4];
#pragma unroll
  for (int kc = 0; kc < 4; ++kc) {
    const int t = 4 * kc + lc;
    src[kc] = (t < kWG ? pA + (uint32_t)t * ld : pB + (uint32_t)(t - kWG) * ld) + lr;
  }
  double* dst[2][2];
#pragma unroll
  for (int nt = 0; nt < 2; ++nt)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int t = 8 * nt + 2 * lc + e;
      dst[nt][e] = (t < kWG ? pA + (uint32_t)t * ld : pB + (uint32_t)(t - kWG) * ld) + lr;
    }
  constexpr int kRB = 4;  // 16 loads in flight; every lane's loads precede the first DMMA of the batch
  for (uint32_t r0 = 0; r0 < rows; r0 += 8 * kRB) {
    double af[kRB][4];
#pragma unroll
    for (int u = 0; u < kRB; ++u) {
      const uint32_t r = r0 + 8 * u;
#pragma unroll
      for (int kc = 0; kc < 4; ++kc) af[u][kc] = r < rows ? src[kc][r] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < kRB; ++u) {
      const uint32_t r = r0 + 8 * u;
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
        double d0 = 0.0, d1 = 0.0;
#pragma unroll
        for (int kc = 0; kc < 4; ++kc) dmma884(d0, d1, af[u][kc], bf[kc][nt]);
        if (r < rows) {
          dst[nt][0][r] = d0;
          dst[nt][1][r] = d1;
        }
      }
    }
  }
}

template <bool MULTI>
__global__ void __launch_bounds__(kSmemMaxWarps * 32, 1) jacobi_smem_kernel(SmemParams P) {
  extern __shared__ __align__(16) double smem[];
  cg::cluster_group cluster = cg::this_cluster();
  const unsigned rank = MULTI ? cluster.block_rank() : 0u, csize = MULTI ? cluster.num_blocks() : 1u;
  const JacobiJob job = P.jobs[blockIdx.x / csize];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t ld = P.ld;
  const uint32_t colsU = (job.cols + 15u) & ~15u;               // columns in the tournament
  const uint32_t G = colsU / kWG, npairs = G / 2;
  const uint32_t Gc = (G + csize - 1) / csize;                  // groups per CTA
  const uint32_t rows = (min(job.rows, job.rows_nz ? job.rows_nz : job.rows) + 7u) & ~7u;  // staged rows
  double* mat = smem;                                           // [cap_cols][ld]
  double* sHall = mat + (uint64_t)P.cap_cols * ld;              // [nw][kSH]
  double* s_red = sHall + (uint64_t)P.nw * kSH;                 // [32]
  double* s_pub = s_red + 32;                                   // [4]: amax, ratio^2, rotations (bits), spare
  double* sH = sHall + (uint64_t)warp * kSH;
  double* W = job.w;
  auto sync_all = [&]() {
    if (MULTI) cluster.sync();
    else __syncthreads();
  };
  auto group_ptr = [&](uint32_t grp) -> double* {  // first column of a group, wherever it lives
    const uint32_t owner = grp / Gc, loc = grp - owner * Gc;
    double* base = MULTI ? cluster.map_shared_rank(mat, owner) : mat;
    return base + (uint64_t)loc * kWG * ld;
  };
  // ---- stage this CTA's columns (zero beyond the job's extents) ----
  const uint32_t my_cols = min(Gc, G > rank * Gc ? G - rank * Gc : 0u) * kWG;
  for (uint32_t c = warp; c < my_cols; c += P.nw) {
    const uint32_t j = rank * Gc * kWG + c;
    const double* wj = W + (uint64_t)j * job.rows;
    for (uint32_t i = lane; i < rows; i += 32)
      mat[(uint64_t)c * ld + i] = (j < job.cols_pad && i < job.rows) ? __ldcg(wj + i) : 0.0;
  }
  sync_all();
  const uint32_t pw = rank * P.nw + warp;  // this warp's pair slot
  double* keep = P.keep ? P.keep + (uint64_t)(blockIdx.x / csize) * P.keep_stride : nullptr;  // G x 64 carried blocks
  unsigned long long total_rot = 0;
  double last_ratio = 0.0, prev_ratio = INFINITY;
#ifdef RK_SMEM_PROBE
  long long pt[6] = {0, 0, 0, 0, 0, 0}, pt0 = 0;  // gram, ratio, rounds, xz, step barrier, sweep head/tail
  long long skipped = 0, worked = 0;
#define PROBE_T0() pt0 = clock64()
#define PROBE_ADD(i) do { const long long now_ = clock64(); pt[i] += now_ - pt0; pt0 = now_; } while (0)
#else
#define PROBE_T0()
#define PROBE_ADD(i)
#endif
  int sweep = 0;
  constexpr int kSmemMaxSweeps = 40;
  bool go = job.cols >= 2;
  while (go) {
    // ---- alpha_max of the sweep (freeze threshold, svd.cpp:222-231) ----
    double amax = 0.0;
    for (uint32_t c = warp; c < my_cols; c += P.nw) {
      const double* x = mat + (uint64_t)c * ld;
      double a = 0.0;
      for (uint32_t i = lane; i < rows; i += 32) a += x[i] * x[i];
      amax = fmax(amax, warp_sum(a));
    }
    if (lane == 0) s_red[warp] = amax;
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
      for (uint32_t i = 0; i < P.nw; ++i) t = fmax(t, s_red[i]);
      s_pub[0] = t;
    }
    sync_all();
    amax = 0.0;
    for (unsigned r = 0; r < csize; ++r) amax = fmax(amax, (MULTI ? cluster.map_shared_rank(s_pub, r) : s_pub)[0]);
    const double freeze = kJacobiTol * kJacobiTol * amax;
    uint32_t nrot = 0;
    double best_g2 = 0.0, best_prod = 1.0;  // the largest gamma^2 / (alpha_p alpha_q) as a fraction
    for (uint32_t step = 0; step + 1 < G; ++step) {
      if (pw < npairs) {
        const uint32_t gA = rr_slot(pw, step, G), gB = rr_slot(G - 1 - pw, step, G);
        double* pA = group_ptr(gA);
        double* pB = group_ptr(gB);
        double* keepA = keep ? keep + (uint64_t)gA * (kWG * kWG) : nullptr;
        double* keepB = keep ? keep + (uint64_t)gB * (kWG * kWG) : nullptr;
        PROBE_T0();
        if (step == 0 || !keep) {
          smem_gram(pA, pB, ld, rows, sH);
        } else {
          smem_gram_cross(pA, pB, ld, rows, keepA, keepB, sH);
        }
        PROBE_ADD(0);
        // fresh ratios of the 16 columns' pairs; does any pair this step rotates exceed the threshold?
        const bool any_need = fresh_scan(sH, freeze, step == 0, best_g2, best_prod);
        PROBE_ADD(1);
#ifdef RK_SMEM_PROBE
        if (any_need) ++worked; else ++skipped;
#endif
        if (any_need) {
          step_rounds(sH, step == 0, freeze, nrot, keepA, keepB);
          PROBE_ADD(2);
          smem_xz(pA, pB, ld, rows, sH);
          PROBE_ADD(3);
        } else if (keep && step == 0) {  // seed the carried blocks with the fresh ones
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const int t = lane + 32 * u, i = t >> 3, j = t & 7;
            __stcg(keepA + t, sH[i * kWS + j]);
            __stcg(keepB + t, sH[(kWG + i) * kWS + kWG + j]);
          }
        }
      }
      PROBE_T0();
      sync_all();
      PROBE_ADD(4);
    }
    // ---- the sweep's rotations and largest fresh ratio, over the cluster ----
    unsigned long long r64 = nrot;
    double max_r2 = best_g2 / best_prod;
    for (int o = 16; o; o >>= 1) {
      r64 += __shfl_xor_sync(0xffffffffu, r64, o);
      max_r2 = fmax(max_r2, __shfl_xor_sync(0xffffffffu, max_r2, o));
    }
    if (lane == 0) {
      s_red[warp] = max_r2;
      s_red[16 + warp] = __longlong_as_double((long long)r64);
    }
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
      unsigned long long rr = 0;
      for (uint32_t i = 0; i < P.nw; ++i) {
        t = fmax(t, s_red[i]);
        rr += (unsigned long long)__double_as_longlong(s_red[16 + i]);
      }
      s_pub[1] = t;
      s_pub[2] = __longlong_as_double((long long)rr);
    }
    sync_all();
    double t = 0.0;
    unsigned long long rot = 0;
    for (unsigned r = 0; r < csize; ++r) {
      const double* pub = MULTI ? cluster.map_shared_rank(s_pub, r) : s_pub;
      t = fmax(t, pub[1]);
      rot += (unsigned long long)__double_as_longlong(pub[2]);
    }
    total_rot += rot;
    last_ratio = sqrt(t);
    ++sweep;
    const bool stagnant = sweep >= 4 && last_ratio < 1e-4 && last_ratio > 0.25 * prev_ratio;
    if (rot == 0 || last_ratio < P.stop_ratio || stagnant || sweep >= kSmemMaxSweeps) go = false;
#ifdef RK_SMEM_PROBE
    if (blockIdx.x == 0 && tid == 0)
      printf("[smem] sweep %d rot %llu ratio %.2e | G %u rows %u cl %u | cyc gram %lld ratio %lld rounds %lld xz %lld bar %lld | worked %lld skipped %lld\n",
             sweep, rot, last_ratio, G, rows, csize, pt[0], pt[1], pt[2], pt[3], pt[4], worked, skipped);
#endif
    prev_ratio = last_ratio;
    sync_all();  // everyone has read the published values before the next sweep overwrites them
  }
  // ---- write back (only the staged rows: the rest of the slot was and stays zero) ----
  for (uint32_t c = warp; c < my_cols; c += P.nw) {
    const uint32_t j = rank * Gc * kWG + c;
    if (j >= job.cols_pad) continue;
    double* wj = W + (uint64_t)j * job.rows;
    for (uint32_t i = lane; i < rows && i < job.rows; i += 32) wj[i] = mat[(uint64_t)c * ld + i];
  }
  if (rank == 0 && tid == 0) {
    job.stats[0] = (uint64_t)sweep;
    job.stats[1] = total_rot;
    job.stats[2] = 0ull;
    job.stats[3] = (uint64_t)__double_as_longlong(last_ratio);
    job.stats[4] = job.stats[5] = job.stats[6] = 0ull;
  }
}

// ===========================================================================
// Wide pair blocks (matrices too large for shared memory: c4's 1024^2, c5's 2048^2)
// ===========================================================================
// The 16-column warp steps above move 3 x 16 columns through L2/HBM for every
// 0.9 flop per byte: at 1024+ rows the batch streams from HBM and the kernel is
// bandwidth-bound. Here a CTA owns a pair of 32-column groups for one tournament
// step (one launch per step; the kernel boundary is the step's barrier):
//   1. H = X^T X (64 x 64, X = the pair's 64 columns) on the FP64 tensor cores: every
//      warp takes a slab of rows and the 36 upper 8 x 8 tiles (8 loads feed 36 DMMAs
//      per 4 rows), the slabs are added in warp order in shared memory;
//   2. the inner solve on H in shared memory: the 64 columns are 8 sub-groups of 8;
//      four warps run the sub-group pairs of an inner step (cross pairs A x B only,
//      all pairs in tournament step 0) with the 16-column rounds (step_rounds), then
//      H <- Z~^T H Z~ and Z <- Z Z~ by DMMA (columns, barrier, rows);
//   3. X <- X Z (Z 64 x 64) by DMMA, 128 DMMAs per 16 loads.
// 11 flop per byte of L2/HBM traffic instead of 0.9. Every cross pair of columns is
// rotated once per sweep, as in the narrower kernels; convergence is measured on the
// sub-blocks as they enter their rounds, and jacobi_cluster_kernel certifies on W.
constexpr int kWide = 64, kWideS = 65, kWideG = 32;  // pair-block columns, smem stride, columns per group

struct WideParams {
  const JacobiJob* jobs;
  uint32_t G;     // groups of kWideG columns (even)
  uint32_t step;  // tournament step
};

// per-job scratch in stats: [4] rotations of the sweep, [5] max ratio^2 bits, [6] alpha_max bits, [7] done
__global__ void __launch_bounds__(256) wide_sweep_begin(const JacobiJob* jobs) {
  const JacobiJob job = jobs[blockIdx.x];
  if (job.stats[7]) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __shared__ double red[8];
  double amax = 0.0;
  for (uint32_t j = warp; j < job.cols_pad; j += 8) {
    const double* wj = job.w + (uint64_t)j * job.rows;
    double a = 0.0;
    for (uint32_t i = lane; i < job.rows; i += 32) {
      const double x = __ldcg(wj + i);
      a += x * x;
    }
    amax = fmax(amax, warp_sum(a));
  }
  if (lane == 0) red[warp] = amax;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < 8; ++i) amax = fmax(amax, red[i]);
    job.stats[4] = 0ull;
    job.stats[5] = 0ull;
    job.stats[6] = (uint64_t)__double_as_longlong(amax);
  }
}

__global__ void wide_sweep_end(const JacobiJob* jobs, uint32_t njobs, double stop_ratio, int max_sweeps,
                               uint32_t* active, int debug) {
  const uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= njobs) return;
  const JacobiJob job = jobs[q];
  if (job.stats[7]) return;
  const unsigned long long rot = job.stats[4];
  const double ratio = sqrt(__longlong_as_double((long long)job.stats[5]));
  if (debug && q == 0) printf("[wide] job 0 sweep %d: rot %llu ratio %.3e\n", (int)job.stats[0] + 1, rot, ratio);
  job.stats[0] += 1ull;
  job.stats[1] += rot;
  job.stats[3] = (uint64_t)__double_as_longlong(ratio);
  if (rot == 0 || ratio < stop_ratio || (int)job.stats[0] >= max_sweeps) job.stats[7] = 1ull;
  else atomicAdd(active, 1u);
}

__global__ void wide_finish(const JacobiJob* jobs, uint32_t njobs) {
  const uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= njobs) return;
  const JacobiJob job = jobs[q];
  job.stats[2] = 0ull;
  job.stats[4] = job.stats[5] = job.stats[6] = job.stats[7] = 0ull;
}

// C (64 x 16 columns col_of(0..15) of S, stride kWideS) <- C Z16 (Z16 16 x 16 row-major, stride kWN)
template <typename F>
__device__ __forceinline__ void wide_cols_update(double* S, F col_of, const double* sZ) {
  const int lane = threadIdx.x & 31, lr = lane >> 2, lc = lane & 3;
  double bf[4][2];
#pragma unroll
  for (int kc = 0; kc < 4; ++kc)
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) bf[kc][nt] = sZ[(4 * kc + lc) * kWN + 8 * nt + lr];
  int cin[4], cout[2][2];
#pragma unroll
  for (int kc = 0; kc < 4; ++kc) cin[kc] = col_of(4 * kc + lc);
#pragma unroll
  for (int nt = 0; nt < 2; ++nt)
#pragma unroll
    for (int e = 0; e < 2; ++e) cout[nt][e] = col_of(8 * nt + 2 * lc + e);
#pragma unroll
  for (int rt = 0; rt < kWide / 8; ++rt) {
    const int r = 8 * rt + lr;
    double a[4];
#pragma unroll
    for (int kc = 0; kc < 4; ++kc) a[kc] = S[r * kWideS + cin[kc]];
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
      double d0 = 0.0, d1 = 0.0;
#pragma unroll
      for (int kc = 0; kc < 4; ++kc) dmma884(d0, d1, a[kc], bf[kc][nt]);
      S[r * kWideS + cout[nt][0]] = d0;
      S[r * kWideS + cout[nt][1]] = d1;
    }
    __syncwarp();  // the tile's reads precede its writes for every lane (a fragment spans the 16 columns)
  }
}

// R (16 rows row_of(0..15) x 64 of S) <- Z16^T R
template <typename F>
__device__ __forceinline__ void wide_rows_update(double* S, F row_of, const double* sZ) {
  const int lane = threadIdx.x & 31, lr = lane >> 2, lc = lane & 3;
  double af[2][4];  // A = Z16^T: A[8 mt + lr][4 kc + lc] = Z16[4 kc + lc][8 mt + lr]
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int kc = 0; kc < 4; ++kc) af[mt][kc] = sZ[(4 * kc + lc) * kWN + 8 * mt + lr];
  int rin[4], rout[2];
#pragma unroll
  for (int kc = 0; kc < 4; ++kc) rin[kc] = row_of(4 * kc + lc);
#pragma unroll
  for (int mt = 0; mt < 2; ++mt) rout[mt] = row_of(8 * mt + lr);
#pragma unroll
  for (int nt = 0; nt < kWide / 8; ++nt) {
    double b[4];
#pragma unroll
    for (int kc = 0; kc < 4; ++kc) b[kc] = S[rin[kc] * kWideS + 8 * nt + lr];
    double d[2][2];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
      d[mt][0] = d[mt][1] = 0.0;
#pragma unroll
      for (int kc = 0; kc < 4; ++kc) dmma884(d[mt][0], d[mt][1], af[mt][kc], b[kc]);
    }
    __syncwarp();
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
      S[rout[mt] * kWideS + 8 * nt + 2 * lc] = d[mt][0];
      S[rout[mt] * kWideS + 8 * nt + 2 * lc + 1] = d[mt][1];
    }
  }
  __syncwarp();
}

__global__ void __launch_bounds__(256, 2) jacobi_wide_step_kernel(WideParams P) {
  extern __shared__ __align__(16) double wsm[];
  const JacobiJob job = P.jobs[blockIdx.y];
  if (job.stats[7]) return;  // converged in an earlier sweep
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, lr = lane >> 2, lc = lane & 3;
  const uint32_t rows = job.rows, G = P.G, step = P.step, pw = blockIdx.x;
  double* H = wsm;                       // 64 x 65
  double* Z = H + kWide * kWideS;        // 64 x 65
  double* sHall = Z + kWide * kWideS;    // 4 x kSH (the inner solve's warps)
  __shared__ int s_any;
  __shared__ double s_red[8];
  __shared__ unsigned s_rot;
  const uint32_t gA = rr_slot(pw, step, G), gB = rr_slot(G - 1 - pw, step, G);
  double* XA = job.w + (uint64_t)gA * kWideG * rows;
  double* XB = job.w + (uint64_t)gB * kWideG * rows;
  const double freeze = kJacobiTol * kJacobiTol * __longlong_as_double((long long)job.stats[6]);
  if (tid == 0) {
    s_any = 0;
    s_rot = 0u;
  }
  for (int t = tid; t < kWide * kWideS; t += 256) Z[t] = ((t / kWideS) == (t % kWideS)) ? 1.0 : 0.0;

  // ---- 1. H = X^T X. The 36 upper 8 x 8 tiles in four sets -- the two diagonal 4 x 4
  // super-blocks (10 tiles each, 4 column tiles to load) and the two halves of the
  // off-diagonal one (8 tiles, 6 column tiles) -- times two halves of the rows: a
  // warp holds 10 accumulator tiles (not 36), so two CTAs share an SM ----
  {
    const int ts = warp & 3, rh = warp >> 2;
    const uint32_t slab = rows / 2, r_lo = rh * slab;
    auto tile_ptr = [&](int t) -> const double* {  // column 8 t + lr of the pair block
      return (t < 4 ? XA : XB) + (uint64_t)(8 * (t & 3) + lr) * rows + r_lo + lc;
    };
    auto put = [&](int i, int j, const double (&acc)[2]) {  // tile (i, j) and its mirror
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int r = 8 * i + lr, c = 8 * j + 2 * lc + e;
        const double v = (rh == 0 ? 0.0 : H[r * kWideS + c]) + acc[e];
        H[r * kWideS + c] = v;
        if (i != j) H[c * kWideS + r] = v;
      }
    };
    constexpr int kKBw = 4;  // k-steps whose loads are in flight together
    if (ts == 0 || ts == 3) {
      const int base = ts == 0 ? 0 : 4;
      const double* src[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) src[t] = tile_ptr(base + t);
      double acc[10][2];
#pragma unroll
      for (int i = 0; i < 10; ++i) acc[i][0] = acc[i][1] = 0.0;
      for (uint32_t k0 = 0; k0 < slab; k0 += 4 * kKBw) {
        double a[kKBw][4];
#pragma unroll
        for (int u = 0; u < kKBw; ++u)
#pragma unroll
          for (int t = 0; t < 4; ++t) a[u][t] = __ldcg(src[t] + k0 + 4 * u);
#pragma unroll
        for (int u = 0; u < kKBw; ++u) {
          int idx = 0;
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = i; j < 4; ++j) {
              dmma884(acc[idx][0], acc[idx][1], a[u][i], a[u][j]);
              ++idx;
            }
        }
      }
      for (int turn = 0; turn < 2; ++turn) {  // the row halves summed in order
        if (rh == turn) {
          int idx = 0;
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = i; j < 4; ++j) {
              put(base + i, base + j, acc[idx]);
              ++idx;
            }
        }
        __syncthreads();
      }
    } else {
      const int r0 = ts == 1 ? 0 : 2;
      const double* srcR[2];
      const double* srcC[4];
#pragma unroll
      for (int t = 0; t < 2; ++t) srcR[t] = tile_ptr(r0 + t);
#pragma unroll
      for (int t = 0; t < 4; ++t) srcC[t] = tile_ptr(4 + t);
      double acc[8][2];
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = 0.0;
      for (uint32_t k0 = 0; k0 < slab; k0 += 4 * kKBw) {
        double ar[kKBw][2], ac[kKBw][4];
#pragma unroll
        for (int u = 0; u < kKBw; ++u) {
#pragma unroll
          for (int t = 0; t < 2; ++t) ar[u][t] = __ldcg(srcR[t] + k0 + 4 * u);
#pragma unroll
          for (int t = 0; t < 4; ++t) ac[u][t] = __ldcg(srcC[t] + k0 + 4 * u);
        }
#pragma unroll
        for (int u = 0; u < kKBw; ++u)
#pragma unroll
          for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) dmma884(acc[4 * i + j][0], acc[4 * i + j][1], ar[u][i], ac[u][j]);
      }
      for (int turn = 0; turn < 2; ++turn) {
        if (rh == turn) {
#pragma unroll
          for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) put(r0 + i, 4 + j, acc[4 * i + j]);
        }
        __syncthreads();
      }
    }
  }

  // ---- 2. the inner solve: sub-groups 0..3 = group A, 4..7 = group B ----
  uint32_t nrot = 0;
  double best_g2 = 0.0, best_prod = 1.0;
  const int n_inner = step == 0 ? 7 : 4;
  for (int it = 0; it < n_inner; ++it) {
    bool need = false;
    int sa = 0, sb = 0;
    double* sH = sHall + (warp & 3) * kSH;
    if (warp < 4) {
      if (step == 0) {
        sa = (int)rr_slot((uint32_t)warp, (uint32_t)it, 8u);
        sb = (int)rr_slot((uint32_t)(7 - warp), (uint32_t)it, 8u);
      } else {
        sa = warp;
        sb = 4 + ((warp + it) & 3);
      }
      // the pair's 16 x 16 block of H
      for (int t = lane; t < kWN * kWN; t += 32) {
        const int r = t >> 4, c = t & 15;
        const int mr = r < 8 ? 8 * sa + r : 8 * sb + r - 8, mc = c < 8 ? 8 * sa + c : 8 * sb + c - 8;
        sH[r * kWS + c] = H[mr * kWideS + mc];
      }
      __syncwarp();
      const bool intra = step == 0 && it == 0;
      need = fresh_scan(sH, freeze, intra, best_g2, best_prod);
      if (need) {
        step_rounds(sH, intra, freeze, nrot);
        auto idx_of = [&](int t) { return t < 8 ? 8 * sa + t : 8 * sb + t - 8; };
        wide_cols_update(H, idx_of, sH);
        wide_cols_update(Z, idx_of, sH);
        if (lane == 0) s_any = 1;
      }
    }
    __syncthreads();
    if (warp < 4 && need) {
      auto idx_of = [&](int t) { return t < 8 ? 8 * sa + t : 8 * sb + t - 8; };
      wide_rows_update(H, idx_of, sH);
    }
    __syncthreads();
  }
  // the step's statistics
  {
    unsigned r32 = nrot;
    double r2 = best_g2 / best_prod;
    for (int o = 16; o; o >>= 1) {
      r32 += __shfl_xor_sync(0xffffffffu, r32, o);
      r2 = fmax(r2, __shfl_xor_sync(0xffffffffu, r2, o));
    }
    if (lane == 0) {
      s_red[warp] = r2;
      if (r32) atomicAdd(&s_rot, r32);
    }
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
      for (int i = 0; i < 4; ++i) t = fmax(t, s_red[i]);
      if (s_rot) atomicAdd(reinterpret_cast<unsigned long long*>(job.stats + 4), (unsigned long long)s_rot);
      atomicMax(reinterpret_cast<unsigned long long*>(job.stats + 5), (unsigned long long)__double_as_longlong(t));
    }
  }
  if (!s_any) return;  // nothing rotated: Z = I

  // ---- 3. X <- X Z: this warp's slab, 16 rows at a time ----
  {
    const uint32_t slab = rows / 8, r_lo = warp * slab;
    const uint64_t cs4 = (uint64_t)4 * rows;  // four columns on
    const double* inA = XA + (uint64_t)lc * rows + r_lo + lr;  // column 4 kc + lc, kc < 8: group A
    const double* inB = XB + (uint64_t)lc * rows + r_lo + lr;
    for (uint32_t r0 = 0; r0 < slab; r0 += 16) {
      double a[2][16];
#pragma unroll
      for (int u = 0; u < 2; ++u)
#pragma unroll
        for (int kc = 0; kc < 16; ++kc) a[u][kc] = __ldcg((kc < 8 ? inA : inB) + (uint64_t)(kc & 7) * cs4 + r0 + 8 * u);
#pragma unroll
      for (int nt = 0; nt < 8; ++nt) {
        double d[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
        for (int kc = 0; kc < 16; ++kc) {
          const double b = Z[(4 * kc + lc) * kWideS + 8 * nt + lr];
          dmma884(d[0][0], d[0][1], a[0][kc], b);
          dmma884(d[1][0], d[1][1], a[1][kc], b);
        }
        double* o0 = (nt < 4 ? XA : XB) + (uint64_t)(8 * (nt & 3) + 2 * lc) * rows + r_lo + r0 + lr;
        double* o1 = o0 + rows;
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          o0[8 * u] = d[u][0];
          o1[8 * u] = d[u][1];
        }
      }
    }
  }
}

// ===========================================================================
// finalize
// ===========================================================================

constexpr int kFThreads = 1024;
// finalize_kernel leaves the output columns' flags in the high bits of order[j]
constexpr uint32_t kOrderFlip = 0x80000000u, kOrderDef = 0x40000000u, kOrderSrc = 0x3fffffffu;

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
  __syncthreads();  // order[] gets its flag bits below
  for (uint32_t j = warp; j < J.k; j += nw) {
    const uint32_t src = J.order[j];
    const double s = sig[src];
    const bool deficient = !(s > thr && s > 0.0);
    const double* wj = J.w + (uint64_t)src * rows;
    // sign convention on u = w / s: first index of the largest |u|
    double best = -1.0;
    uint32_t arg = 0;
    if (!deficient) {
      // the first index (in the ORIGINAL row order) of the largest |u|
      const uint32_t* rp = J.row_perm;
      uint32_t argo = 0xffffffffu;
      for (uint32_t i = lane; i < rows; i += 32) {
        const double mag = fabs(wj[i] / s);
        const uint32_t io = rp ? rp[i] : i;
        if (mag > best || (mag == best && io < argo)) { best = mag; arg = i; argo = io; }
      }
      for (int o = 16; o; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const uint32_t oa = __shfl_xor_sync(0xffffffffu, arg, o);
        const uint32_t oo = __shfl_xor_sync(0xffffffffu, argo, o);
        if (ob > best || (ob == best && oo < argo)) { best = ob; arg = oa; argo = oo; }
      }
    }
    const bool flip = !deficient && (wj[arg] / s) < 0.0;
    if (lane == 0) {
      if (J.sigma) J.sigma[j] = s;
      if (J.deficient) J.deficient[j] = deficient ? 1 : 0;
      J.order[j] = src | (flip ? kOrderFlip : 0u) | (deficient ? kOrderDef : 0u);
    }
  }
}

// u / payload / v_out of output columns [32 bx, 32 bx + 32) and rows
// [32 by, 32 by + 32): a 32 x 32 tile read along W's columns (coalesced), written
// along the row-major outputs (coalesced) through shared memory. Same arithmetic
// as the reference: u = flip * (w / s), payload = u * s.
__global__ void __launch_bounds__(256) finalize_write_kernel(const FinalJob* jobs) {
  const FinalJob J = jobs[blockIdx.z];
  __shared__ double tile[32][33];
  __shared__ uint32_t s_src[32];
  __shared__ double s_sig[32];
  const uint32_t j0 = blockIdx.x * 32, i0 = blockIdx.y * 32;
  if (j0 >= J.k) return;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 8 warps
  if (threadIdx.x < 32) {
    const uint32_t j = j0 + tx;
    const uint32_t o = j < J.k ? J.order[j] : 0u;
    s_src[tx] = o;
    s_sig[tx] = j < J.k ? J.scratch[o & kOrderSrc] : 0.0;
  }
  __syncthreads();
  // a tile whose 32 columns all have sigma = 0 (deficient: u = 0, payload = 0): zeros out, no read of W
  // (c3: ~370 of every block's 512 columns)
  if (!J.v_out && __syncthreads_and(s_sig[tx] == 0.0 && ((s_src[tx] & kOrderDef) != 0u || j0 + tx >= J.k))) {
    for (int r = ty; r < 32; r += 8) {
      const uint32_t i = i0 + r, j = j0 + tx;
      if (i < J.rows && j < J.k) {
        if (J.u) J.u[(uint64_t)i * J.k + j] = 0.0;
        if (J.payload) J.payload[(uint64_t)i * J.k + j] = 0.0;
      }
    }
    return;
  }
  auto pass = [&](const double* src_base, uint64_t ld, uint32_t nrows, double* out_u, double* out_p, bool is_v) {
    if (i0 >= nrows) return;
    for (int c = ty; c < 32; c += 8) {
      const uint32_t j = j0 + c, i = i0 + tx;
      double x = 0.0;
      if (j < J.k && i < nrows) x = src_base[(uint64_t)(s_src[c] & kOrderSrc) * ld + i];
      tile[c][tx] = x;
    }
    __syncthreads();
    for (int r = ty; r < 32; r += 8) {
      const uint32_t i = i0 + r, j = j0 + tx;
      if (i < nrows && j < J.k) {
        const uint32_t io = (!is_v && J.row_perm) ? J.row_perm[i] : i;  // output row
        const uint32_t o = s_src[tx];
        const double s = s_sig[tx], w = tile[tx][r];
        const bool def = (o & kOrderDef) != 0u, flip = (o & kOrderFlip) != 0u;
        if (is_v) {
          out_u[(uint64_t)i * J.k + j] = flip ? -w : w;
        } else {
          const double u = def ? 0.0 : (flip ? -(w / s) : (w / s));
          if (out_u) out_u[(uint64_t)io * J.k + j] = u;
          if (out_p) out_p[(uint64_t)io * J.k + j] = def ? (s > 0.0 ? w : 0.0) : u * s;
        }
      }
    }
    __syncthreads();
  };
  if (J.u || J.payload) pass(J.w, J.rows, J.rows, J.u, J.payload, false);
  if (J.v_out) pass(J.v_in, J.ldv, J.cols, J.v_out, nullptr, true);
}

// ===========================================================================
// orthonormal completion (one CTA, deterministic) -- svd.cpp:150-201
// u is row-major rows x cols
// ===========================================================================

// One CTA. Same candidate rule as the reference (e_0, e_1, ... ; the first whose
// residual after two orthogonalization passes against the placed columns exceeds
// 0.5, else the best one, then one touch-up pass) with two changes that keep the
// choice: the passes are classical Gram-Schmidt over the whole CTA (projections
// of w onto all placed columns at once, twice -- CGS2 -- instead of the
// reference's column-by-column MGS; the completion basis of an exactly
// degenerate cluster is not unique anyway), and the scan resumes after the
// leading candidates already known to be dead -- rejected with a clear margin
// (residual < 0.5 - 1e-6) or taken -- for an earlier column: the placed span only
// grows, so their residual can only shrink and the reference would reject them
// again. This removes the O(deficient^2) rescans that made rank-deficient
// 512-row blocks take minutes. If no candidate passes, the dead ones are scanned
// too (the reference's best-residual fallback over all candidates).
constexpr int kCThreads = 1024;

__device__ double block_sum(double x, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  x = warp_sum(x);
  __syncthreads();
  if (lane == 0) red[warp] = x;
  __syncthreads();
  double t = 0.0;
  for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += red[i];
  return t;
}

__global__ void __launch_bounds__(kCThreads) complete_kernel(double* u, uint32_t rows, uint32_t cols,
                                                             const uint8_t* deficient, int* fail) {
  extern __shared__ double cw[];
  double* w = cw;
  double* best = cw + rows;
  double* proj = best + rows;
  __shared__ double red[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  uint32_t start = 0;
  // w <- (I - U_p U_p^T)^2 e_cand over the placed columns p (not deficient, or < j)
  auto orth_candidate = [&](uint32_t cand, uint32_t j) -> double {
    for (uint32_t i = tid; i < rows; i += blockDim.x) w[i] = (i == cand) ? 1.0 : 0.0;
    __syncthreads();
    for (int pass = 0; pass < 2; ++pass) {
      for (uint32_t c = tid; c < cols; c += blockDim.x) {
        double acc = 0.0;
        if (!deficient[c] || c < j)
          for (uint32_t i = 0; i < rows; ++i) acc += u[(uint64_t)i * cols + c] * w[i];
        proj[c] = acc;
      }
      __syncthreads();
      for (uint32_t i = warp; i < rows; i += nw) {
        double acc = 0.0;
        for (uint32_t c = lane; c < cols; c += 32) acc += u[(uint64_t)i * cols + c] * proj[c];
        acc = warp_sum(acc);
        if (lane == 0) w[i] -= acc;
      }
      __syncthreads();
    }
    double nn = 0.0;
    for (uint32_t i = tid; i < rows; i += blockDim.x) nn += w[i] * w[i];
    return sqrt(block_sum(nn, red));
  };
  for (uint32_t j = 0; j < cols; ++j) {
    if (!deficient[j]) continue;
    double best_norm = -1.0;
    bool found = false, leading = true;
    uint32_t next_start = start;
    for (int phase = 0; phase < 2 && !found; ++phase) {
      const uint32_t c0 = phase == 0 ? start : 0, c1 = phase == 0 ? rows : start;
      for (uint32_t cand = c0; cand < c1; ++cand) {
        const double wn = orth_candidate(cand, j);
        const bool take = wn > 0.5;
        if (take || wn > best_norm) {
          best_norm = wn;
          for (uint32_t i = tid; i < rows; i += blockDim.x) best[i] = w[i];
        }
        if (phase == 0 && leading) {
          if (take || wn < 0.5 - 1e-6) next_start = cand + 1;
          else leading = false;
        }
        __syncthreads();
        if (take) {
          found = true;
          break;
        }
      }
    }
    start = next_start;
    if (!(best_norm > 0.0)) {
      // no independent direction (svd.cpp:183-186)
      if (tid == 0) *fail = 1;
      return;
    }
    for (uint32_t i = tid; i < rows; i += blockDim.x) u[(uint64_t)i * cols + j] = best[i] / best_norm;
    __syncthreads();
    if (best_norm <= 0.5) {
      for (uint32_t i = tid; i < rows; i += blockDim.x) w[i] = u[(uint64_t)i * cols + j];
      __syncthreads();
      for (uint32_t c = tid; c < cols; c += blockDim.x) {
        double acc = 0.0;
        if (!deficient[c] || c < j)
          for (uint32_t i = 0; i < rows; ++i) acc += u[(uint64_t)i * cols + c] * w[i];
        proj[c] = acc;
      }
      __syncthreads();
      for (uint32_t i = warp; i < rows; i += nw) {
        double acc = 0.0;
        for (uint32_t c = lane; c < cols; c += 32) acc += u[(uint64_t)i * cols + c] * proj[c];
        acc = warp_sum(acc);
        if (lane == 0) w[i] -= acc;
      }
      __syncthreads();
      double nn = 0.0;
      for (uint32_t i = tid; i < rows; i += blockDim.x) nn += w[i] * w[i];
      const double wn = sqrt(block_sum(nn, red));
      for (uint32_t i = tid; i < rows; i += blockDim.x) u[(uint64_t)i * cols + j] = w[i] / wn;
      __syncthreads();
    }
  }
}

// ===========================================================================
// apply_q: out(:, c) = H_0 ... H_{K-1} [x(:, c); 0] -- warp per column
// ===========================================================================

__device__ void apply_q_body(const QrJob& qr, const double* x, uint32_t x_rows, uint32_t ncols, double* out);

__global__ void apply_q_kernel(QrJob qr, const double* x, uint32_t x_rows, uint32_t ncols, double* out) {
  apply_q_body(qr, x, x_rows, ncols, out);
}

// one job per blockIdx.y (the wide blocks' reduced route: slot = Q [R V; 0])
__global__ void apply_q_batched_kernel(const ApplyQJob* jobs) {
  const ApplyQJob j = jobs[blockIdx.y];
  apply_q_body(j.qr, j.x, j.x_rows, j.ncols, j.out);
}

// The same product with the columns in registers: a warp owns CW columns of one job
// (element i of a column in lane i % 32, slot i / 32), so each reflector is read once
// per CW columns and the CW dot products reduce side by side. For m <= 32 E.
template <int CW, int E>
__global__ void __launch_bounds__(256) apply_q_regs_kernel(const ApplyQJob* jobs) {
  const ApplyQJob j = jobs[blockIdx.y];
  const int lane = threadIdx.x & 31;
  const uint32_t m = j.qr.m, K = j.qr.m < j.qr.n ? j.qr.m : j.qr.n;
  const uint32_t w0 = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t c0 = w0 * CW; c0 < j.ncols; c0 += nw * CW) {
    double o[CW][E];
#pragma unroll
    for (int cw = 0; cw < CW; ++cw)
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const uint32_t i = lane + 32 * e, c = c0 + cw;
        o[cw][e] = (c < j.ncols && i < j.x_rows) ? j.x[(uint64_t)c * j.x_rows + i] : 0.0;
      }
    for (int kk = (int)K - 1; kk >= 0; --kk) {
      const double beta = j.qr.beta[kk];
      if (beta == 0.0) continue;
      const double* __restrict__ v = j.qr.a + (uint64_t)kk * j.qr.lda;  // v0 on the diagonal, then below
      double vv[E];
      double d[CW];
#pragma unroll
      for (int cw = 0; cw < CW; ++cw) d[cw] = 0.0;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const uint32_t i = lane + 32 * e;
        vv[e] = (i >= (uint32_t)kk && i < m) ? __ldg(v + i) : 0.0;
#pragma unroll
        for (int cw = 0; cw < CW; ++cw) d[cw] = fma(vv[e], o[cw][e], d[cw]);
      }
#pragma unroll
      for (int off = 16; off; off >>= 1)
#pragma unroll
        for (int cw = 0; cw < CW; ++cw) d[cw] += __shfl_xor_sync(0xffffffffu, d[cw], off);
#pragma unroll
      for (int cw = 0; cw < CW; ++cw) {
        const double bw = beta * d[cw];
#pragma unroll
        for (int e = 0; e < E; ++e) o[cw][e] = fma(-bw, vv[e], o[cw][e]);
      }
    }
#pragma unroll
    for (int cw = 0; cw < CW; ++cw)
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const uint32_t i = lane + 32 * e, c = c0 + cw;
        if (c < j.ncols && i < m) j.out[(uint64_t)c * m + i] = o[cw][e];
      }
  }
}

// a warp per output column: the reflectors applied last to first (svd.cpp:111-132)
__device__ void apply_q_body(const QrJob& qr, const double* x, uint32_t x_rows, uint32_t ncols, double* out) {
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

}  // namespace

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
  // largest even group size (<= gcap) whose two staged groups fit the budget; a
  // smaller cap trades longer tournaments for more CTAs per SM (latency hiding)
  const uint32_t gcap = (uint32_t)tuning().jacobi_gmax;
  // columns longer than 16 lanes x 32 registers: 8 groups of 32 lanes keep the A
  // column in registers (E <= 32); without the cap the plan falls back to the
  // shared-memory rounds (E = 0), several times slower
  const uint32_t gtop = (rows > 16 * 32 && rows <= 32 * 32 && !with_v) ? std::min<uint32_t>(gcap, 8) : gcap;
  // long columns run the Gram-assisted warp kernel first (groups of 8), which needs
  // a width divisible by 16: prefer such plans (pass 0), else any (pass 1)
  const bool want16 = rows >= 512 && !with_v;
  for (int pass = want16 ? 0 : 1; pass < 2; ++pass)
    for (uint32_t gmax = gtop; gmax >= 2; gmax -= 2) {
      G = (uint32_t)ceil_div(cols ? cols : 1, gmax);
      if (G < 2) G = 2;
      if (G & 1) ++G;
      g = (uint32_t)ceil_div(cols ? cols : 1, G);
      if (g & 1) ++g;
      if (g < 2) g = 2;
      if (pass == 0 && (g * G) % 16 != 0) continue;
      if (jacobi_smem(rows, g, g * G, with_v) <= smem_budget) return;
    }
  fail(RK_INVALID_ARGUMENT, "Jacobi: a " + std::to_string(rows) + "-row matrix does not fit shared memory");
}

size_t jacobi_smem(uint32_t rows, uint32_t g, uint32_t cols_pad, bool with_v) {
  return (size_t)2 * g * (rows + 8) * 8 + (with_v ? (size_t)2 * g * (cols_pad + 8) * 8 : 0) + (size_t)2 * g * 8;
}
// The shared-memory Jacobi over a batch: every job gets the smallest cluster whose
// shared memory holds its staged matrix (a function of the job's own shape), jobs
// of one cluster size share a launch. false (nothing launched): a job does not fit.
static bool jacobi_smem_batched(const std::vector<JacobiJob>& jobs, const JacobiJob* d_jobs, cudaStream_t s,
                                size_t smem_optin, double stop_ratio, const SideStream* side) {
  struct Shape { uint32_t cl, cap_cols, nw, rows; };
  auto shape_of = [&](const JacobiJob& j, Shape& sh) {
    const uint32_t colsU = (j.cols + 15u) & ~15u, G = colsU / kWG, npairs = G / 2;
    const uint32_t rows = (std::min(j.rows, j.rows_nz ? j.rows_nz : j.rows) + 7u) & ~7u;
    // clusters of more than two CTAs lose to the direct kernel (measured on c2's 256 x 256: 11.5 vs 6.1 ms)
    const uint32_t cl_max = (uint32_t)std::max(1, std::min(8, tuning().jacobi_smem_cl));
    for (uint32_t cl = 1; cl <= cl_max; cl *= 2) {
      const uint32_t Gc = (uint32_t)ceil_div(G, cl), nw = (uint32_t)ceil_div(npairs, cl);
      const size_t bytes = ((size_t)Gc * kWG * (rows + 4) + (size_t)nw * kSH + kSmemMisc) * sizeof(double);
      if (nw <= (uint32_t)kSmemMaxWarps && bytes <= smem_optin) {
        sh = {cl, Gc * kWG, std::max(nw, 1u), rows};
        return true;
      }
    }
    return false;
  };
  // contiguous runs of one cluster size (a launch addresses jobs by blockIdx)
  std::vector<Shape> shapes(jobs.size());
  for (size_t i = 0; i < jobs.size(); ++i)
    if (!shape_of(jobs[i], shapes[i])) return false;
  bool forked = false;
  // the groups' carried diagonal blocks: (columns / 8) x 64 doubles per job, allocated before any
  // launch is forked to the side stream and freed in stream order after the join
  uint64_t keep_stride = 0;
  for (const Shape& sh : shapes) keep_stride = std::max<uint64_t>(keep_stride, (uint64_t)sh.cap_cols * sh.cl * kWG);
  DBuf<double> keep_all;
  if (tuning().jacobi_carry) keep_all.alloc(jobs.size() * keep_stride, s);
  for (size_t i0 = 0; i0 < jobs.size();) {
    size_t i1 = i0;
    Shape m = shapes[i0];
    while (i1 < jobs.size() && shapes[i1].cl == m.cl) {
      m.cap_cols = std::max(m.cap_cols, shapes[i1].cap_cols);
      m.nw = std::max(m.nw, shapes[i1].nw);
      m.rows = std::max(m.rows, shapes[i1].rows);
      ++i1;
    }
    // the widest and the tallest job of a run may differ: the layout must still fit
    size_t bytes = ((size_t)m.cap_cols * (m.rows + 4) + (size_t)m.nw * kSH + kSmemMisc) * sizeof(double);
    while (bytes > smem_optin && i1 > i0 + 1) {  // shorten the run until its envelope fits
      --i1;
      m = shapes[i0];
      for (size_t i = i0; i < i1; ++i) {
        m.cap_cols = std::max(m.cap_cols, shapes[i].cap_cols);
        m.nw = std::max(m.nw, shapes[i].nw);
        m.rows = std::max(m.rows, shapes[i].rows);
      }
      bytes = ((size_t)m.cap_cols * (m.rows + 4) + (size_t)m.nw * kSH + kSmemMisc) * sizeof(double);
    }
    const unsigned n = (unsigned)(i1 - i0);
    double* keep = keep_all.get() ? keep_all.get() + (uint64_t)i0 * keep_stride : nullptr;
    SmemParams P{d_jobs + i0, m.rows + 4, m.cap_cols, m.nw, stop_ratio, keep, keep_stride};
    // runs are independent (disjoint jobs): every run but the last goes to the side
    // stream, so a short run of clustered jobs shares the device with the main run
    const bool aside = side && side->stream && i1 < jobs.size();
    cudaStream_t ls = aside ? side->stream : s;
    if (aside && !forked) {
      RK_CUDA_CHECK(cudaEventRecord(side->fork, s));
      RK_CUDA_CHECK(cudaStreamWaitEvent(side->stream, side->fork, 0));
      forked = true;
    }
    if (m.cl == 1) {
      RK_CUDA_CHECK(cudaFuncSetAttribute(jacobi_smem_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
      jacobi_smem_kernel<false><<<n, m.nw * 32, bytes, ls>>>(P);
      RK_LAUNCH_CHECK();
    } else {
      void* args[] = {&P};
      RK_CUDA_CHECK(cudaFuncSetAttribute(jacobi_smem_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
      launch_cluster_kernel((const void*)jacobi_smem_kernel<true>, n * m.cl, m.cl, m.nw * 32, bytes, ls, args);
    }
    i0 = i1;
  }
  if (forked) {
    RK_CUDA_CHECK(cudaEventRecord(side->join, side->stream));
    RK_CUDA_CHECK(cudaStreamWaitEvent(s, side->join, 0));
  }
  return true;
}

// The wide pair-block kernel over a homogeneous batch (one launch per tournament
// step; the host reads the number of unconverged jobs once per sweep).
static bool jacobi_wide_batched(const std::vector<JacobiJob>& jobs, const JacobiJob* d_jobs, cudaStream_t s,
                                double stop_ratio) {
  const uint32_t rows = jobs[0].rows, cols_pad = jobs[0].cols_pad;
  if (rows % 128 != 0 || cols_pad % (2 * kWideG) != 0 || cols_pad < 4 * kWideG) return false;  // slabs of 16-row batches
  const uint32_t G = cols_pad / kWideG, njobs = (uint32_t)jobs.size();
  const size_t smem = ((size_t)2 * kWide * kWideS + 4 * kSH) * sizeof(double);
  RK_CUDA_CHECK(cudaFuncSetAttribute(jacobi_wide_step_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  DBuf<uint32_t> active(1, s);
  constexpr int kWideMaxSweeps = 30;
  for (int sweep = 0; sweep < kWideMaxSweeps; ++sweep) {
    wide_sweep_begin<<<njobs, 256, 0, s>>>(d_jobs);
    RK_LAUNCH_CHECK();
    for (uint32_t step = 0; step + 1 < G; ++step) {
      WideParams P{d_jobs, G, step};
      jacobi_wide_step_kernel<<<dim3(G / 2, njobs), 256, smem, s>>>(P);
      RK_LAUNCH_CHECK();
    }
    active.zero();
    wide_sweep_end<<<(unsigned)ceil_div(njobs, 256), 256, 0, s>>>(d_jobs, njobs, stop_ratio, kWideMaxSweeps, active.get(),
                                                                      tuning().jacobi_debug ? 1 : 0);
    RK_LAUNCH_CHECK();
    std::vector<uint32_t> h;
    to_host(h, active.get(), 1, s);
    sync(s);
    if (h[0] == 0) break;
  }
  wide_finish<<<(unsigned)ceil_div(njobs, 256), 256, 0, s>>>(d_jobs, njobs);
  RK_LAUNCH_CHECK();
  return true;
}

bool jacobi_smem_try(std::vector<JacobiJob>& jobs, cudaStream_t s, size_t smem_optin, const SideStream* side) {
  const Tuning& tn = tuning();
  if (jobs.empty() || tn.jacobi_smem == 0) return false;
  for (const JacobiJob& j : jobs)
    if (j.v || j.pre) return false;
  // largest first: runs of one cluster size are contiguous, and the longest jobs of
  // a launch start first (the last wave is the short ones)
  std::stable_sort(jobs.begin(), jobs.end(), [](const JacobiJob& a, const JacobiJob& b) {
    return std::max(a.cols, 1u) * (uint64_t)(a.rows_nz ? a.rows_nz : a.rows) >
           std::max(b.cols, 1u) * (uint64_t)(b.rows_nz ? b.rows_nz : b.rows);
  });
  DBuf<JacobiJob> dj(jobs.size(), s);
  to_device(dj.get(), jobs.data(), jobs.size(), s);
  if (!jacobi_smem_batched(jobs, dj.get(), s, smem_optin, tn.jacobi_check >= 0 ? tn.jacobi_check : 1e-7, side)) return false;
  for (JacobiJob& j : jobs) j.pre = 1;
  return true;
}

bool jacobi_smem_fits(const JacobiJob& j, size_t smem_optin) {
  if (j.v || tuning().jacobi_smem == 0) return false;
  const uint32_t colsU = (j.cols + 15u) & ~15u, G = colsU / kWG, npairs = G / 2;
  const uint32_t rows = (std::min(j.rows, j.rows_nz ? j.rows_nz : j.rows) + 7u) & ~7u;
  const uint32_t cl_max = (uint32_t)std::max(1, std::min(8, tuning().jacobi_smem_cl));
  for (uint32_t cl = 1; cl <= cl_max; cl *= 2) {
    const uint32_t Gc = (uint32_t)ceil_div(G, cl), nw = (uint32_t)ceil_div(npairs, cl);
    const size_t bytes = ((size_t)Gc * kWG * (rows + 4) + (size_t)nw * kSH + kSmemMisc) * sizeof(double);
    if (nw <= (uint32_t)kSmemMaxWarps && bytes <= smem_optin) return true;
  }
  return false;
}

void jacobi_batched(std::vector<JacobiJob>& jobs, cudaStream_t s, int sms, size_t smem_optin, bool latency) {
  if (jobs.empty()) return;
  // jobs in one launch share rows / cols_pad / with_v (the caller groups them);
  // the group layout is a function of (rows, cols_pad) only
  const uint32_t rows = jobs[0].rows, cols_pad = jobs[0].cols_pad;
  const bool with_v = jobs[0].v != nullptr;
  uint32_t g, G;
  const size_t budget = std::min<size_t>(smem_optin, 200 * 1024);
  jacobi_plan(rows, cols_pad, with_v, budget, g, G);
  // a single latency-critical matrix (the merge): smaller groups, 32 lanes per
  // pair (shorter dot and update chains per round), up to 16 CTAs per matrix
  unsigned max_cluster = 8;
  if (latency && jobs.size() == 1 && !with_v) {
    const uint32_t g1 = (uint32_t)tuning().jacobi_single_g;
    if (g1 >= 2 && g1 % 2 == 0 && g1 < g && cols_pad % g1 == 0 && (cols_pad / g1) % 2 == 0 && rows <= 32u * 32u) {
      g = g1;
      G = cols_pad / g1;
      max_cluster = 16;
    }
  }
  for (JacobiJob& j : jobs) {
    if (j.rows != rows || j.cols_pad != cols_pad || (j.v != nullptr) != with_v)
      fail(RK_RUNTIME, "jacobi_batched: heterogeneous batch");
    if (j.cols > cols_pad) fail(RK_RUNTIME, "jacobi_batched: cols > cols_pad");
  }
  if (g * G != cols_pad) fail(RK_RUNTIME, "jacobi_batched: cols_pad is not a planned width");
  // Gram-route matrices: Gram-assisted warp Jacobi, then the direct kernel
  // certifies convergence on W (check_first)
  // Where it pays (measured): long columns in a batch -- c4's 1024 blocks of 1024
  // rows: 7.5 s vs 12.2 s for the direct kernel. At 256 rows it ties on c2's 64
  // blocks (7.30 vs 7.23 ms) and is 2x slower on a single matrix (the L2 latency of
  // streaming X twice per step is not hidden at 8 warps per SM). RK_JACOBI_WARP=0/1
  // forces it off/on.
  const Tuning& tn = tuning();
  const bool warp_default = rows >= 512 && !latency;  // a function of the shape only (see latency)
  bool use_warp = (tn.jacobi_warp >= 0 ? tn.jacobi_warp == 1 : warp_default) && !with_v && cols_pad % 16 == 0;
  // matrices that fit shared memory: the resident Gram-assisted kernel first (any
  // conditioning: it measures convergence on fresh Grams and the direct kernel
  // certifies) -- here, or already run by the caller over a larger batch (pre)
  bool all_pre = true, any_pre = false;
  for (const JacobiJob& j : jobs) {
    all_pre = all_pre && j.pre;
    any_pre = any_pre || j.pre;
  }
  if (any_pre && !all_pre) {  // the caller's shared-memory pass took only the jobs that fit: finish the two sets apart
    std::vector<JacobiJob> done, rest;
    for (const JacobiJob& j : jobs) (j.pre ? done : rest).push_back(j);
    jacobi_batched(done, s, sms, smem_optin, latency);
    jacobi_batched(rest, s, sms, smem_optin, latency);
    return;
  }
  bool use_smem = all_pre || (!latency && jacobi_smem_try(jobs, s, smem_optin, nullptr));
  if (use_smem) use_warp = false;
  // large matrices: the wide pair-block kernel (RK_JACOBI_WIDE=0: the 16-column warp kernel)
  bool use_wide = false;
  if ((use_warp || (latency && tn.jacobi_warp != 0)) && !use_smem && !with_v && tn.jacobi_wide && rows >= 1024) {
    DBuf<JacobiJob> djw(jobs.size(), s);
    to_device(djw.get(), jobs.data(), jobs.size(), s);
    use_wide = jacobi_wide_batched(jobs, djw.get(), s, tn.jacobi_check >= 0 ? tn.jacobi_check : 1e-7);
  }
  if (use_wide) use_warp = true;  // the direct kernel starts with the certifying check
  else if (use_warp) {
    WarpParams WP{nullptr, cols_pad / kWG, tn.jacobi_check >= 0 ? tn.jacobi_check : 1e-7};
    DBuf<JacobiJob> djw(jobs.size(), s);
    to_device(djw.get(), jobs.data(), jobs.size(), s);
    WP.jobs = djw.get();
    void* wargs[] = {&WP};
    const unsigned wcl = (unsigned)std::min<uint64_t>(8, ceil_div(cols_pad / 16, kJWarps));
    RK_CUDA_CHECK(cudaFuncSetAttribute(jacobi_warp_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    launch_cluster_kernel((const void*)jacobi_warp_kernel, (unsigned)jobs.size() * wcl, wcl, kJThreads, 0, s, wargs);
  }
  const size_t smem = jacobi_smem(rows, g, g * G, with_v);
  // cluster size: enough CTAs for the SMs at the occupancy the shared memory allows
  const unsigned per_sm = (unsigned)std::max<size_t>(1, std::min<size_t>(8, (228 * 1024) / (smem + 2048)));
  unsigned cl = (unsigned)std::max<uint64_t>(1, (uint64_t)sms * per_sm / jobs.size());
  cl = std::min<unsigned>({cl, G / 2, max_cluster});
  unsigned p2 = 1;
  while (p2 * 2 <= cl) p2 *= 2;
  cl = p2;
  if (tn.jacobi_cluster) {  // tuning override
    const unsigned v = (unsigned)tn.jacobi_cluster;
    if (v >= 1 && v <= 16 && v <= G / 2) cl = v;
  }
  DBuf<JacobiJob> dj(jobs.size(), s);
  to_device(dj.get(), jobs.data(), jobs.size(), s);
  // the convergence check (tail_check) takes over once a sweep's max ratio is
  // below check_ratio. Measured on c2: batched blocks 6.41 ms at 1e-7, 6.07 ms
  // anywhere in 3e-6 .. 1e-4 (one full sweep fewer; a check that finds too many
  // violators costs less than the sweep it replaces); the single latency-bound
  // merge is best at 1e-7 (1.71 vs 1.76 ms). A check certifies with the
  // reference's rule whatever the threshold.
  const double check_default = latency ? 1e-7 : 1e-5;
  JacobiParams P{dj.get(), g, G, with_v ? 1 : 0, tn.jacobi_check >= 0 ? tn.jacobi_check : check_default,
                 (use_warp || use_smem) ? 1 : 0, tn.jacobi_debug ? 1 : 0};
  void* kargs[] = {&P};
  // lanes per pair: enough lane groups for the g pairs of a round; E = column
  // elements per lane held in registers by the cross rounds (0: shared-memory path)
  int Q = 32;
  while (Q > 8 && (kJThreads / Q) < (int)g) Q /= 2;
  if (tn.jacobi_q) {  // tuning override (must give >= g lane groups)
    const int qv = tn.jacobi_q;
    if ((qv == 8 || qv == 16 || qv == 32) && kJThreads / qv >= (int)g) Q = qv;
  }
  int E = 1;
  while (E * Q < (int)rows) E *= 2;
  if (E < 4) E = 4;
  if (E > 32 || with_v) E = 0;  // a[E] + b[E] must stay in registers
  const bool exact = E > 0 && (int)rows == Q * E;
  // well-conditioned square jobs: FP32 sweeps + an orthogonal FP64 right factor
  // first (rk_precond.cu); the FP64 kernel below then finishes and certifies
  if (!use_warp && !with_v) {
    bool all = true;
    for (const JacobiJob& j : jobs) all = all && precondition_eligible(j);
    if (all) precondition_fp32(jobs, s, sms, smem_optin, g, G, Q);
  }
  auto launch = [&](auto kern) {
    RK_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    RK_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    RK_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    launch_cluster_kernel((const void*)kern, (unsigned)jobs.size() * cl, cl, kJThreads, smem, s, kargs);
  };
#define RK_JAC_E(QQ)                                                                   \
  switch (E) {                                                                         \
    case 4: exact ? launch(jacobi_cluster_kernel<QQ, 4, true>) : launch(jacobi_cluster_kernel<QQ, 4, false>); break;   \
    case 8: exact ? launch(jacobi_cluster_kernel<QQ, 8, true>) : launch(jacobi_cluster_kernel<QQ, 8, false>); break;   \
    case 16: exact ? launch(jacobi_cluster_kernel<QQ, 16, true>) : launch(jacobi_cluster_kernel<QQ, 16, false>); break; \
    case 32: exact ? launch(jacobi_cluster_kernel<QQ, 32, true>) : launch(jacobi_cluster_kernel<QQ, 32, false>); break; \
    default: launch(jacobi_cluster_kernel<QQ, 0, false>); break;                       \
  }
  const bool unroll = tn.jacobi_unroll;
  if (unroll && Q == 16 && E == 16 && exact && g == 16) {
    launch(jacobi_cluster_kernel<16, 16, true, 16>);  // c2's blocks: compile-time group count
  } else if (unroll && Q == 32 && E == 8 && exact && g == 8) {
    launch(jacobi_cluster_kernel<32, 8, true, 8>);  // c2's merge (latency plan)
  } else if (Q == 8) { RK_JAC_E(8) }
  else if (Q == 16) { RK_JAC_E(16) }
  else { RK_JAC_E(32) }
#undef RK_JAC_E
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
  uint32_t kmax = 0, rmax = 0;
  for (const FinalJob& f : jobs) {
    kmax = std::max(kmax, f.k);
    rmax = std::max(rmax, f.v_out ? std::max(f.rows, f.cols) : f.rows);
  }
  if (kmax == 0 || rmax == 0) return;
  const dim3 grid((unsigned)ceil_div(kmax, 32), (unsigned)ceil_div(rmax, 32), (unsigned)jobs.size());
  finalize_write_kernel<<<grid, 256, 0, s>>>(dj.get());
  RK_LAUNCH_CHECK();
}

void complete_columns_device(double* u, uint32_t rows, uint32_t cols, const uint8_t* deficient, int* d_fail,
                             cudaStream_t s) {
  const size_t smem = ((size_t)2 * rows + cols) * 8;
  if (smem > 200 * 1024) fail(RK_RUNTIME, "orthonormal completion: matrix too large");
  RK_CUDA_CHECK(cudaFuncSetAttribute(complete_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  complete_kernel<<<1, kCThreads, smem, s>>>(u, rows, cols, deficient, d_fail);
  RK_LAUNCH_CHECK();
}

namespace {
// apply_q with the reflectors staged through shared memory a panel of kP at a time:
// a CTA owns 8 warps x CW columns of one job; the panel's reflectors (rows >= their
// diagonal, zeros above) are loaded once per CTA with coalesced reads, then every warp
// applies them to its columns from shared memory. Replaces a dependent L2 round trip
// per reflector with one per panel (c3's 512 wide blocks: 3.1 -> ~0.3 ms).
constexpr int kPanel = 16;
template <int CW, int E>
__global__ void __launch_bounds__(256) apply_q_panel_kernel(const ApplyQJob* jobs) {
  extern __shared__ __align__(16) double vs[];  // kPanel x (32 E)
  const ApplyQJob j = jobs[blockIdx.y];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t m = j.qr.m, K = j.qr.m < j.qr.n ? j.qr.m : j.qr.n;
  const uint32_t ld = 32 * E;
  const uint32_t c0 = (blockIdx.x * 8 + warp) * CW;
  double o[CW][E];
#pragma unroll
  for (int cw = 0; cw < CW; ++cw)
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const uint32_t i = lane + 32 * e, c = c0 + cw;
      o[cw][e] = (c < j.ncols && i < j.x_rows) ? j.x[(uint64_t)c * j.x_rows + i] : 0.0;
    }
  __shared__ double sbeta[kPanel];
  for (int p1 = (int)K; p1 > 0; p1 -= kPanel) {
    const int p0 = p1 - kPanel > 0 ? p1 - kPanel : 0;
    const int np = p1 - p0;
    __syncthreads();  // the previous panel is consumed
    for (int t = threadIdx.x; t < np * (int)ld; t += blockDim.x) {
      const int q = t / (int)ld, i = t % (int)ld, kk = p0 + q;
      vs[q * ld + i] = (i >= kk && (uint32_t)i < m) ? j.qr.a[(uint64_t)kk * j.qr.lda + i] : 0.0;
    }
    if (threadIdx.x < np) sbeta[threadIdx.x] = j.qr.beta[p0 + threadIdx.x];
    __syncthreads();
    for (int q = np - 1; q >= 0; --q) {  // last reflector first
      const double beta = sbeta[q];
      if (beta == 0.0) continue;
      const double* v = vs + q * ld;
      double vv[E];
      double d[CW];
#pragma unroll
      for (int cw = 0; cw < CW; ++cw) d[cw] = 0.0;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        vv[e] = v[lane + 32 * e];
#pragma unroll
        for (int cw = 0; cw < CW; ++cw) d[cw] = fma(vv[e], o[cw][e], d[cw]);
      }
#pragma unroll
      for (int off = 16; off; off >>= 1)
#pragma unroll
        for (int cw = 0; cw < CW; ++cw) d[cw] += __shfl_xor_sync(0xffffffffu, d[cw], off);
#pragma unroll
      for (int cw = 0; cw < CW; ++cw) {
        const double bw = beta * d[cw];
#pragma unroll
        for (int e = 0; e < E; ++e) o[cw][e] = fma(-bw, vv[e], o[cw][e]);
      }
    }
  }
#pragma unroll
  for (int cw = 0; cw < CW; ++cw)
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const uint32_t i = lane + 32 * e, c = c0 + cw;
      if (c < j.ncols && i < m) j.out[(uint64_t)c * m + i] = o[cw][e];
    }
}
}  // namespace

void apply_q_batched(const std::vector<ApplyQJob>& jobs, cudaStream_t s) {
  if (jobs.empty()) return;
  uint32_t cmax = 0;
  for (const ApplyQJob& j : jobs) cmax = std::max(cmax, j.ncols);
  if (!cmax) return;
  uint32_t mmax = 0;
  for (const ApplyQJob& j : jobs) mmax = std::max(mmax, j.qr.m);
  DBuf<ApplyQJob> dj(jobs.size(), s);
  to_device(dj.get(), jobs.data(), jobs.size(), s);
  {  // factored with T kept: the compact-WY apply on the tensor cores
    uint32_t nbw = jobs[0].wy_nb;
    for (const ApplyQJob& j : jobs)
      if (j.wy_nb != nbw || j.qr.split || !j.qr.tmat) nbw = 0;
    if (nbw && tuning().apply_q_wy && apply_q_wy_batched(dj.get(), jobs.size(), mmax, cmax, nbw, s)) return;
  }
  constexpr int kCW = 4;
  auto panel = [&](auto kern, int cw, int e) {
    const size_t smem = (size_t)kPanel * 32 * e * sizeof(double);
    RK_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const dim3 grid((unsigned)ceil_div(cmax, 8 * (uint64_t)cw), (unsigned)jobs.size());
    kern<<<grid, 256, smem, s>>>(dj.get());
  };
  const unsigned gr = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(ceil_div((uint64_t)cmax, 8 * kCW), 64));
  const dim3 grid(gr, (unsigned)jobs.size());
  if (!tuning().apply_q_regs && mmax <= 128) panel(apply_q_panel_kernel<kCW, 4>, kCW, 4);
  else if (!tuning().apply_q_regs && mmax <= 256) panel(apply_q_panel_kernel<kCW, 8>, kCW, 8);
  else if (!tuning().apply_q_regs && mmax <= 512) panel(apply_q_panel_kernel<kCW, 16>, kCW, 16);
  else if (!tuning().apply_q_regs && mmax <= 1024) panel(apply_q_panel_kernel<2, 32>, 2, 32);
  else if (mmax <= 128) apply_q_regs_kernel<kCW, 4><<<grid, 256, 0, s>>>(dj.get());
  else if (mmax <= 256) apply_q_regs_kernel<kCW, 8><<<grid, 256, 0, s>>>(dj.get());
  else if (mmax <= 512) apply_q_regs_kernel<kCW, 16><<<grid, 256, 0, s>>>(dj.get());
  else if (mmax <= 1024) apply_q_regs_kernel<2, 32><<<grid, 256, 0, s>>>(dj.get());
  else {
    const unsigned gx = (unsigned)std::min<uint64_t>(ceil_div((uint64_t)cmax * 32, 256), 64);
    apply_q_batched_kernel<<<dim3(gx, (unsigned)jobs.size()), 256, 0, s>>>(dj.get());
  }
  RK_LAUNCH_CHECK();
}

void apply_q_device(const QrJob& qr, const double* x, uint32_t x_rows, uint32_t ncols, double* out, cudaStream_t s) {
  if (!ncols) return;
  unsigned grid = (unsigned)std::min<uint64_t>(ceil_div((uint64_t)ncols * 32, 256), 4096);
  apply_q_kernel<<<grid, 256, 0, s>>>(qr, x, x_rows, ncols, out);
  RK_LAUNCH_CHECK();
}

}  // namespace rk
