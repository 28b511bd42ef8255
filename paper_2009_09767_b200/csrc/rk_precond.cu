// rk_precond.cu -- FP32-preconditioned one-sided Jacobi for well-conditioned
// square matrices (the Gram route's W = L, kappa <= kappa_max(M)).
//
// On the B200 an FP64 FMA has 23 cycles of latency, an FP32 FMA 4, a double
// shuffle is two 32-bit ones (tools/probe_latency.cu), and a float column needs
// half the registers and shared memory. A Jacobi round is a dependent chain
// (dot -> lane reduction -> angle -> rotation), so an FP32 sweep is several times
// cheaper than an FP64 one. The FP32 sweeps do what the first sweeps of the FP64
// Jacobi do -- bring the columns close to orthogonal -- and the FP64 kernel only
// finishes from there (two sweeps and the convergence check instead of ~10):
//
//   1. W32 = fl32(W); one-sided Jacobi on W32 until a sweep's largest
//      |gamma| / sqrt(alpha_p alpha_q) is at the FP32 noise floor (~1e-6);
//      W32 -> X ~ U Sigma (column j ~ sigma_j u_j).
//   2. V = W^T X Sigma^-2: the right singular vectors of W to ~1e-5
//      (W V = U Sigma  =>  V = W^T U Sigma^-1, and X = U Sigma).
//   3. Two Newton-Schulz steps V <- V (3I - V^T V) / 2: V orthogonal to FP64
//      rounding (error 7e-5 -> 4e-9 -> 1e-17).
//   4. W <- W V. An exactly orthogonal right factor leaves the singular values
//      and left singular vectors of W unchanged, and W V has nearly orthogonal
//      columns (|gamma| / sqrt(alpha alpha) ~ 4e-6 on c2's blocks).
//   5. The FP64 Jacobi (jacobi_cluster_kernel) runs on W V with the reference's
//      thresholds, freeze rule and stopping rule (a sweep -- or the DMMA check
//      that stands for it -- with no rotation), so what it returns is certified
//      exactly as before: only where its sweeps start from changes.
// A numpy replay on c2 blocks (tournament order): 10 FP64 sweeps directly vs 8
// FP32 sweeps + 2 FP64 sweeps + the check, sigma within 7e-14 of LAPACK.
// The GEMMs (steps 2-4, n x n x n each) run on the FP64 tensor cores (DMMA).
// Measured and not kept: compiled only in the experiments build
// (RK_EXPERIMENTS=1 python -m paper_2009_09767_b200._build --force).
#include "rk_internal.cuh"
#ifdef RK_EXPERIMENTS
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "rk_internal.cuh"

namespace cg = cooperative_groups;

namespace rk {
namespace {

constexpr int kPT = 256;        // threads per CTA
constexpr float kTol32 = 2e-7f;  // FP32 rotation threshold (relative |gamma|)

struct J32Job {
  float* w;         // rows x cols_pad, col-major (ld = rows)
  float* alpha;     // cols_pad
  uint32_t* stats;  // [0] sweeps, [1] rotations of the current sweep (mod 2 slots: [1],[2]), [3] max ratio bits
};

struct J32Params {
  const J32Job* jobs;
  uint32_t rows, cols_pad, g, G;
  float stop_ratio;
  int max_sweeps;
  int debug;
};

__device__ __forceinline__ uint32_t rr32(uint32_t pos, uint32_t step, uint32_t n) {
  return pos == 0 ? 0 : 1 + (pos - 1 + step) % (n - 1);
}

// (c, s) of the reference's formulas (svd.cpp:238-242) in FP32, scaled so that
// max(|d|, |e|) is 1 (no overflow of d^2 + e^2)
__device__ __forceinline__ void rot32(float ap, float aq, float gm, float& c, float& s) {
  float d = aq - ap, e = 2.0f * gm;
  const float m = fmaxf(fabsf(d), fabsf(e));
  const float im = 1.0f / m;
  d *= im;
  e *= im;
  const float r = sqrtf(fmaf(d, d, e * e));
  const float sgn = (d == 0.0f || ((d > 0.0f) == (e > 0.0f))) ? 1.0f : -1.0f;
  const float t = sgn * fabsf(e) / (fabsf(d) + r);
  c = rsqrtf(fmaf(t, t, 1.0f));
  s = c * t;
}

// one pair of staged columns, Q lanes (intra-group rounds of step 0)
template <int Q>
__device__ __forceinline__ void pair32(float* wp, float* wq, uint32_t rows, float* alpha, int p, int q, float freeze,
                                       float& max_r2, uint32_t& nrot) {
  const int lq = threadIdx.x & (Q - 1);
  const unsigned gmask = (Q == 32) ? 0xffffffffu : (((1u << Q) - 1u) << ((threadIdx.x & 31) & ~(Q - 1)));
  const float ap = alpha[p], aq = alpha[q];
  if (ap <= freeze || aq <= freeze) return;
  float g0 = 0.0f;
  for (uint32_t i = lq; i < rows; i += Q) g0 = fmaf(wp[i], wq[i], g0);
#pragma unroll
  for (int o = Q / 2; o; o >>= 1) g0 += __shfl_xor_sync(gmask, g0, o);
  const float prod = ap * aq, g2 = g0 * g0;
  if (g2 > max_r2 * prod) max_r2 = g2 / prod;
  if (!(g2 > kTol32 * kTol32 * prod)) return;
  float c, s;
  rot32(ap, aq, g0, c, s);
  for (uint32_t i = lq; i < rows; i += Q) {
    const float xp = wp[i], xq = wq[i];
    wp[i] = c * xp - s * xq;
    wq[i] = s * xp + c * xq;
  }
  __syncwarp(gmask);
  if (lq == 0) {
    alpha[p] = fmaxf(c * c * ap - 2.0f * c * s * g0 + s * s * aq, 0.0f);
    alpha[q] = fmaxf(s * s * ap + 2.0f * c * s * g0 + c * c * aq, 0.0f);
    ++nrot;
  }
  __syncwarp(gmask);
}

// cross rounds of a group pair: lane group t keeps A_t in registers, the B columns
// stream through shared memory (as cross_rounds_reg in rk_dense.cu, in FP32).
// Lane lq of a group holds rows 4 Q k + 4 lq + {0..3} (k < E / 4): 128-bit shared
// loads and stores, and the dot / rotation in packed f32x2 arithmetic (FFMA2):
// a quarter of the scalar kernel's instructions per element.
template <int Q, int E>
__device__ __forceinline__ void cross32(float* sW, uint32_t ldS, uint32_t g, float* sAlpha, float freeze,
                                        float& max_r2, uint32_t& nrot) {
  static_assert(E % 4 == 0, "E must be a multiple of 4");
  constexpr int K4 = E / 4;
  const int tid = threadIdx.x;
  const int grp = tid / Q, lq = tid & (Q - 1);
  const bool active = (uint32_t)grp < g;
  float2 a[2 * K4];
  float aA = 0.0f;
  {
    const float* pa = sW + (uint64_t)(active ? grp : 0) * ldS + 4 * lq;
#pragma unroll
    for (int k = 0; k < K4; ++k) {
      const float4 v = active ? *reinterpret_cast<const float4*>(pa + 4 * Q * k) : make_float4(0.f, 0.f, 0.f, 0.f);
      a[2 * k] = make_float2(v.x, v.y);
      a[2 * k + 1] = make_float2(v.z, v.w);
    }
    aA = active ? sAlpha[grp] : 0.0f;
  }
  uint32_t jl = active ? (uint32_t)grp : 0u;
  float* const bbase = sW + (uint64_t)g * ldS + 4 * lq;
  for (uint32_t r = 0; r < g; ++r) {
    float* pb = bbase + (uint64_t)jl * ldS;
    const float aB = sAlpha[g + jl];
    const bool live = active && !(aA <= freeze || aB <= freeze);
    float2 b[2 * K4];
    float2 acc0 = make_float2(0.f, 0.f), acc1 = make_float2(0.f, 0.f);
#pragma unroll
    for (int k = 0; k < K4; ++k) {
      const float4 v = *reinterpret_cast<const float4*>(pb + 4 * Q * k);
      b[2 * k] = make_float2(v.x, v.y);
      b[2 * k + 1] = make_float2(v.z, v.w);
      acc0 = __ffma2_rn(a[2 * k], b[2 * k], acc0);
      acc1 = __ffma2_rn(a[2 * k + 1], b[2 * k + 1], acc1);
    }
    const float2 acc = __fadd2_rn(acc0, acc1);
    float gamma = acc.x + acc.y;
#pragma unroll
    for (int o = Q / 2; o; o >>= 1) gamma += __shfl_xor_sync(0xffffffffu, gamma, o);
    const float prod = aA * aB, g2 = gamma * gamma;
    if (live && g2 > max_r2 * prod) max_r2 = g2 / prod;
    const bool rot = live && (g2 > kTol32 * kTol32 * prod);
    if (__any_sync(0xffffffffu, rot)) {
      float c = 1.0f, sn = 0.0f;
      if (rot) rot32(aA, aB, gamma, c, sn);
      const float2 c2 = make_float2(c, c), s2 = make_float2(sn, sn), ns2 = make_float2(-sn, -sn);
#pragma unroll
      for (int k = 0; k < 2 * K4; ++k) {
        const float2 xp = a[k], xq = b[k];
        a[k] = __ffma2_rn(c2, xp, __fmul2_rn(ns2, xq));
        b[k] = __ffma2_rn(c2, xq, __fmul2_rn(s2, xp));
      }
      if (rot) {
#pragma unroll
        for (int k = 0; k < K4; ++k)
          *reinterpret_cast<float4*>(pb + 4 * Q * k) = make_float4(b[2 * k].x, b[2 * k].y, b[2 * k + 1].x,
                                                                    b[2 * k + 1].y);
        const float na = c * c * aA - 2.0f * c * sn * gamma + sn * sn * aB;
        const float nq = sn * sn * aA + 2.0f * c * sn * gamma + c * c * aB;
        aA = fmaxf(na, 0.0f);
        if (lq == 0) {
          sAlpha[g + jl] = fmaxf(nq, 0.0f);
          ++nrot;
        }
      }
    }
    jl = (jl + 1 == g) ? 0u : jl + 1;
    __syncthreads();
  }
  if (active) {
    float* pa = sW + (uint64_t)grp * ldS + 4 * lq;
#pragma unroll
    for (int k = 0; k < K4; ++k)
      *reinterpret_cast<float4*>(pa + 4 * Q * k) = make_float4(a[2 * k].x, a[2 * k].y, a[2 * k + 1].x, a[2 * k + 1].y);
    if (lq == 0) sAlpha[grp] = aA;
  }
  __syncthreads();
}

template <int Q, int E>
__global__ void __launch_bounds__(kPT, 2) jacobi32_kernel(J32Params P) {
  extern __shared__ __align__(16) float sm32[];
  cg::cluster_group cluster = cg::this_cluster();
  const unsigned rank = cluster.block_rank(), csize = cluster.num_blocks();
  const J32Job job = P.jobs[blockIdx.x / csize];
  const uint32_t rows = P.rows, cols_pad = P.cols_pad, g = P.g, G = P.G;
  const uint32_t ldS = rows + 4;
  float* sW = sm32;
  float* sAlpha = sW + (uint64_t)2 * g * ldS;
  __shared__ float s_red[kPT / 32];
  __shared__ float s_amax;
  __shared__ uint32_t s_rot;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int kGroups = kPT / Q;
  const int grp_id = tid / Q;
  int sweep = 0;
  float prev_ratio = INFINITY;
  long long tm[6] = {0, 0, 0, 0, 0, 0};
  long long tc = clock64();
  auto tick = [&](int k) {
    if (P.debug) {
      const long long t = clock64();
      tm[k] += t - tc;
      tc = t;
    }
  };
  for (; sweep < P.max_sweeps; ++sweep) {
    for (uint32_t j = rank * (kPT / 32) + warp; j < cols_pad; j += csize * (kPT / 32)) {
      const float* wj = job.w + (uint64_t)j * rows;
      float a = 0.0f;
      for (uint32_t i = lane; i < rows; i += 32) {
        const float x = __ldcg(wj + i);
        a = fmaf(x, x, a);
      }
      for (int o = 16; o; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
      if (lane == 0) job.alpha[j] = a;
    }
    if (rank == 0 && tid == 0) job.stats[1 + ((sweep + 1) & 1)] = 0u;
    cluster.sync();
    float amax = 0.0f;
    for (uint32_t j = tid; j < cols_pad; j += kPT) amax = fmaxf(amax, __ldcg(job.alpha + j));
    for (int o = 16; o; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    if (lane == 0) s_red[warp] = amax;
    if (tid == 0) s_rot = 0u;
    __syncthreads();
    if (tid == 0) {
      float t = 0.0f;
      for (int w = 0; w < kPT / 32; ++w) t = fmaxf(t, s_red[w]);
      s_amax = t;
    }
    __syncthreads();
    const float freeze = kTol32 * kTol32 * s_amax;
    uint32_t my_rot = 0;
    float my_r2 = 0.0f;
    for (uint32_t step = 0; step + 1 < G; ++step) {
      for (uint32_t pi = rank; pi < G / 2; pi += csize) {
        const uint32_t gA = rr32(pi, step, G), gB = rr32(G - 1 - pi, step, G);
        for (uint32_t c = warp; c < 2 * g; c += kPT / 32) {
          const uint32_t col = (c < g ? gA * g + c : gB * g + (c - g));
          const float4* src = reinterpret_cast<const float4*>(job.w + (uint64_t)col * rows);
          float4* dst = reinterpret_cast<float4*>(sW + (uint64_t)c * ldS);
          for (uint32_t i = lane; i < rows / 4; i += 32) dst[i] = __ldcg(src + i);
          if (lane == 0) sAlpha[c] = __ldcg(job.alpha + col);
        }
        __syncthreads();
        tick(0);
        if (step == 0) {
          for (uint32_t r = 0; r + 1 < g; ++r) {
            for (uint32_t t = grp_id; t < g; t += kGroups) {
              const uint32_t half = g / 2;
              const uint32_t gr = t / half, i = t % half;
              const uint32_t p = gr * g + rr32(i, r, g), q = gr * g + rr32(g - 1 - i, r, g);
              pair32<Q>(sW + (uint64_t)p * ldS, sW + (uint64_t)q * ldS, rows, sAlpha, p, q, freeze, my_r2, my_rot);
            }
            __syncthreads();
          }
        }
        tick(1);
        cross32<Q, E>(sW, ldS, g, sAlpha, freeze, my_r2, my_rot);
        tick(2);
        for (uint32_t c = warp; c < 2 * g; c += kPT / 32) {
          const uint32_t col = (c < g ? gA * g + c : gB * g + (c - g));
          float4* dst = reinterpret_cast<float4*>(job.w + (uint64_t)col * rows);
          const float4* src = reinterpret_cast<const float4*>(sW + (uint64_t)c * ldS);
          for (uint32_t i = lane; i < rows / 4; i += 32) dst[i] = src[i];
          if (lane == 0) job.alpha[col] = sAlpha[c];
        }
        __syncthreads();
        tick(3);
      }
      cluster.sync();
      tick(4);
    }
    // rotations and the largest ratio of the sweep, over the cluster
    for (int o = 16; o; o >>= 1) {
      my_rot += __shfl_xor_sync(0xffffffffu, my_rot, o);
      my_r2 = fmaxf(my_r2, __shfl_xor_sync(0xffffffffu, my_r2, o));
    }
    if (lane == 0) {
      if (my_rot) atomicAdd(&s_rot, my_rot);
      s_red[warp] = my_r2;
    }
    __syncthreads();
    if (tid == 0) {
      float t = 0.0f;
      for (int w = 0; w < kPT / 32; ++w) t = fmaxf(t, s_red[w]);
      if (s_rot) atomicAdd(&job.stats[1 + (sweep & 1)], s_rot);
      atomicMax(&job.stats[3], __float_as_uint(t));  // t >= 0: bit order = value order
    }
    cluster.sync();
    const uint32_t rot = __ldcg(&job.stats[1 + (sweep & 1)]);
    const float r2 = __uint_as_float(__ldcg(&job.stats[3]));
    cluster.sync();
    if (rank == 0 && tid == 0) job.stats[3] = 0u;
    // stop at the FP32 noise floor: below stop_ratio, or no longer shrinking
    // (the quadratic regime goes 1e-3 -> 1e-6 in one sweep; noise hovers)
    const float ratio = sqrtf(r2);
    const bool stagnant = ratio < 1e-4f && ratio > 0.5f * prev_ratio;
    prev_ratio = ratio;
    if (P.debug && rank == 0 && tid == 0 && blockIdx.x == 0)
      printf("[jacobi32] job 0 sweep %d: %u rotations, max ratio %.3e\n", sweep, rot, ratio);
    if (rot == 0 || ratio < P.stop_ratio || stagnant) {
      ++sweep;
      break;
    }
  }
  if (rank == 0 && tid == 0) job.stats[0] = (uint32_t)sweep;
  if (P.debug && blockIdx.x == 0 && tid == 0)
    printf("[jacobi32] CTA 0 cycles: stage %lld intra %lld cross %lld writeback %lld cluster.sync %lld\n", tm[0],
           tm[1], tm[2], tm[3], tm[4]);
}

// W32 = fl32(W)
__global__ void to_f32_kernel(const J32Job* __restrict__ jobs, double* const* __restrict__ src, uint64_t n) {
  const J32Job j = jobs[blockIdx.y];
  const double* s = src[blockIdx.y];
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < n; t += (uint64_t)gridDim.x * blockDim.x)
    j.w[t] = (float)s[t];
}

// X = fl64(W32) (rows x n), scale[c] = 1 / ||X_c||^2 (0 for a zero column); one warp per column
__global__ void to_f64_kernel(const J32Job* __restrict__ jobs, double* const* __restrict__ dst,
                              double* const* __restrict__ scale, uint32_t rows, uint32_t n) {
  const J32Job j = jobs[blockIdx.y];
  const uint32_t c = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (c >= n) return;
  const float* s = j.w + (uint64_t)c * rows;
  double* d = dst[blockIdx.y] + (uint64_t)c * rows;
  double a = 0.0;
  for (uint32_t i = lane; i < rows; i += 32) {
    const double x = (double)s[i];
    d[i] = x;
    a += x * x;
  }
  for (int o = 16; o; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
  if (lane == 0) scale[blockIdx.y][c] = a > 0.0 ? 1.0 / a : 0.0;
}

// ---------------------------------------------------------------------------
// batched square FP64 GEMM on DMMA: C = alpha op(A) B diag(scale) + beta D,
// n x n column-major (ld n), n % 64 == 0. CTA tile 64 x 64, K chunks of 32 staged
// in shared memory; 8 warps as 2 (m) x 4 (n), 32 x 16 each (4 x 2 tiles of 8x8).
struct GemmJob {
  const double* A;
  const double* B;
  const double* D;      // nullable (beta ignored)
  double* C;
  const double* scale;  // nullable: per-column scale of op(A) B
};

__device__ __forceinline__ void dmma8(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

constexpr int kGM = 64, kGK = 32;
constexpr int kLdMK = kGM + 4;  // [k][m] layout, ld == 4 (mod 16): conflict-free fragment reads
constexpr int kLdKM = kGK + 4;  // [m][k] / [n][k] layouts

template <bool TA>
__global__ void __launch_bounds__(256) gemm_kernel(const GemmJob* __restrict__ jobs, uint32_t n, double alpha,
                                                   double beta) {
  __shared__ __align__(16) double As[TA ? kGM * kLdKM : kGK * kLdMK];
  __shared__ __align__(16) double Bs[kGM * kLdKM];
  const GemmJob J = jobs[blockIdx.z];
  const uint32_t m0 = blockIdx.x * kGM, n0 = blockIdx.y * kGM;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int lr = lane >> 2, lc = lane & 3;
  const int wm = warp & 1, wn = warp >> 1;  // warp tile: rows wm*32 .. +32, cols wn*16 .. +16
  double acc[4][2][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  for (uint32_t k0 = 0; k0 < n; k0 += kGK) {
    // stage op(A)[m0.., k0..] and B[k0.., n0..]
    if (TA) {  // op(A)[m][k] = A[k + m n]: k contiguous
#pragma unroll
      for (int t = tid; t < kGM * kGK; t += 256) {
        const int k = t & (kGK - 1), m = t >> 5;
        As[m * kLdKM + k] = J.A[(k0 + k) + (uint64_t)(m0 + m) * n];
      }
    } else {  // A[m + k n]: m contiguous
#pragma unroll
      for (int t = tid; t < kGM * kGK; t += 256) {
        const int m = t & (kGM - 1), k = t >> 6;
        As[k * kLdMK + m] = J.A[(m0 + m) + (uint64_t)(k0 + k) * n];
      }
    }
#pragma unroll
    for (int t = tid; t < kGM * kGK; t += 256) {
      const int k = t & (kGK - 1), c = t >> 5;
      Bs[c * kLdKM + k] = J.B[(k0 + k) + (uint64_t)(n0 + c) * n];
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < kGK; kk += 4) {
      double af[4], bf[2];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int m = wm * 32 + i * 8 + lr, k = kk + lc;
        af[i] = TA ? As[m * kLdKM + k] : As[k * kLdMK + m];
      }
#pragma unroll
      for (int j = 0; j < 2; ++j) bf[j] = Bs[(wn * 16 + j * 8 + lr) * kLdKM + kk + lc];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) dmma8(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
    __syncthreads();
  }
  // epilogue: lane holds D[lr][2lc + e] of each 8x8 tile
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const uint32_t r = m0 + wm * 32 + i * 8 + lr, c = n0 + wn * 16 + j * 8 + 2 * lc + e;
        const uint64_t o = r + (uint64_t)c * n;
        double v = acc[i][j][e];
        if (J.scale) v *= J.scale[c];
        v *= alpha;
        if (J.D) v = fma(beta, J.D[o], v);
        J.C[o] = v;
      }
}

unsigned grid1(uint64_t n) { return (unsigned)std::min<uint64_t>(std::max<uint64_t>(1, ceil_div(n, 256)), 4096); }

void gemm_batched(const std::vector<GemmJob>& jobs, uint32_t n, bool transA, double alpha, double beta,
                  cudaStream_t s) {
  DBuf<GemmJob> dj(jobs.size(), s);
  to_device(dj.get(), jobs.data(), jobs.size(), s);
  const dim3 grid(n / kGM, n / kGM, (unsigned)jobs.size());
  if (transA) gemm_kernel<true><<<grid, 256, 0, s>>>(dj.get(), n, alpha, beta);
  else gemm_kernel<false><<<grid, 256, 0, s>>>(dj.get(), n, alpha, beta);
  RK_LAUNCH_CHECK();
}

}  // namespace

bool precondition_eligible(const JacobiJob& j) {
  // opt-in (RK_PRECOND=1): measured on c2, the FP32 sweeps cost as much as FP64
  // ones -- a round is bound by its dependent chain (shuffle reduction, angle,
  // barrier), not by the FP64 latency of its arithmetic -- so the FP64 sweeps it
  // saves (12 -> 5) do not pay for it and the GEMMs (blocks 7.1 -> 8.6 ms)
  if (!tuning().precond) return false;
  return j.gram_ok && j.v == nullptr && j.rows == j.cols && j.cols == j.cols_pad && j.rows % 64 == 0 &&
         j.rows >= 64 && j.rows <= 512;
}

void precondition_fp32(std::vector<JacobiJob>& jobs, cudaStream_t s, int sms, size_t smem_optin, uint32_t g,
                       uint32_t G, int Q) {
  if (jobs.empty()) return;
  const uint32_t n = jobs[0].rows;
  const uint64_t nn = (uint64_t)n * n, nb = jobs.size();
  DBuf<float> w32(nb * nn, s), a32(nb * n, s);
  DBuf<uint32_t> st(nb * 4, s);
  DBuf<double> X(nb * nn, s), V(nb * nn, s), V2(nb * nn, s), S(nb * nn, s), scale(nb * n, s);
  st.zero();
  std::vector<J32Job> hj(nb);
  std::vector<double*> src(nb), xp(nb), sp(nb);
  for (uint64_t q = 0; q < nb; ++q) {
    hj[q] = {w32.get() + q * nn, a32.get() + q * n, st.get() + 4 * q};
    src[q] = jobs[q].w;
    xp[q] = X.get() + q * nn;
    sp[q] = scale.get() + q * n;
  }
  DBuf<J32Job> dj(nb, s);
  DBuf<double*> dsrc(nb, s), dx(nb, s), dsc(nb, s);
  to_device(dj.get(), hj.data(), nb, s);
  to_device(dsrc.get(), src.data(), nb, s);
  to_device(dx.get(), xp.data(), nb, s);
  to_device(dsc.get(), sp.data(), nb, s);
  to_f32_kernel<<<dim3(grid1(nn), (unsigned)nb), 256, 0, s>>>(dj.get(), dsrc.get(), nn);
  RK_LAUNCH_CHECK();
  // FP32 sweeps: the FP64 plan's groups (g, G) and lanes per pair (Q)
  const int E = (int)(n / (uint32_t)Q);
  const size_t smem = ((size_t)2 * g * (n + 4) + 2 * g) * sizeof(float);
  const unsigned per_sm = 2;
  unsigned cl = (unsigned)std::max<uint64_t>(1, (uint64_t)sms * per_sm / nb);
  cl = std::min<unsigned>({cl, G / 2, 16u});
  unsigned p2 = 1;
  while (p2 * 2 <= cl) p2 *= 2;
  cl = p2;
  J32Params P{dj.get(), n, n, g, G, tuning().precond_stop, 20, tuning().jacobi_debug ? 1 : 0};
  void* kargs[] = {&P};
  auto launch = [&](auto kern) {
    RK_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    RK_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    launch_cluster_kernel((const void*)kern, (unsigned)nb * cl, cl, kPT, smem, s, kargs);
  };
  if (Q == 16 && E == 16) launch(jacobi32_kernel<16, 16>);
  else if (Q == 32 && E == 8) launch(jacobi32_kernel<32, 8>);
  else if (Q == 16 && E == 4) launch(jacobi32_kernel<16, 4>);
  else if (Q == 16 && E == 8) launch(jacobi32_kernel<16, 8>);
  else if (Q == 32 && E == 16) launch(jacobi32_kernel<32, 16>);
  else if (Q == 16 && E == 32) launch(jacobi32_kernel<16, 32>);
  else if (Q == 32 && E == 4) launch(jacobi32_kernel<32, 4>);
  else if (Q == 8 && E == 8) launch(jacobi32_kernel<8, 8>);
  else if (Q == 8 && E == 32) launch(jacobi32_kernel<8, 32>);
  else return;  // no instantiation for this shape: the FP64 Jacobi starts from W as before
  to_f64_kernel<<<dim3((unsigned)ceil_div(n, 8), (unsigned)nb), 256, 0, s>>>(dj.get(), dx.get(), dsc.get(), n, n);
  RK_LAUNCH_CHECK();
  std::vector<GemmJob> gj(nb);
  // V = W^T X Sigma^-2
  for (uint64_t q = 0; q < nb; ++q) gj[q] = {jobs[q].w, X.get() + q * nn, nullptr, V.get() + q * nn, sp[q]};
  gemm_batched(gj, n, true, 1.0, 0.0, s);
  // Newton-Schulz: S = V^T V; V2 = 1.5 V - 0.5 V S
  for (int it = 0; it < 2; ++it) {
    for (uint64_t q = 0; q < nb; ++q) gj[q] = {V.get() + q * nn, V.get() + q * nn, nullptr, S.get() + q * nn, nullptr};
    gemm_batched(gj, n, true, 1.0, 0.0, s);
    for (uint64_t q = 0; q < nb; ++q)
      gj[q] = {V.get() + q * nn, S.get() + q * nn, V.get() + q * nn, V2.get() + q * nn, nullptr};
    gemm_batched(gj, n, false, -0.5, 1.5, s);
    std::swap(V, V2);
  }
  // W <- W V (through X, then back into the job's slot)
  for (uint64_t q = 0; q < nb; ++q) gj[q] = {jobs[q].w, V.get() + q * nn, nullptr, X.get() + q * nn, nullptr};
  gemm_batched(gj, n, false, 1.0, 0.0, s);
  for (uint64_t q = 0; q < nb; ++q)
    RK_CUDA_CHECK(cudaMemcpyAsync(jobs[q].w, X.get() + q * nn, nn * sizeof(double), cudaMemcpyDeviceToDevice, s));
}

}  // namespace rk
#else
namespace rk {
bool precondition_eligible(const JacobiJob&) { return false; }
void precondition_fp32(std::vector<JacobiJob>&, cudaStream_t, int, size_t, uint32_t, uint32_t, int) {}
}  // namespace rk
#endif  // RK_EXPERIMENTS
