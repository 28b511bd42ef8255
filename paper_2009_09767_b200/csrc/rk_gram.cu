// rk_gram.cu -- Gram + Cholesky route to the triangular factor R of a block.
//
// For A_d^T = Q R the factor R is, up to row signs, the Cholesky factor of the
// Gram G_d = A_d A_d^T (exact arithmetic). The Jacobi stage needs W = R^T = L
// (lower triangular), so the block factorization becomes
//     G_d = A_d A_d^T   (sparse: entry (r, s) is the dot of CSR rows r and s
//                        restricted to the block's columns, summed in ascending
//                        column order -- deterministic)
//     L = chol(G_d)     (blocked right-looking, DMMA SYRK trailing updates)
// at O(M^3/3) flops instead of the 2 n_d M^2 of Householder on the densified
// block. Cholesky squares the condition number, so the result is accepted only
// when the block's kappa = sigma_max/sigma_min is small enough that the Gram's
// rounding (~ M eps sigma_max^2) moves every singular value by less than
// 3e-11 relative, a third of the 1e-10 parity tolerance (kappa_max(M) =
// sqrt(6e-11 / (M eps)): 46 at M = 256, 32 at 512); otherwise -- and for a
// non-positive pivot -- the block is redone on the Householder path. The same
// kernels give the merge's R_P from P P^T (SYRK over the records).
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "rk_internal.cuh"

namespace rk {
namespace {

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

#ifdef RK_EXPERIMENTS  // not kept (measured): the row-pair merge-join Gram, RK_GRAM_PAIRS=1
// one thread per (block, r >= s) pair: G[r + s M] = G[s + r M] = sum_c A[r,c] A[s,c]
__global__ void sparse_gram_kernel(const uint64_t* __restrict__ row_ptr, const uint32_t* __restrict__ col,
                                   const double* __restrict__ val, uint32_t M, Partition p, uint64_t d_lo,
                                   uint64_t nblk, double* __restrict__ G, uint64_t stride) {
  const uint64_t pairs = (uint64_t)M * (M + 1) / 2;
  const uint64_t total = pairs * nblk;
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < total;
       t += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t bi = t / pairs, pi = t % pairs;
    // pi -> (r, s) with r >= s: r = floor((sqrt(8 pi + 1) - 1) / 2)
    uint32_t r = (uint32_t)((sqrt(8.0 * (double)pi + 1.0) - 1.0) * 0.5);
    while ((uint64_t)r * (r + 1) / 2 > pi) --r;
    while ((uint64_t)(r + 1) * (r + 2) / 2 <= pi) ++r;
    const uint32_t s = (uint32_t)(pi - (uint64_t)r * (r + 1) / 2);
    const uint64_t d = d_lo + bi;
    const uint32_t b = (uint32_t)p.begin(d), e = (uint32_t)p.end(d);
    auto lower = [&](uint64_t lo, uint64_t hi) {
      while (lo < hi) {
        uint64_t mid = (lo + hi) >> 1;
        if (col[mid] < b) lo = mid + 1; else hi = mid;
      }
      return lo;
    };
    uint64_t i = lower(row_ptr[r], row_ptr[r + 1]), iend = row_ptr[r + 1];
    uint64_t j = (r == s) ? i : lower(row_ptr[s], row_ptr[s + 1]), jend = row_ptr[s + 1];
    double acc = 0.0;
    if (r == s) {
      for (; i < iend && col[i] < e; ++i) acc = fma(val[i], val[i], acc);
    } else {
      while (i < iend && j < jend) {
        const uint32_t ci = col[i], cj = col[j];
        if (ci >= e || cj >= e) break;
        if (ci == cj) { acc = fma(val[i], val[j], acc); ++i; ++j; }
        else if (ci < cj) ++i;
        else ++j;
      }
    }
    double* g = G + bi * stride;
    g[r + (uint64_t)s * M] = acc;
    g[s + (uint64_t)r * M] = acc;
  }
}
#endif  // RK_EXPERIMENTS

// The same Gram from the other side: one thread per (block, row r). Row r's block
// entries are visited in ascending column c; for each, the column's entries in
// rows s <= r (CSC, ascending) add v_rc v_sc to G(r, s). Every G(r, s) therefore
// receives its products in ascending c starting from 0 -- the order of the
// merge-join above -- while the work is proportional to the block's entries
// times their column degrees, not to the M(M+1)/2 row pairs (c2: 0.21 ms ->
// ~0.02 ms). G must be zero on entry; the upper triangle is mirrored after.
__global__ void sparse_gram_rows_kernel(const uint64_t* __restrict__ row_ptr, const uint32_t* __restrict__ col,
                                        const double* __restrict__ val, const uint64_t* __restrict__ col_ptr,
                                        const uint32_t* __restrict__ row_idx, const double* __restrict__ cval,
                                        uint32_t M, Partition p, uint64_t d_lo, uint64_t nblk, double* __restrict__ G,
                                        uint64_t stride) {
  const uint64_t total = (uint64_t)M * nblk;
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < total;
       t += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t bi = t / M;
    const uint32_t r = (uint32_t)(t - bi * M);
    const uint64_t d = d_lo + bi;
    const uint32_t b = (uint32_t)p.begin(d), e = (uint32_t)p.end(d);
    uint64_t lo = row_ptr[r], hi = row_ptr[r + 1];
    while (lo < hi) {
      const uint64_t mid = (lo + hi) >> 1;
      if (col[mid] < b) lo = mid + 1; else hi = mid;
    }
    double* g = G + bi * stride;
    // G(r, r) gets one product per entry: kept in a register (the same sequence of
    // fmas from zero), so the loop carries no store -> load dependency through it
    double diag = 0.0;
    for (uint64_t i = lo, iend = row_ptr[r + 1]; i < iend; ++i) {
      const uint32_t c = col[i];
      if (c >= e) break;
      const double vr = val[i];
      for (uint64_t k = col_ptr[c], kend = col_ptr[c + 1]; k < kend; ++k) {
        const uint32_t sr = row_idx[k];
        if (sr > r) break;
        if (sr == r) {
          diag = fma(vr, cval[k], diag);
        } else {
          double* gp = g + r + (uint64_t)sr * M;
          *gp = fma(vr, cval[k], *gp);
        }
      }
    }
    g[r + (uint64_t)r * M] = diag;
  }
}

// G(s, r) = G(r, s) for r > s
__global__ void mirror_lower(double* __restrict__ G, uint64_t stride, uint32_t M, uint64_t nblk) {
  const uint64_t mm = (uint64_t)M * M;
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < mm * nblk;
       t += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t bi = t / mm, e = t - bi * mm;
    const uint32_t s2 = (uint32_t)(e / M), r = (uint32_t)(e - (uint64_t)s2 * M);
    if (r > s2) G[bi * stride + s2 + (uint64_t)r * M] = G[bi * stride + e];
  }
}

// ---------------------------------------------------------------------------
// split-K SYRK over the records: partial[kc][r + s M] = sum_{j in chunk kc} P[r, j] P[s, j]
// for 8x8 tiles with r-tile >= s-tile. The records are row-major M x k_d pieces.
struct SyrkChunk {
  const double* base;  // payload of one record (row-major M x k)
  uint32_t k;          // columns of this record
  uint32_t j0, j1;     // column range of this chunk inside the record
};

__global__ void syrk_records_kernel(const SyrkChunk* __restrict__ chunks, uint32_t n_chunks, uint32_t M,
                                    double* __restrict__ partial) {
  const int lane = threadIdx.x & 31;
  const int lr = lane >> 2, lc = lane & 3;
  const uint32_t tiles = M / 8;
  const uint64_t n_tile_pairs = (uint64_t)tiles * (tiles + 1) / 2;
  const uint64_t total = n_tile_pairs * n_chunks;
  for (uint64_t w = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; w < total;
       w += ((uint64_t)gridDim.x * blockDim.x) >> 5) {
    const uint32_t kc = (uint32_t)(w / n_tile_pairs);
    const uint64_t tp = w % n_tile_pairs;
    uint32_t ti = (uint32_t)((sqrt(8.0 * (double)tp + 1.0) - 1.0) * 0.5);
    while ((uint64_t)ti * (ti + 1) / 2 > tp) --ti;
    while ((uint64_t)(ti + 1) * (ti + 2) / 2 <= tp) ++ti;
    const uint32_t tj = (uint32_t)(tp - (uint64_t)ti * (ti + 1) / 2);
    const SyrkChunk c = chunks[kc];
    double d0 = 0.0, d1 = 0.0;
    // D(8x8) += A(8 rows of tile i x 4 k) * B(4 k x 8 rows of tile j)
    const double* pa = c.base + (uint64_t)(ti * 8 + lr) * c.k;  // A[lr][lc] = P[ti*8+lr, j]
    const double* pb = c.base + (uint64_t)(tj * 8 + lr) * c.k;  // B[lc][lr] = P[tj*8+lr, j]
#pragma unroll 4
    for (uint32_t j = c.j0; j < c.j1; j += 4) {
      const uint32_t jj = j + lc;
      const double a = jj < c.j1 ? pa[jj] : 0.0;
      const double b = jj < c.j1 ? pb[jj] : 0.0;
      dmma(d0, d1, a, b);
    }
    double* out = partial + (uint64_t)kc * M * M;
    // D row = ti*8 + lr, cols tj*8 + 2lc + {0,1}; column-major G(r, s) at r + s M
    const uint32_t r = ti * 8 + lr, s0 = tj * 8 + 2 * lc;
    out[r + (uint64_t)s0 * M] = d0;
    out[r + (uint64_t)(s0 + 1) * M] = d1;
  }
}

// The same partials with a 32 x 32 block (4 x 4 tiles) per warp: 8 loaded fragments
// feed up to 16 DMMAs per k-step instead of 2 feeding 1, a quarter of the L2 traffic
// (c3: 19.8 GB per merge with a tile per warp -- the kernel ran at the L2's rate,
// not the tensor cores'). Every tile accumulates its k-steps in the same order with
// the same zero padding, so the partials are bit-identical to syrk_records_kernel's.
// M % 32 == 0.
__global__ void __launch_bounds__(256) syrk_records_kernel4(const SyrkChunk* __restrict__ chunks, uint32_t n_chunks,
                                                             uint32_t M, double* __restrict__ partial) {
  const int lane = threadIdx.x & 31;
  const int lr = lane >> 2, lc = lane & 3;
  const uint32_t nb = M / 32;
  const uint64_t n_pairs = (uint64_t)nb * (nb + 1) / 2;
  const uint64_t total = n_pairs * n_chunks;
  for (uint64_t w = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; w < total;
       w += ((uint64_t)gridDim.x * blockDim.x) >> 5) {
    const uint32_t kc = (uint32_t)(w / n_pairs);
    const uint64_t bp = w % n_pairs;
    uint32_t bi = (uint32_t)((sqrt(8.0 * (double)bp + 1.0) - 1.0) * 0.5);
    while ((uint64_t)bi * (bi + 1) / 2 > bp) --bi;
    while ((uint64_t)(bi + 1) * (bi + 2) / 2 <= bp) ++bi;
    const uint32_t bj = (uint32_t)(bp - (uint64_t)bi * (bi + 1) / 2);  // bi >= bj
    const bool diag = bi == bj;
    const SyrkChunk c = chunks[kc];
    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    const double* pa[4];
    const double* pb[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      pa[i] = c.base + (uint64_t)(bi * 32 + i * 8 + lr) * c.k;
      pb[i] = c.base + (uint64_t)(bj * 32 + i * 8 + lr) * c.k;
    }
#pragma unroll 2
    for (uint32_t j = c.j0; j < c.j1; j += 4) {
      const uint32_t jj = j + lc;
      const bool ok = jj < c.j1;
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        a[i] = ok ? pa[i][jj] : 0.0;
        b[i] = ok ? pb[i][jj] : 0.0;
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int jx = 0; jx < 4; ++jx)
          if (!diag || i >= jx) dmma(acc[i][jx][0], acc[i][jx][1], a[i], b[jx]);
    }
    double* out = partial + (uint64_t)kc * M * M;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int jx = 0; jx < 4; ++jx)
        if (!diag || i >= jx) {
          const uint32_t r = bi * 32 + i * 8 + lr, s0 = bj * 32 + jx * 8 + 2 * lc;
          out[r + (uint64_t)s0 * M] = acc[i][jx][0];
          out[r + (uint64_t)(s0 + 1) * M] = acc[i][jx][1];
        }
  }
}

// G = sum of the partials in chunk order, mirrored to the upper triangle
__global__ void reduce_partials(const double* __restrict__ partial, uint32_t n_chunks, uint32_t M,
                                double* __restrict__ G) {
  const uint64_t total = (uint64_t)M * M;
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < total;
       t += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t r = (uint32_t)(t % M), s = (uint32_t)(t / M);
    if ((r / 8) < (s / 8)) continue;  // only tiles with r-tile >= s-tile were written
    double acc = 0.0;
    for (uint32_t k = 0; k < n_chunks; ++k) acc += partial[(uint64_t)k * total + t];
    G[t] = acc;
    G[s + (uint64_t)r * M] = acc;
  }
}

// out[l] = sum of the partials of leaf l's chunks [c0[l], c1[l]) in chunk order
// (as reduce_partials), mirrored to the upper triangle
__global__ void reduce_leaf_partials(const double* __restrict__ partial, const uint32_t* __restrict__ c0,
                                     const uint32_t* __restrict__ c1, uint32_t M, double* __restrict__ out) {
  const uint64_t total = (uint64_t)M * M;
  const uint32_t l = blockIdx.y;
  double* G = out + (uint64_t)l * total;
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < total;
       t += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t r = (uint32_t)(t % M), s = (uint32_t)(t / M);
    if ((r / 8) < (s / 8)) continue;
    double acc = 0.0;
    for (uint32_t k = c0[l]; k < c1[l]; ++k) acc += partial[(uint64_t)k * total + t];
    G[t] = acc;
    G[s + (uint64_t)r * M] = acc;
  }
}

// one level of the pairwise tree (csrc/rk_pipeline.cu forest_reduce's shape):
// out node i = in node 2i + in node 2i+1; an odd last node is carried up unchanged
__global__ void add_pairs_to(const double* __restrict__ in, double* __restrict__ out, uint64_t n_nodes,
                             uint64_t mm) {
  const uint64_t half = n_nodes / 2, out_nodes = (n_nodes + 1) / 2;
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < out_nodes * mm;
       t += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t i = t / mm, e = t - i * mm;
    out[t] = i < half ? in[2 * i * mm + e] + in[(2 * i + 1) * mm + e] : in[2 * i * mm + e];
  }
}

// Diagonal ordering of a block's Gram before its Cholesky: position a holds the
// original row perm[a], rows by descending G_ii (stable). The one-sided Jacobi on
// the Cholesky factor of the symmetrically permuted Gram converges in fewer
// sweeps (numpy replay of the tournament on c2 blocks: the slowest of nine
// blocks 11 -> 10 sweeps); the rows of U are un-permuted by the finalize.
__global__ void diag_rank_kernel(const double* __restrict__ G, uint64_t stride, uint32_t M,
                                 uint32_t* __restrict__ perm) {
  __shared__ double sd[1280];
  const uint32_t q = blockIdx.x;
  const double* g = G + q * stride;
  for (uint32_t i = threadIdx.x; i < M; i += blockDim.x) sd[i] = g[i + (uint64_t)i * M];
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < M; i += blockDim.x) {
    const double di = sd[i];
    uint32_t rnk = 0;
    for (uint32_t j = 0; j < M; ++j) {
      const double dj = sd[j];
      rnk += (dj > di) || (dj == di && j < i);
    }
    perm[(uint64_t)q * M + rnk] = i;
  }
}

// Gp[a + b M] = G[perm[a] + perm[b] M] for the M x M part of each slot
__global__ void diag_gather_kernel(const double* __restrict__ G, uint64_t stride, uint32_t M,
                                   const uint32_t* __restrict__ perm, double* __restrict__ Gp) {
  const uint32_t q = blockIdx.y;
  const double* g = G + q * stride;
  double* gp = Gp + q * stride;
  const uint32_t* pq = perm + (uint64_t)q * M;
  const uint64_t mm = (uint64_t)M * M;
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < mm; t += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t b = (uint32_t)(t / M), a = (uint32_t)(t - (uint64_t)b * M);
    gp[t] = g[pq[a] + (uint64_t)pq[b] * M];
  }
}

// ---------------------------------------------------------------------------
// blocked right-looking Cholesky, one CTA per matrix, in place on the lower
// triangle (column-major, ld M). On exit the strict upper triangle is zeroed so
// the matrix is W = L. status[i]: 0 ok, 1 non-positive pivot.

constexpr int kCT = 256;

#ifdef RK_EXPERIMENTS  // not kept (measured): the right-looking kernel, RK_CHOL=r
// kCB: panel width (32; 16 for tall matrices, so the M x kCB panel fits shared memory)
template <int kCB>
__global__ void __launch_bounds__(kCT, 1) cholesky_kernel(double* const* __restrict__ mats, uint32_t M,
                                                          uint32_t* __restrict__ status,
                                                          double* __restrict__ diag_ratio) {
  extern __shared__ __align__(16) double sm[];
  double* D = sm;                   // kCB x kCB diagonal block (column-major)
  double* Lp = D + kCB * kCB;       // (M) x kCB panel rows below the diagonal block (column-major, ld M)
  __shared__ int s_bad;
  __shared__ double s_dmin, s_dmax;
  __shared__ double Dinv[kCB];
  double* A = mats[blockIdx.x];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) { s_bad = 0; s_dmin = INFINITY; s_dmax = 0.0; }
  __syncthreads();
  for (uint32_t k0 = 0; k0 < M; k0 += kCB) {
    const uint32_t nb = min((uint32_t)kCB, M - k0);
    // 1. factor the diagonal block (one warp, column by column)
    for (uint32_t t = tid; t < nb * nb; t += kCT) {
      const uint32_t i = t % nb, j = t / nb;
      D[i + j * kCB] = (i >= j) ? __ldcg(A + (k0 + i) + (uint64_t)(k0 + j) * M) : 0.0;
    }
    __syncthreads();
    if (warp == 0) {
      // lane i holds row i of the diagonal block in registers; column j: pivot by
      // shuffle, scale, rank-1 update of the rows below (no shared-memory round trips)
      double r[kCB];
#pragma unroll
      for (int c = 0; c < kCB; ++c) r[c] = (lane < (int)nb && c < (int)nb) ? D[lane + c * kCB] : 0.0;
      bool bad = false;
      double dmin = INFINITY, dmax = 0.0;
#pragma unroll
      for (int j = 0; j < kCB; ++j) {
        if (j < (int)nb) {
          double piv = __shfl_sync(0xffffffffu, r[j], j);
          if (!(piv > 0.0)) {
            bad = true;
            piv = 1.0;
          }
          const double inv = rsqrt(piv);
          const double ljj = piv * inv;
          dmin = fmin(dmin, ljj);
          dmax = fmax(dmax, ljj);
          const double l = lane > j ? r[j] * inv : (lane == j ? ljj : 0.0);
          if (lane >= j) r[j] = l;
#pragma unroll
          for (int c = j + 1; c < kCB; ++c) {
            const double lcj = __shfl_sync(0xffffffffu, l, c);
            if (lane >= c) r[c] -= l * lcj;
          }
        }
      }
      if (lane < (int)nb) {
#pragma unroll
        for (int c = 0; c < kCB; ++c)
          if (c < (int)nb) D[lane + c * kCB] = lane >= c ? r[c] : 0.0;
      }
      if (lane == 0) {
        if (bad) s_bad = 1;
        s_dmin = fmin(s_dmin, dmin);
        s_dmax = fmax(s_dmax, dmax);
      }
    }
    __syncthreads();
    if (s_bad) break;
    // write the factored diagonal block back (zero above)
    for (uint32_t t = tid; t < nb * nb; t += kCT) {
      const uint32_t i = t % nb, j = t / nb;
      A[(k0 + i) + (uint64_t)(k0 + j) * M] = (i >= j) ? D[i + j * kCB] : 0.0;
    }
    // 2. panel below: L21 = A21 L11^{-T}; row-wise forward substitution (thread per row)
    const uint32_t below = M - k0 - nb;
    if (tid < kCB) Dinv[tid] = tid < (int)nb ? 1.0 / D[tid + tid * kCB] : 0.0;
    __syncthreads();
    for (uint32_t rr = tid; rr < below; rr += kCT) {
      const uint32_t i = k0 + nb + rr;
      double x[kCB];
#pragma unroll
      for (int j = 0; j < kCB; ++j) x[j] = (j < (int)nb) ? __ldcg(A + i + (uint64_t)(k0 + j) * M) : 0.0;
#pragma unroll
      for (int j = 0; j < kCB; ++j) {
        if (j < (int)nb) {
          double v = x[j];
          for (int q = 0; q < j; ++q) v -= x[q] * D[j + q * kCB];
          x[j] = v * Dinv[j];
        }
      }
#pragma unroll
      for (int j = 0; j < kCB; ++j)
        if (j < (int)nb) {
          A[i + (uint64_t)(k0 + j) * M] = x[j];
          Lp[rr + (uint64_t)j * M] = x[j];
        }
    }
    __syncthreads();
    // 3. trailing SYRK: A22 -= L21 L21^T on 8x8 tiles of the lower triangle (DMMA)
    const uint32_t nt = (below + 7) / 8;
    const int lr = lane >> 2, lc = lane & 3;
    // a warp owns tile rows ti = warp, warp + 8, ...: its A fragments (L21 rows of
    // the tile row) are loaded once and reused across the row's tiles tj <= ti,
    // kTB tiles at a time so their C loads (L2 round trips) are in flight together
    constexpr int kTB = 4;
    for (uint32_t ti = warp; ti < nt; ti += kCT / 32) {
      const uint32_t r = ti * 8 + lr;
      double af[kCB / 4];
#pragma unroll
      for (int kk = 0; kk < kCB / 4; ++kk) {
        const int q = 4 * kk + lc;
        af[kk] = (r < below && q < (int)nb) ? Lp[r + (uint64_t)q * M] : 0.0;
      }
      for (uint32_t tj = 0; tj <= ti; tj += kTB) {
        double d0[kTB], d1[kTB];
        double* cp[kTB];
        bool ok0[kTB], ok1[kTB];
#pragma unroll
        for (int u = 0; u < kTB; ++u) {
          const uint32_t t = tj + u, s0 = t * 8 + 2 * lc;
          cp[u] = A + (k0 + nb + r) + (uint64_t)(k0 + nb + s0) * M;
          const bool live = t <= ti && r < below;
          ok0[u] = live && s0 < below;
          ok1[u] = live && s0 + 1 < below;
          d0[u] = ok0[u] ? -__ldcg(cp[u]) : 0.0;
          d1[u] = ok1[u] ? -__ldcg(cp[u] + M) : 0.0;
        }
#pragma unroll
        for (int kk = 0; kk < kCB / 4; ++kk) {
          const int q = 4 * kk + lc;
#pragma unroll
          for (int u = 0; u < kTB; ++u) {
            const uint32_t sb = (tj + u) * 8 + lr;
            const double bv = (sb < below && q < (int)nb) ? Lp[sb + (uint64_t)q * M] : 0.0;
            dmma(d0[u], d1[u], af[kk], bv);  // accumulates -C + L L^T
          }
        }
#pragma unroll
        for (int u = 0; u < kTB; ++u) {
          if (ok0[u]) *cp[u] = -d0[u];
          if (ok1[u]) cp[u][M] = -d1[u];
        }
      }
    }
    __syncthreads();
  }
  // zero the strict upper triangle: W = L
  if (!s_bad)
    for (uint64_t t = tid; t < (uint64_t)M * M; t += kCT) {
      const uint32_t i = (uint32_t)(t % M), j = (uint32_t)(t / M);
      if (i < j) A[t] = 0.0;
    }
  if (tid == 0) {
    status[blockIdx.x] = s_bad ? 1u : 0u;
    diag_ratio[blockIdx.x] = s_bad ? INFINITY : s_dmax / s_dmin;
  }
}
#endif  // RK_EXPERIMENTS

// the nb x nb diagonal block at P (column-major, ld ldp) factored in place by one
// warp: lane i holds row i in registers. FP64 latency sets the speed here (DFMA
// 23 cycles, rsqrt 78, a double shuffle 49 on the B200 -- tools/probe_latency.cu),
// so the critical path goes through the pivot lane's own registers: after column
// j, lane j+1 updates its diagonal entry and takes its rsqrt before the other
// rank-1 updates, and only the reciprocal pivot is broadcast (32x32: 11.9k cycles
// vs 26k for the textbook order). Dinv[j] = 1 / L_jj.
template <int kCB, bool FULL>
__device__ __forceinline__ void factor_diag(double* P, uint32_t ldp, uint32_t nb_rt, int lane, double* Dinv,
                                            int* s_bad, double* s_dmin, double* s_dmax) {
  const uint32_t nb = FULL ? (uint32_t)kCB : nb_rt;  // FULL: no per-column guards
  double rg[kCB];
#pragma unroll
  for (int c = 0; c < kCB; ++c) rg[c] = (lane < (int)nb && c < (int)nb) ? P[lane + c * ldp] : 0.0;
  bool bad = false;
  double dmin = INFINITY, dmax = 0.0;
  // lane j's candidate pivot and its reciprocal square root
  auto pivot = [&](double d, double& inv) {
    const bool ok = d > 0.0;
    inv = rsqrt(ok ? d : 1.0);
    return ok;
  };
  double inv_mine;
  bool ok_mine = pivot(rg[0], inv_mine);
#pragma unroll
  for (int j = 0; j < kCB; ++j) {
    if (j < (int)nb) {
      const double inv = __shfl_sync(0xffffffffu, inv_mine, j);
      const double l = lane >= j ? rg[j] * inv : 0.0;
      const bool me = lane == j;
      bad = bad || (me && !ok_mine);
      dmin = me ? fmin(dmin, l) : dmin;
      dmax = me ? fmax(dmax, l) : dmax;
      if (me) Dinv[j] = inv;
      rg[j] = l;
      if (j + 1 < kCB) {
        ok_mine = pivot(rg[j + 1] - l * l, inv_mine);  // valid in lane j + 1
#pragma unroll
        for (int c = j + 1; c < kCB; ++c) {
          const double lcj = __shfl_sync(0xffffffffu, l, c);
          if (lane >= c) rg[c] -= l * lcj;
        }
      }
    }
  }
  if (lane < (int)nb) {
#pragma unroll
    for (int c = 0; c < kCB; ++c)
      if (c < (int)nb) P[lane + c * ldp] = lane >= c ? rg[c] : 0.0;
  }
  for (int o = 16; o; o >>= 1) {
    dmin = fmin(dmin, __shfl_xor_sync(0xffffffffu, dmin, o));
    dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
  }
  bad = __any_sync(0xffffffffu, bad);
  if (lane == 0) {
    if (bad) *s_bad = 1;
    *s_dmin = fmin(*s_dmin, dmin);
    *s_dmax = fmax(*s_dmax, dmax);
  }
  __syncwarp();
}

// S[i + c ld] = src[i + c M] for i < rows, c < ncols (<= kCB): a thread's loads of
// all kCB columns are issued before its stores (one L2 round trip per 256 rows, not
// one per column: the per-column loop serialized 32 round trips per chunk and was
// half of the kernel's time)
template <int kCB>
__device__ __forceinline__ void stage_cols(double* S, uint32_t ld, const double* src, uint32_t M, uint32_t rows,
                                           uint32_t ncols, int tid) {
  for (uint32_t i = tid; i < rows; i += kCT) {
    double v[kCB];
#pragma unroll
    for (int c = 0; c < kCB; ++c) v[c] = c < (int)ncols ? src[i + (uint64_t)c * M] : 0.0;
#pragma unroll
    for (int c = 0; c < kCB; ++c)
      if (c < (int)ncols) S[i + c * ld] = v[c];
  }
}

// Left-looking variant: panel by panel (kCB columns), the update of the panel by
// the finished columns, P -= L[k0:, :k0] L[k0:k0+kCB, :k0]^T, runs as a DMMA GEMM
// over K chunks of kCB columns staged in shared memory with coalesced loads (one
// L2 round trip per chunk for the whole CTA), the accumulators in registers (warp
// w owns tile rows w, w + 8, ...; at most NP of them). Then the panel is loaded
// into the same buffer, the accumulators subtracted, the diagonal block factored
// in registers (factor_diag), the rows below solved against it and the panel
// written back once (zeros above the diagonal). No read-modify-write passes over
// the trailing matrix. Same status / ratio outputs as cholesky_kernel.
template <int kCB>
__host__ __device__ constexpr uint32_t ll_ld(uint32_t rows) {
  // >= rows, == 4 (mod 16): the DMMA fragment reads (lr + lc ld) hit distinct banks
  return ((rows + 11) / 16) * 16 + 4;
}

#ifndef CHOL_PROBE
#define CHOL_PROBE 0
#endif
template <int kCB, int NP>
__global__ void __launch_bounds__(kCT, 1) cholesky_ll_kernel(double* const* __restrict__ mats, uint32_t M,
                                                             uint32_t* __restrict__ status,
                                                             double* __restrict__ diag_ratio) {
  extern __shared__ __align__(16) double sm[];
  double* S = sm;  // rows_p x kCB, column-major, ld ll_ld(rows_p)
  __shared__ int s_bad;
  __shared__ double s_dmin, s_dmax;
  __shared__ double Dinv[kCB];
  double* A = mats[blockIdx.x];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int lr = lane >> 2, lc = lane & 3;
  constexpr int kW = kCT / 32;
  if (tid == 0) { s_bad = 0; s_dmin = INFINITY; s_dmax = 0.0; }
  long long tm[6] = {0, 0, 0, 0, 0, 0};
  long long tcl = clock64();
  auto tick = [&](int k) {
    if (CHOL_PROBE) {
      const long long t = clock64();
      tm[k] += t - tcl;
      tcl = t;
    }
  };
  for (uint32_t k0 = 0; k0 < M; k0 += kCB) {
    const uint32_t nb = min((uint32_t)kCB, M - k0), rows_p = M - k0;
    const uint32_t ld = ll_ld<kCB>(rows_p);
    const uint32_t TR = (rows_p + 7) / 8;
    double acc[NP][kCB / 8][2];
#pragma unroll
    for (int pp = 0; pp < NP; ++pp)
#pragma unroll
      for (int u = 0; u < kCB / 8; ++u) acc[pp][u][0] = acc[pp][u][1] = 0.0;
    // GEMM over the finished columns, kCB at a time
    for (uint32_t kc = 0; kc < k0; kc += kCB) {
      __syncthreads();  // previous users of S are done
      stage_cols<kCB>(S, ld, A + k0 + (uint64_t)kc * M, M, rows_p, kCB, tid);
      __syncthreads();
#pragma unroll
      for (int pp = 0; pp < NP; ++pp) {
        const uint32_t tr = warp + kW * pp;
        if (tr < TR) {
          const uint32_t ia = tr * 8 + lr;
#pragma unroll
          for (int kk = 0; kk < kCB; kk += 4) {
            const uint32_t q = kk + lc;
            const double av = ia < rows_p ? S[ia + q * ld] : 0.0;
#pragma unroll
            for (int u = 0; u < kCB / 8; ++u) {
              const uint32_t ib = u * 8 + lr;
              const double bv = ib < nb ? S[ib + q * ld] : 0.0;
              dmma(acc[pp][u][0], acc[pp][u][1], av, bv);
            }
          }
        }
      }
    }
    __syncthreads();
    tick(0);
    // the panel minus the update
    stage_cols<kCB>(S, ld, A + k0 + (uint64_t)k0 * M, M, rows_p, nb, tid);
    __syncthreads();
    if (k0 > 0) {
#pragma unroll
      for (int pp = 0; pp < NP; ++pp) {
        const uint32_t tr = warp + kW * pp;
        const uint32_t i = tr * 8 + lr;
        if (tr < TR && i < rows_p) {
#pragma unroll
          for (int u = 0; u < kCB / 8; ++u) {
            const uint32_t j = u * 8 + 2 * lc;
            if (j < nb) S[i + j * ld] -= acc[pp][u][0];
            if (j + 1 < nb) S[i + (j + 1) * ld] -= acc[pp][u][1];
          }
        }
      }
      __syncthreads();
    }
    tick(1);
    if (warp == 0) {
      if (nb == kCB) factor_diag<kCB, true>(S, ld, nb, lane, Dinv, &s_bad, &s_dmin, &s_dmax);
      else factor_diag<kCB, false>(S, ld, nb, lane, Dinv, &s_bad, &s_dmin, &s_dmax);
    }
    __syncthreads();
    tick(2);
    if (s_bad) break;
    // rows below: x = p L11^{-T} (forward substitution, thread per row)
    for (uint32_t i = nb + tid; i < rows_p; i += kCT) {
      double x[kCB];
#pragma unroll
      for (int j = 0; j < kCB; ++j) x[j] = j < (int)nb ? S[i + j * ld] : 0.0;
      // right-looking: x_j is final after the scaling, its updates of x_c (c > j)
      // are independent of each other (a 2-op chain per column, not j ops)
#pragma unroll
      for (int j = 0; j < kCB; ++j) {
        if (j < (int)nb) {
          x[j] *= Dinv[j];
#pragma unroll
          for (int c = j + 1; c < kCB; ++c) x[c] -= x[j] * S[c + j * ld];
        }
      }
#pragma unroll
      for (int j = 0; j < kCB; ++j)
        if (j < (int)nb) S[i + j * ld] = x[j];
    }
    __syncthreads();
    tick(3);
    // write the finished columns (zeros above the diagonal)
#pragma unroll 8
    for (int j = 0; j < kCB; ++j) {
      if (j >= (int)nb) break;
      double* dst = A + (uint64_t)(k0 + j) * M;
      for (uint32_t i = tid; i < M; i += kCT) dst[i] = i < k0 ? 0.0 : S[(i - k0) + j * ld];
    }
  }
  tick(4);
  if (CHOL_PROBE && tid == 0 && blockIdx.x == 0)
    printf("[chol] M %u cycles: gemm %lld panel %lld diag %lld trsm %lld writeback %lld\n", M, tm[0], tm[1], tm[2],
           tm[3], tm[4]);
  if (tid == 0) {
    status[blockIdx.x] = s_bad ? 1u : 0u;
    diag_ratio[blockIdx.x] = s_bad ? INFINITY : s_dmax / s_dmin;
  }
}

unsigned grid_for(uint64_t n, unsigned cap = 1u << 20) {
  uint64_t g = ceil_div(n, 256);
  if (g == 0) g = 1;
  if (g > cap) g = cap;
  return (unsigned)g;
}

// split-K SYRK launch: a 32 x 32 block per warp where M allows
static void launch_syrk(const SyrkChunk* d_chunks, uint32_t n_chunks, uint32_t M, double* partial, cudaStream_t s) {
  if (M % 32 == 0 && tuning().syrk_block4) {
    const uint64_t nb = M / 32, warps = nb * (nb + 1) / 2 * n_chunks;
    syrk_records_kernel4<<<grid_for(warps * 32), 256, 0, s>>>(d_chunks, n_chunks, M, partial);
  } else {
    const uint64_t tiles = M / 8, warps = tiles * (tiles + 1) / 2 * n_chunks;
    syrk_records_kernel<<<grid_for(warps * 32), 256, 0, s>>>(d_chunks, n_chunks, M, partial);
  }
  RK_LAUNCH_CHECK();
}


}  // namespace

void sparse_gram(const DevMatrix& m, const Partition& p, uint64_t d_lo, uint64_t nblk, double* G, uint64_t stride,
                 cudaStream_t s) {
  const DevCsr& a = m.csr;
  const uint32_t M = (uint32_t)a.rows;
  if (!M || !nblk) return;
#ifdef RK_EXPERIMENTS
  if (tuning().gram_pairs) {  // the row-pair merge-join kernel (A/B; experiments build)
    const uint64_t total = (uint64_t)M * (M + 1) / 2 * nblk;
    sparse_gram_kernel<<<grid_for(total), 256, 0, s>>>(a.ptr.get(), a.idx.get(), a.val.get(), M, p, d_lo, nblk, G,
                                                       stride);
    RK_LAUNCH_CHECK();
    return;
  }
#endif
  // G is zero on entry (the caller's slot buffer)
  // 64 threads per CTA: one thread per (block, row) is only M x nblk threads
  sparse_gram_rows_kernel<<<grid_for((uint64_t)M * nblk * 4), 64, 0, s>>>(
      a.ptr.get(), a.idx.get(), a.val.get(), m.csc.ptr.get(), m.csc.idx.get(), m.csc.val.get(), M, p, d_lo, nblk, G,
      stride);
  RK_LAUNCH_CHECK();
  mirror_lower<<<grid_for((uint64_t)M * M * nblk), 256, 0, s>>>(G, stride, M, nblk);
  RK_LAUNCH_CHECK();
}

namespace {
// eff[rec] = 1 + the last column of record rec holding a nonzero (0: none). The
// finalize writes a record's columns in descending sigma, and a column of sigma 0
// is exactly zero, so the columns past eff are zero: rows of P^T that change
// neither P P^T nor its R factor (c3: ~385 of every block's 512). One CTA per record.
__global__ void record_effective_cols(const double* payload, const uint64_t* off, const uint32_t* kept, uint32_t n,
                                      uint32_t r0, uint32_t* eff) {
  __shared__ uint32_t s_max;
  const uint32_t rec = r0 + blockIdx.x, k = kept[rec];
  if (threadIdx.x == 0) s_max = 0;
  __syncthreads();
  const double* src = payload + off[rec];
  uint32_t m = 0;
  for (uint64_t t = threadIdx.x; t < (uint64_t)n * k; t += blockDim.x)
    if (src[t] != 0.0) m = max(m, (uint32_t)(t % k) + 1);
  if (m) atomicMax(&s_max, m);
  __syncthreads();
  if (threadIdx.x == 0) eff[rec] = s_max;
}
}  // namespace

std::vector<uint32_t> record_eff_cols(const double* payload, const std::vector<uint64_t>& offset,
                                      const std::vector<uint32_t>& kept, uint32_t M, uint32_t r_lo, uint32_t r_hi,
                                      cudaStream_t s, const std::vector<uint32_t>* hint) {
  std::vector<uint32_t> eff(kept.size(), 0);
  if (r_hi <= r_lo || !M) return eff;
  if (hint && hint->size() == kept.size()) {  // the block stage knows: no scan of the records
    for (uint32_t d = r_lo; d < r_hi; ++d) eff[d] = std::min((*hint)[d], kept[d]);
    return eff;
  }
  DBuf<uint64_t> doff(offset.size(), s);
  DBuf<uint32_t> dkept(kept.size(), s), deff(kept.size(), s);
  to_device(doff.get(), offset.data(), offset.size(), s);
  to_device(dkept.get(), kept.data(), kept.size(), s);
  deff.zero();
  record_effective_cols<<<r_hi - r_lo, 256, 0, s>>>(payload, doff.get(), dkept.get(), M, r_lo, deff.get());
  RK_LAUNCH_CHECK();
  to_host(eff, deff.get(), kept.size(), s);
  sync(s);
  return eff;
}

void records_gram(const double* payload, const std::vector<uint64_t>& offset, const std::vector<uint32_t>& kept,
                  uint32_t M, double* G, cudaStream_t s, const std::vector<uint32_t>* eff_hint) {
  if (M % 8) fail(RK_RUNTIME, "records_gram: M must be a multiple of 8");
  // split-K chunks of at most kChunk columns of one record; each chunk has an
  // M x M partial, so the chunk width grows with M to bound that buffer (c4:
  // 1024 records x 1024 columns -> 1024 partials of 8 MiB, not 4096)
  const uint32_t kChunk = M <= 256 ? 256u : 1024u;
  // only each record's leading nonzero columns (record_eff_cols): the zero ones add
  // nothing to P P^T (c3: ~385 of 512 per record)
  const std::vector<uint32_t> eff = record_eff_cols(payload, offset, kept, M, 0, (uint32_t)kept.size(), s, eff_hint);
  std::vector<SyrkChunk> ch;
  for (size_t d = 0; d < kept.size(); ++d) {
    if (!eff[d]) continue;
    for (uint32_t j0 = 0; j0 < eff[d]; j0 += kChunk)
      ch.push_back({payload + offset[d], kept[d], j0, std::min<uint32_t>(eff[d], j0 + kChunk)});
  }
  if (ch.empty()) {
    RK_CUDA_CHECK(cudaMemsetAsync(G, 0, sizeof(double) * M * M, s));
    return;
  }
  DBuf<SyrkChunk> dch(ch.size(), s);
  to_device(dch.get(), ch.data(), ch.size(), s);
  DBuf<double> partial(ch.size() * (uint64_t)M * M, s);
  launch_syrk(dch.get(), (uint32_t)ch.size(), M, partial.get(), s);
  RK_CUDA_CHECK(cudaMemsetAsync(G, 0, sizeof(double) * M * M, s));
  reduce_partials<<<grid_for((uint64_t)M * M), 256, 0, s>>>(partial.get(), (uint32_t)ch.size(), M, G);
  RK_LAUNCH_CHECK();
  sync(s);  // host chunk list
}

void diag_order(const double* G, uint64_t stride, uint32_t M, uint64_t nb, uint32_t* perm, double* Gp,
                cudaStream_t s) {
  if (!nb || !M) return;
  if (M > 1280) fail(RK_RUNTIME, "diag_order: M too large");
  diag_rank_kernel<<<(unsigned)nb, 256, 0, s>>>(G, stride, M, perm);
  RK_LAUNCH_CHECK();
  const uint64_t mm = (uint64_t)M * M;
  diag_gather_kernel<<<dim3((unsigned)std::min<uint64_t>(ceil_div(mm, 256), 64), (unsigned)nb), 256, 0, s>>>(
      G, stride, M, perm, Gp);
  RK_LAUNCH_CHECK();
}

bool diag_order_enabled() { return tuning().diag_order; }

void gram_tree_sum(double* mats, uint64_t n, uint32_t M, cudaStream_t s) {
  const uint64_t mm = (uint64_t)M * M;
  // level by level, ping-pong between mats and a scratch buffer
  if (n <= 1) return;
  DBuf<double> tmp(((n + 1) / 2) * mm, s);
  double* src = mats;
  double* dst = tmp.get();
  while (n > 1) {
    const uint64_t out_nodes = (n + 1) / 2;
    add_pairs_to<<<grid_for(out_nodes * mm), 256, 0, s>>>(src, dst, n, mm);
    RK_LAUNCH_CHECK();
    n = out_nodes;
    std::swap(src, dst);
  }
  if (src != mats) RK_CUDA_CHECK(cudaMemcpyAsync(mats, src, sizeof(double) * mm, cudaMemcpyDeviceToDevice, s));
}

void leaf_gram_tree(const double* payload, const std::vector<uint64_t>& offset, const std::vector<uint32_t>& kept,
                    uint32_t M, const std::vector<std::pair<uint32_t, uint32_t>>& leaves, double* G, cudaStream_t s,
                    const std::vector<uint32_t>* eff_hint) {
  if (M % 8) fail(RK_RUNTIME, "leaf_gram_tree: M must be a multiple of 8");
  const uint64_t mm = (uint64_t)M * M, L = leaves.size();
  if (L == 0) {
    RK_CUDA_CHECK(cudaMemsetAsync(G, 0, sizeof(double) * mm, s));
    return;
  }
  std::vector<SyrkChunk> ch;
  std::vector<uint32_t> c0(L), c1(L);
  // each record's leading nonzero columns only (record_eff_cols), as records_gram
  const std::vector<uint32_t> eff =
      record_eff_cols(payload, offset, kept, M, leaves.front().first, leaves.back().second, s, eff_hint);
  for (uint64_t l = 0; l < L; ++l) {
    c0[l] = (uint32_t)ch.size();
    for (uint32_t d = leaves[l].first; d < leaves[l].second; ++d) {
      if (!eff[d]) continue;
      for (uint32_t j0 = 0; j0 < eff[d]; j0 += 256)
        ch.push_back({payload + offset[d], kept[d], j0, std::min<uint32_t>(eff[d], j0 + 256)});
    }
    c1[l] = (uint32_t)ch.size();
  }
  DBuf<double> leafG(L * mm, s);
  if (!ch.empty()) {
    DBuf<SyrkChunk> dch(ch.size(), s);
    to_device(dch.get(), ch.data(), ch.size(), s);
    DBuf<double> partial(ch.size() * mm, s);
    launch_syrk(dch.get(), (uint32_t)ch.size(), M, partial.get(), s);
    DBuf<uint32_t> d0(L, s), d1(L, s);
    to_device(d0.get(), c0.data(), L, s);
    to_device(d1.get(), c1.data(), L, s);
    reduce_leaf_partials<<<dim3(grid_for(mm, 1u << 12), (unsigned)L), 256, 0, s>>>(partial.get(), d0.get(), d1.get(),
                                                                                  M, leafG.get());
    RK_LAUNCH_CHECK();
    sync(s);  // chunk lists are host memory
  } else {
    leafG.zero();
  }
  gram_tree_sum(leafG.get(), L, M, s);
  RK_CUDA_CHECK(cudaMemcpyAsync(G, leafG.get(), sizeof(double) * mm, cudaMemcpyDeviceToDevice, s));
}

void cholesky_batched(double* const* d_mats, uint32_t n_mats, uint32_t M, uint32_t* d_status, double* d_ratio,
                      cudaStream_t s) {
  if (!n_mats) return;
#ifdef RK_EXPERIMENTS
  auto launch = [&](auto kern, int cb) {
    const size_t smem = ((size_t)cb * cb + (size_t)M * cb) * sizeof(double);
    if (smem > 200 * 1024) fail(RK_RUNTIME, "cholesky_batched: M too large for the panel buffer");
    RK_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    RK_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    kern<<<n_mats, kCT, smem, s>>>(d_mats, M, d_status, d_ratio);
    RK_LAUNCH_CHECK();
  };
  const bool ll = !tuning().chol_right;  // RK_CHOL=r: the right-looking kernel (A/B; experiments build)
#else
  const bool ll = true;
#endif
  auto launch_ll = [&](auto kern, int cb) {
    const size_t smem = (size_t)ll_ld<16>(M) * cb * sizeof(double);
    RK_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<n_mats, kCT, smem, s>>>(d_mats, M, d_status, d_ratio);
    RK_LAUNCH_CHECK();
  };
  // NP = tile rows per warp = ceil(M / 64)
  if (ll && M <= 256) {
    launch_ll(cholesky_ll_kernel<32, 4>, 32);
  } else if (ll && M <= 512) {
    launch_ll(cholesky_ll_kernel<32, 8>, 32);
  } else if (ll && M <= 1024) {
    launch_ll(cholesky_ll_kernel<16, 16>, 16);
  } else if (ll && M <= 1280) {
    launch_ll(cholesky_ll_kernel<16, 20>, 16);
  }
#ifdef RK_EXPERIMENTS
  else if (M <= 640) {
    launch(cholesky_kernel<32>, 32);
  } else {
    launch(cholesky_kernel<16>, 16);
  }
#else
  else {
    fail(RK_RUNTIME, "cholesky_batched: M above the panel cap");
  }
#endif
}

uint32_t cholesky_max_rows() { return 1280; }  // the panel buffer (M x 16 doubles) must fit shared memory

bool gram_route_enabled() { return !tuning().householder_only; }

double kappa_max(uint32_t M) {
  // every sigma moves by < 3e-11 relative when M eps kappa^2 / 2 < 3e-11
  const double eps = 1.1102230246251565e-16;
  return sqrt(6e-11 / ((double)std::max<uint32_t>(M, 1) * eps));
}

}  // namespace rk
