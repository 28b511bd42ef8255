// rk_spmm.cu -- right-vector recovery V = A^T U Sigma^-1 (reference:
// recover_right_vectors, proj/src/proxy.cpp:48-72).
//
// One warp per column c of A (= row c of V): the column's CSC entries are
// visited in ascending row order -- the order in which the reference's
// (row, col)-sorted entry loop accumulates into V(c, :) -- and every product
// and sum uses round-to-nearest without contraction, then the row is scaled by
// 1/sigma. Given identical U and sigma the result is bit-identical to the
// reference. U's retained columns are gathered once into a compact M x r table
// (L2-resident); V rows are written once, 16-byte vectorised, with streaming
// stores: the kernel is bound by the 8*N*r-byte V write.
#include <cstdlib>

#include "rk_internal.cuh"

namespace rk {
namespace {

__global__ void gather_u(const double* u, uint32_t rows, uint32_t u_cols, const uint32_t* retained, uint32_t r,
                         const double* sigma, double* u_ret, double* inv) {
  const uint64_t total = (uint64_t)rows * r;
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < total;
       t += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t i = t / r, jj = t % r;
    u_ret[t] = u[i * u_cols + retained[jj]];
    if (i == 0) inv[jj] = __ddiv_rn(1.0, sigma[retained[jj]]);
  }
}

// r even: each lane owns column pairs (2*lane + 64*k, +1)
template <bool kPairs>
__global__ void __launch_bounds__(256) spmm_kernel(const uint64_t* __restrict__ col_ptr,
                                                   const uint32_t* __restrict__ row_idx,
                                                   const double* __restrict__ val, const double* __restrict__ u_ret,
                                                   const double* __restrict__ inv, uint32_t r, uint64_t col_lo,
                                                   uint64_t col_hi, double* __restrict__ v) {
  constexpr int kMax = 16;  // up to 32 * kMax (pairs: 64 * kMax/2 ... ) columns in registers per pass
  const int lane = threadIdx.x & 31;
  const uint64_t warp0 = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t c = col_lo + warp0; c < col_hi; c += nwarps) {
    const uint64_t e0 = col_ptr[c], e1 = col_ptr[c + 1];
    double* vrow = v + (c - col_lo) * r;
    if (kPairs) {
      for (uint32_t base = 0; base < r; base += 64 * (kMax / 2)) {
        double2 acc[kMax / 2];
#pragma unroll
        for (int k = 0; k < kMax / 2; ++k) acc[k] = make_double2(0.0, 0.0);
        for (uint64_t e = e0; e < e1; ++e) {
          const double x = val[e];
          const double2* ur = reinterpret_cast<const double2*>(u_ret + (uint64_t)row_idx[e] * r);
#pragma unroll
          for (int k = 0; k < kMax / 2; ++k) {
            const uint32_t j = base + 64 * k + 2 * lane;
            if (j < r) {
              const double2 uu = ur[j / 2];
              acc[k].x = __dadd_rn(acc[k].x, __dmul_rn(x, uu.x));
              acc[k].y = __dadd_rn(acc[k].y, __dmul_rn(x, uu.y));
            }
          }
        }
#pragma unroll
        for (int k = 0; k < kMax / 2; ++k) {
          const uint32_t j = base + 64 * k + 2 * lane;
          if (j < r) {
            double2 o;
            o.x = __dmul_rn(acc[k].x, inv[j]);
            o.y = __dmul_rn(acc[k].y, inv[j + 1]);
            __stcs(reinterpret_cast<double2*>(vrow + j), o);
          }
        }
      }
    } else {
      for (uint32_t base = 0; base < r; base += 32 * kMax) {
        double acc[kMax];
#pragma unroll
        for (int k = 0; k < kMax; ++k) acc[k] = 0.0;
        for (uint64_t e = e0; e < e1; ++e) {
          const double x = val[e];
          const double* ur = u_ret + (uint64_t)row_idx[e] * r;
#pragma unroll
          for (int k = 0; k < kMax; ++k) {
            const uint32_t j = base + 32 * k + lane;
            if (j < r) acc[k] = __dadd_rn(acc[k], __dmul_rn(x, ur[j]));
          }
        }
#pragma unroll
        for (int k = 0; k < kMax; ++k) {
          const uint32_t j = base + 32 * k + lane;
          if (j < r) __stcs(vrow + j, __dmul_rn(acc[k], inv[j]));
        }
      }
    }
  }
}

// Half a warp per column (two columns per warp in flight), r % 32 == 0 and
// r <= 32 * kH (used for r <= 256): lane l of a half owns the double pairs 2 l + 32 k. Twice the
// columns' load chains (col_ptr -> entries -> U rows) in flight per warp of the
// one-warp-per-column kernel; same arithmetic and entry order, so V is the same
// bits.
template <int kH>
__global__ void __launch_bounds__(256) spmm_half_kernel(const uint64_t* __restrict__ col_ptr,
                                                        const uint32_t* __restrict__ row_idx,
                                                        const double* __restrict__ val,
                                                        const double* __restrict__ u_ret,
                                                        const double* __restrict__ inv, uint32_t r, uint64_t col_lo,
                                                        uint64_t col_hi, double* __restrict__ v) {
  const int lane = threadIdx.x & 31, half = lane >> 4, l = lane & 15;
  const uint64_t warp0 = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t c0 = col_lo + 2 * warp0; c0 < col_hi; c0 += 2 * nwarps) {
    const uint64_t c = c0 + half;
    const bool live = c < col_hi;
    const uint64_t e0 = live ? col_ptr[c] : 0, e1 = live ? col_ptr[c + 1] : 0;
    double2 acc[kH];
#pragma unroll
    for (int k = 0; k < kH; ++k) acc[k] = make_double2(0.0, 0.0);
    for (uint64_t e = e0; e < e1; ++e) {
      const double x = val[e];
      const double2* ur = reinterpret_cast<const double2*>(u_ret + (uint64_t)row_idx[e] * r);
#pragma unroll
      for (int k = 0; k < kH; ++k) {
        const uint32_t j = 32 * k + 2 * l;
        if (j < r) {
          const double2 uu = ur[j / 2];
          acc[k].x = __dadd_rn(acc[k].x, __dmul_rn(x, uu.x));
          acc[k].y = __dadd_rn(acc[k].y, __dmul_rn(x, uu.y));
        }
      }
    }
    if (live) {
      double* vrow = v + (c - col_lo) * r;
#pragma unroll
      for (int k = 0; k < kH; ++k) {
        const uint32_t j = 32 * k + 2 * l;
        if (j < r) {
          double2 o;
          o.x = __dmul_rn(acc[k].x, inv[j]);
          o.y = __dmul_rn(acc[k].y, inv[j + 1]);
          __stcs(reinterpret_cast<double2*>(vrow + j), o);
        }
      }
    }
  }
}

// The warp-per-column kernel with V's rows leaving through the TMA engine: a warp
// accumulates its column's V row (r doubles, r even, r * 8 <= kTmaRowBytes) in
// registers, writes it to a per-warp staging row in shared memory, and one lane
// issues a bulk copy shared -> global (cp.async.bulk, the Blackwell TMA's 1-D mode):
// whole 16-byte-aligned rows go out as bulk transactions instead of 32 x 16 B store
// instructions per 512 B, and the warp moves on while the copy drains. Same
// arithmetic and entry order as spmm_kernel: V is the same bits.
constexpr int kTmaRowBytes = 4096;

// every writing thread fences its generic-proxy smem writes for the async proxy
// (fence_for_bulk), the warp synchronises, then one lane issues the copy
__device__ __forceinline__ void fence_for_bulk() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void bulk_store_row(double* g, const double* s, uint32_t bytes) {
  const uint32_t sa = (uint32_t)__cvta_generic_to_shared(s);
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(g), "r"(sa), "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

__global__ void __launch_bounds__(256) spmm_tma_kernel(const uint64_t* __restrict__ col_ptr,
                                                       const uint32_t* __restrict__ row_idx,
                                                       const double* __restrict__ val,
                                                       const double* __restrict__ u_ret,
                                                       const double* __restrict__ inv, uint32_t r, uint64_t col_lo,
                                                       uint64_t col_hi, double* __restrict__ v) {
  constexpr int kMaxPairs = kTmaRowBytes / 16 / 32;  // double2 accumulators per lane (8 at 4 KB rows)
  __shared__ __align__(128) double stage[8][kTmaRowBytes / 8];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double* srow = stage[wid];
  const uint64_t warp0 = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t c = col_lo + warp0; c < col_hi; c += nwarps) {
    const uint64_t e0 = col_ptr[c], e1 = col_ptr[c + 1];
    double2 acc[kMaxPairs];
#pragma unroll
    for (int k = 0; k < kMaxPairs; ++k) acc[k] = make_double2(0.0, 0.0);
    for (uint64_t e = e0; e < e1; ++e) {
      const double x = val[e];
      const double2* ur = reinterpret_cast<const double2*>(u_ret + (uint64_t)row_idx[e] * r);
#pragma unroll
      for (int k = 0; k < kMaxPairs; ++k) {
        const uint32_t j = 64 * k + 2 * lane;
        if (j < r) {
          const double2 uu = ur[j / 2];
          acc[k].x = __dadd_rn(acc[k].x, __dmul_rn(x, uu.x));
          acc[k].y = __dadd_rn(acc[k].y, __dmul_rn(x, uu.y));
        }
      }
    }
    if (lane == 0) bulk_wait_read();  // the previous row's copy has read the staging row
    __syncwarp();
#pragma unroll
    for (int k = 0; k < kMaxPairs; ++k) {
      const uint32_t j = 64 * k + 2 * lane;
      if (j < r) {
        double2 o;
        o.x = __dmul_rn(acc[k].x, inv[j]);
        o.y = __dmul_rn(acc[k].y, inv[j + 1]);
        *reinterpret_cast<double2*>(srow + j) = o;
      }
    }
    fence_for_bulk();
    __syncwarp();
    if (lane == 0) bulk_store_row(v + (c - col_lo) * r, srow, r * 8u);
  }
  if (lane == 0) bulk_wait_all();
}

}  // namespace

void recover_v_device(const DevCsc& a, const double* u, uint32_t u_cols, const uint32_t* retained,
                      const double* sigma, uint32_t r, double* v, uint64_t col_lo, uint64_t col_hi,
                      cudaStream_t s) {
  if (r == 0 || col_hi <= col_lo) return;
  DBuf<double> u_ret((uint64_t)a.rows * r, s), inv(r, s);
  const uint64_t tot = (uint64_t)a.rows * r;
  unsigned g1 = (unsigned)std::min<uint64_t>(ceil_div(tot ? tot : 1, 256), 65535);
  gather_u<<<g1, 256, 0, s>>>(u, (uint32_t)a.rows, u_cols, retained, r, sigma, u_ret.get(), inv.get());
  RK_LAUNCH_CHECK();
  int dev = 0;
  cudaGetDevice(&dev);
  const int sms = device_sms(dev);
  const uint64_t cols = col_hi - col_lo;
  unsigned grid = (unsigned)std::min<uint64_t>(ceil_div(cols * 32, 256), (uint64_t)sms * 16);
  if (grid == 0) grid = 1;

  // half a warp per column up to r = 256 (at r = 512 its 32 double2 accumulators
  // per lane cost occupancy: c3 9.3 ms vs 3.9 ms for the warp-per-column kernel)
  if (!tuning().spmm_warp && r % 32 == 0 && r <= 256 && (reinterpret_cast<uintptr_t>(v) & 15) == 0) {
    spmm_half_kernel<8><<<grid, 256, 0, s>>>(a.ptr.get(), a.idx.get(), a.val.get(), u_ret.get(), inv.get(), r, col_lo,
                                             col_hi, v);
  } else if (tuning().spmm_tma && (r & 1) == 0 && r * 8 <= (uint32_t)kTmaRowBytes &&
             (reinterpret_cast<uintptr_t>(v) & 15) == 0) {
    spmm_tma_kernel<<<grid, 256, 0, s>>>(a.ptr.get(), a.idx.get(), a.val.get(), u_ret.get(), inv.get(), r, col_lo,
                                         col_hi, v);
  } else if ((r & 1) == 0 && (reinterpret_cast<uintptr_t>(v) & 15) == 0)
    spmm_kernel<true><<<grid, 256, 0, s>>>(a.ptr.get(), a.idx.get(), a.val.get(), u_ret.get(), inv.get(), r, col_lo,
                                           col_hi, v);
  else
    spmm_kernel<false><<<grid, 256, 0, s>>>(a.ptr.get(), a.idx.get(), a.val.get(), u_ret.get(), inv.get(), r, col_lo,
                                            col_hi, v);
  RK_LAUNCH_CHECK();
}

}  // namespace rk
