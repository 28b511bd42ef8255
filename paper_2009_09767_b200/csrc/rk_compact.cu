// rk_compact.cu -- block compaction: the sparse block A_d (M x N_d) becomes
// the small dense input of its factorization, exactly (orthogonally) equivalent
// to the reference's densified block (proj/src/svd.cpp:381-395, dense_of at
// proj/src/dense_matrix.cpp:62-75) for the purpose of sigma and U:
//
//  * empty columns of A_d are dropped (zero rows of A_d^T never change R);
//  * columns with exactly one entry (m, v) are merged per row m into a single
//    row sqrt(sum v^2) e_m (a Givens/Householder rotation of rows of A_d^T, so
//    A_d A_d^T is unchanged);
//  * columns with two or more entries are kept as rows of T_d.
//
// T_d = [multi-entry columns; merged single-entry rows] has n_d = n_multi +
// n_single rows. When n_d > M the factorization is QR(T_d) -> R, Jacobi on R^T
// ("tall" plan, T_d stored column-major n_d x M). Otherwise Jacobi runs
// directly on W = T_d^T (M x n_d column-major). Both W W^T = A_d A_d^T.
#include "rk_internal.cuh"

namespace rk {
namespace {

constexpr int kT = 256;

// counts[2*i] = multi-entry columns of block d_lo+i
__global__ void multi_counts(const uint64_t* col_ptr, Partition p, uint64_t d_lo, uint32_t* counts) {
  __shared__ uint32_t red[kT / 32];
  const uint64_t d = d_lo + blockIdx.x;
  const uint64_t b = p.begin(d), e = p.end(d);
  uint32_t n = 0;
  for (uint64_t c = b + threadIdx.x; c < e; c += kT) n += (col_ptr[c + 1] - col_ptr[c]) >= 2;
  for (int o = 16; o; o >>= 1) n += __shfl_down_sync(0xffffffffu, n, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = n;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
    for (int w = 0; w < kT / 32; ++w) t += red[w];
    counts[2 * blockIdx.x] = t;
  }
}

// single[i*M + m] = sum of v^2 over single-entry columns of block d_lo+i in row m;
// counts[2*i+1] = rows with a nonzero sum. Warp per (block, row); fixed lane
// assignment and reduction tree -> deterministic.
__global__ void single_sums(const uint64_t* row_ptr, const uint32_t* col_idx, const double* val,
                            const uint64_t* col_ptr, uint64_t rows, Partition p, uint64_t d_lo, uint64_t nblk,
                            double* single, uint32_t* counts) {
  const int lane = threadIdx.x & 31;
  const uint64_t total = nblk * rows;
  for (uint64_t t = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; t < total;
       t += ((uint64_t)gridDim.x * blockDim.x) >> 5) {
    const uint64_t i = t / rows, m = t % rows, d = d_lo + i;
    const uint64_t b = p.begin(d), e = p.end(d);
    uint64_t lo = row_ptr[m], hi = row_ptr[m + 1];
    while (lo < hi) {
      uint64_t mid = (lo + hi) >> 1;
      if (col_idx[mid] < b) lo = mid + 1; else hi = mid;
    }
    double acc = 0.0;
    for (uint64_t k = lo + lane; k < row_ptr[m + 1]; k += 32) {
      const uint32_t c = col_idx[k];
      if (c >= e) break;
      if (col_ptr[c + 1] - col_ptr[c] == 1) acc += val[k] * val[k];
    }
    for (int o = 16; o; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
    if (lane == 0) {
      single[i * rows + m] = acc;
      if (acc > 0.0) atomicAdd(&counts[2 * i + 1], 1u);
    }
  }
}

struct FillPlan {
  uint64_t offset;
  uint32_t n_multi, n_rows;
  uint32_t tall;
};

// CTA per block: scatter multi-entry columns and merged rows into the staging
// buffer (already zeroed)
__global__ void fill_kernel(const uint64_t* col_ptr, const uint32_t* row_idx, const double* val, uint64_t rows,
                            Partition p, uint64_t d_lo, const uint64_t* plan_block, const FillPlan* plans,
                            const double* single, double* staging) {
  __shared__ uint32_t warp_tot[kT / 32];
  __shared__ uint32_t carry;
  const FillPlan pl = plans[blockIdx.x];
  const uint64_t d = plan_block[blockIdx.x];
  const uint64_t i_blk = d - d_lo;
  const uint64_t b = p.begin(d), e = p.end(d);
  double* out = staging + pl.offset;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // index of a compacted row t, column m
  auto put = [&](uint64_t t, uint64_t m, double x) {
    if (pl.tall) out[t + m * (uint64_t)pl.n_rows] = x;  // T_d column-major (n_rows x M)
    else out[m + t * rows] = x;                         // W = T_d^T column-major (M x n_rows)
  };
  for (int phase = 0; phase < 2; ++phase) {
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    const uint64_t lo = phase == 0 ? b : 0, hi = phase == 0 ? e : rows;
    for (uint64_t base = lo; base < hi; base += kT) {
      const uint64_t x = base + threadIdx.x;
      uint32_t f = 0;
      if (x < hi) {
        if (phase == 0) f = (col_ptr[x + 1] - col_ptr[x]) >= 2;
        else f = single[i_blk * rows + x] > 0.0;
      }
      uint32_t inc = f;
      for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
      }
      if (lane == 31) warp_tot[warp] = inc;
      __syncthreads();
      uint32_t before = carry;
      for (int w = 0; w < warp; ++w) before += warp_tot[w];
      const uint32_t idx = before + inc - f;
      if (phase == 0) {
        // a short column is scattered by its own thread; a long one (Zipf columns have up to M
        // entries: one thread's dependent loads were the kernel's long pole) by its whole warp
        const uint64_t k0 = f ? col_ptr[x] : 0, k1 = f ? col_ptr[x + 1] : 0;
        constexpr uint64_t kLong = 8;
        if (f && k1 - k0 <= kLong)
          for (uint64_t k = k0; k < k1; ++k) put(idx, row_idx[k], val[k]);
        unsigned heavy = __ballot_sync(0xffffffffu, f && k1 - k0 > kLong);
        while (heavy) {
          const int src = __ffs(heavy) - 1;
          heavy &= heavy - 1;
          const uint64_t b0 = __shfl_sync(0xffffffffu, k0, src), b1 = __shfl_sync(0xffffffffu, k1, src);
          const uint32_t t = __shfl_sync(0xffffffffu, idx, src);
          for (uint64_t k = b0 + lane; k < b1; k += 32) put(t, row_idx[k], val[k]);
        }
      } else if (f) {
        put(pl.n_multi + idx, x, sqrt(single[i_blk * rows + x]));
      }
      __syncthreads();
      if (threadIdx.x == kT - 1) carry = before + inc;
      __syncthreads();
    }
  }
}

}  // namespace

void compaction_counts(const DevMatrix& a, const Partition& p, uint64_t d_lo, uint64_t d_hi, uint32_t* d_counts,
                       double* d_single, cudaStream_t s) {
  const uint64_t nblk = d_hi - d_lo, rows = a.csr.rows;
  RK_CUDA_CHECK(cudaMemsetAsync(d_counts, 0, 2 * nblk * sizeof(uint32_t), s));
  multi_counts<<<(unsigned)nblk, kT, 0, s>>>(a.csc.ptr.get(), p, d_lo, d_counts);
  RK_LAUNCH_CHECK();
  if (rows) {
    uint64_t warps = nblk * rows;
    uint64_t grid = ceil_div(warps * 32, kT);
    if (grid > (1u << 20)) grid = 1u << 20;
    single_sums<<<(unsigned)grid, kT, 0, s>>>(a.csr.ptr.get(), a.csr.idx.get(), a.csr.val.get(), a.csc.ptr.get(),
                                              rows, p, d_lo, nblk, d_single, d_counts);
    RK_LAUNCH_CHECK();
  }
}

void compaction_fill(const DevMatrix& a, const Partition& p, const std::vector<BlockPlan>& plans, uint64_t d_lo,
                     const double* d_single, double* staging, cudaStream_t s) {
  if (plans.empty()) return;
  std::vector<FillPlan> fp(plans.size());
  std::vector<uint64_t> blk(plans.size());
  for (size_t i = 0; i < plans.size(); ++i) {
    fp[i].offset = plans[i].offset;
    fp[i].n_multi = plans[i].n_multi;
    fp[i].n_rows = plans[i].n_rows;
    fp[i].tall = plans[i].tall ? 1u : 0u;
    blk[i] = plans[i].block;
  }
  DBuf<FillPlan> dfp(fp.size(), s);
  DBuf<uint64_t> dblk(blk.size(), s);
  to_device(dfp.get(), fp.data(), fp.size(), s);
  to_device(dblk.get(), blk.data(), blk.size(), s);
  fill_kernel<<<(unsigned)plans.size(), kT, 0, s>>>(a.csc.ptr.get(), a.csc.idx.get(), a.csc.val.get(), a.csr.rows,
                                                    p, d_lo, dblk.get(), dfp.get(), d_single, staging);
  RK_LAUNCH_CHECK();
  sync(s);  // host plan vectors go out of scope
}

}  // namespace rk
