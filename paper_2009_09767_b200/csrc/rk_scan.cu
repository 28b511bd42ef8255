// rk_scan.cu -- deterministic exclusive prefix sums (offsets for CSR/CSC and
// block compaction). Three passes: tile totals, a single-CTA scan of the
// totals, and a rescan of each tile with its carry-in. Integer sums, so the
// result does not depend on the tiling.
#include "rk_internal.cuh"

namespace rk {
namespace {

constexpr int kThreads = 512;
constexpr int kItems = 8;
constexpr int kTile = kThreads * kItems;

template <class T>
__device__ __forceinline__ uint64_t block_inclusive_scan(uint64_t x, uint64_t* warp_tot) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint64_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_tot[warp] = x;
  __syncthreads();
  if (warp == 0) {
    uint64_t t = lane < (kThreads / 32) ? warp_tot[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint64_t y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    if (lane < kThreads / 32) warp_tot[lane] = t;
  }
  __syncthreads();
  if (warp > 0) x += warp_tot[warp - 1];
  return x;
}

template <class T>
__global__ void tile_totals(const T* in, uint64_t n, uint64_t* totals) {
  __shared__ uint64_t red[kThreads / 32];
  const uint64_t base = (uint64_t)blockIdx.x * kTile;
  uint64_t s = 0;
  for (int i = 0; i < kItems; ++i) {
    uint64_t j = base + (uint64_t)i * kThreads + threadIdx.x;
    if (j < n) s += (uint64_t)in[j];
  }
  for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t t = 0;
    for (int w = 0; w < kThreads / 32; ++w) t += red[w];
    totals[blockIdx.x] = t;
  }
}

// exclusive scan of totals in place (single CTA, chunked)
__global__ void scan_totals(uint64_t* totals, uint64_t n) {
  __shared__ uint64_t warp_tot[kThreads / 32];
  __shared__ uint64_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (uint64_t base = 0; base < n; base += kThreads) {
    uint64_t j = base + threadIdx.x;
    uint64_t x = j < n ? totals[j] : 0;
    uint64_t inc = block_inclusive_scan<uint64_t>(x, warp_tot);
    uint64_t c = carry;
    if (j < n) totals[j] = c + inc - x;
    __syncthreads();
    if (threadIdx.x == kThreads - 1) carry = c + inc;
    __syncthreads();
  }
}

template <class T>
__global__ void tile_scan(const T* in, uint64_t n, const uint64_t* offsets, uint64_t* out) {
  __shared__ uint64_t warp_tot[kThreads / 32];
  const uint64_t base = (uint64_t)blockIdx.x * kTile + (uint64_t)threadIdx.x * kItems;
  uint64_t v[kItems];
  uint64_t s = 0;
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    uint64_t j = base + i;
    v[i] = j < n ? (uint64_t)in[j] : 0;
    s += v[i];
  }
  uint64_t inc = block_inclusive_scan<T>(s, warp_tot);
  uint64_t run = offsets[blockIdx.x] + inc - s;
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    uint64_t j = base + i;
    if (j < n) out[j] = run;
    run += v[i];
  }
  if (base < n && base + kItems >= n) out[n] = run;  // total, written by the owner of the last item
}

template <class T>
void scan_impl(const T* in, uint64_t* out, uint64_t n, cudaStream_t s) {
  if (n == 0) {
    RK_CUDA_CHECK(cudaMemsetAsync(out, 0, sizeof(uint64_t), s));
    return;
  }
  const uint64_t tiles = ceil_div(n, kTile);
  DBuf<uint64_t> totals(tiles, s);
  tile_totals<T><<<(unsigned)tiles, kThreads, 0, s>>>(in, n, totals.get());
  RK_LAUNCH_CHECK();
  scan_totals<<<1, kThreads, 0, s>>>(totals.get(), tiles);
  RK_LAUNCH_CHECK();
  tile_scan<T><<<(unsigned)tiles, kThreads, 0, s>>>(in, n, totals.get(), out);
  RK_LAUNCH_CHECK();
}

}  // namespace

void exclusive_scan_u64(const uint64_t* in, uint64_t* out, uint64_t n, cudaStream_t s) {
  scan_impl<uint64_t>(in, out, n, s);
}
void exclusive_scan_u32to64(const uint32_t* in, uint64_t* out, uint64_t n, cudaStream_t s) {
  scan_impl<uint32_t>(in, out, n, s);
}

}  // namespace rk
