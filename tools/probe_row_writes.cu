// How fast can 4 KB rows of zeros be written to a 16 GiB buffer? (the V recovery at c3: 98 % of V's rows)
//   mode 0: warp per row, 8 x 16-byte st.global.cs per lane (spmm_kernel's stores)
//   mode 1: the same with plain st.global
//   mode 2: lane per row, one 4 KB cp.async.bulk shared -> global from a constant zero row (spmm_tma_kernel)
//   mode 3: flat grid-stride fill, 16 bytes per thread and step (what torch's fill does)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/probe_row_writes tools/probe_row_writes.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
template <int MODE>
__global__ void __launch_bounds__(256) k(double* v, uint64_t rows, const uint64_t* col_ptr) {
  constexpr uint32_t r = 512;
  __shared__ __align__(128) double zrow[r];
  const int lane = threadIdx.x & 31;
  for (uint32_t t = threadIdx.x; t < r; t += blockDim.x) zrow[t] = 0.0;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  const uint64_t warp0 = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  if (MODE == 3) {
    double2* p = reinterpret_cast<double2*>(v);
    const uint64_t n = rows * r / 2;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
      p[i] = make_double2(0.0, 0.0);
    return;
  }
  for (uint64_t base = warp0 * 32; base < rows; base += nwarps * 32) {
    uint64_t dep = 0;
    if (col_ptr) dep = col_ptr[base + lane] - col_ptr[base + lane];  // a dependent load per chunk, as the real kernel
    if (MODE == 2) {
      const uint64_t c = base + lane + dep;
      if (c < rows) {
        const uint32_t sa = (uint32_t)__cvta_generic_to_shared(zrow);
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(v + c * r), "r"(sa), "r"(r * 8u) : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
    } else {
      for (int i = 0; i < 32; ++i) {
        const uint64_t c = base + i + dep;
        if (c >= rows) break;
        double2* row = reinterpret_cast<double2*>(v + c * r);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          if (MODE == 0) __stcs(row + 32 * kk + lane, make_double2(0.0, 0.0));
          else row[32 * kk + lane] = make_double2(0.0, 0.0);
        }
      }
    }
  }
  if (MODE == 2) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
template <int MODE>
float run(double* v, uint64_t rows, const uint64_t* cp, int grid) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e9f;
  for (int it = 0; it < 4; ++it) {
    cudaEventRecord(e0); k<MODE><<<grid, 256>>>(v, rows, cp); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); if (it) best = ms < best ? ms : best;
  }
  return best;
}
int main() {
  const uint64_t rows = 4194304; double* v; cudaMalloc(&v, rows * 512 * 8);
  uint64_t* cp; cudaMalloc(&cp, (rows + 64) * 8); cudaMemset(cp, 0, (rows + 64) * 8);
  const double gb = rows * 512.0 * 8 / 1e9;
  for (int per_sm : {8, 16, 32, 64}) {
    const int grid = 148 * per_sm;
    for (int dep = 0; dep < 2; ++dep) {
      const uint64_t* c = dep ? cp : nullptr;
      printf("grid %5d dep-load %d: st.cs %.3f ms (%.0f GB/s) | st %.3f ms (%.0f GB/s) | bulk %.3f ms (%.0f GB/s) | flat %.3f ms (%.0f GB/s)\n", grid, dep,
             run<0>(v, rows, c, grid), gb / run<0>(v, rows, c, grid) * 1e3, run<1>(v, rows, c, grid), gb / run<1>(v, rows, c, grid) * 1e3,
             run<2>(v, rows, c, grid), gb / run<2>(v, rows, c, grid) * 1e3, run<3>(v, rows, c, grid), gb / run<3>(v, rows, c, grid) * 1e3);
    }
  }
  return 0;
}
