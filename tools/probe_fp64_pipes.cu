// Do DMMA (m8n8k4 f64) and DFMA share an issue pipe on sm_100a? Time N warps per SM doing
// (a) DMMAs only, (b) DFMAs only, (c) both interleaved in one instruction stream.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/probe_fp64_pipes tools/probe_fp64_pipes.cu
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
template <int MODE>
__global__ void k(double* out, int iters, long long* cyc) {
  double d[8][2], f[16];
  const double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-6;
#pragma unroll
  for (int i = 0; i < 8; ++i) d[i][0] = d[i][1] = 0.0;
#pragma unroll
  for (int i = 0; i < 16; ++i) f[i] = i;
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (MODE & 1) {
#pragma unroll
      for (int i = 0; i < 8; ++i) dmma(d[i][0], d[i][1], a, b);
    }
    if (MODE & 2) {
#pragma unroll
      for (int i = 0; i < 16; ++i) asm volatile("fma.rn.f64 %0, %1, %2, %0;" : "+d"(f[i]) : "d"(a), "d"(b));
    }
  }
  const long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += d[i][0] + d[i][1];
#pragma unroll
  for (int i = 0; i < 16; ++i) s += f[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
int main() {
  double* out; long long* cyc; cudaMalloc(&out, 148 * 1024 * 8); cudaMallocManaged(&cyc, 8);
  const int iters = 2000;
  for (int warps : {4, 8, 16, 32}) {
    long long c[4] = {0, 0, 0, 0};
    for (int rep = 0; rep < 2; ++rep) {
      k<1><<<148, warps * 32>>>(out, iters, cyc); cudaDeviceSynchronize(); c[1] = *cyc;
      k<2><<<148, warps * 32>>>(out, iters, cyc); cudaDeviceSynchronize(); c[2] = *cyc;
      k<3><<<148, warps * 32>>>(out, iters, cyc); cudaDeviceSynchronize(); c[3] = *cyc;
    }
    // per SM per iteration: warps * 8 DMMA (512 flop) and warps * 16 DFMA warp-instructions (64 flop)
    printf("warps/SM %2d: dmma-only %.1f cyc/iter (%.1f clk per DMMA per SMSP), dfma-only %.1f cyc/iter (%.2f clk per DFMA per SMSP), both %.1f cyc/iter (sum %.1f)\n",
           warps, (double)c[1] / iters, (double)c[1] / iters / (warps * 8 / 4.0), (double)c[2] / iters,
           (double)c[2] / iters / (warps * 16 / 4.0), (double)c[3] / iters, (double)(c[1] + c[2]) / iters);
  }
  return 0;
}
