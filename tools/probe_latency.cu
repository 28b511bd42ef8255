// Latency probes on one warp (clock64): dependent FP64 chains, double shuffles,
// rsqrt/sqrt/div, and three ways to factor a 32x32 SPD block in one warp.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/probe tools/probe_latency.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void chains(double* out, long long* cyc, double x0) {
  const int lane = threadIdx.x;
  double x = x0 + lane * 1e-3;
  long long t0, t1;
  // 1. DFMA chain
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) x = fma(x, 0.999999, 1e-7);
  t1 = clock64();
  if (lane == 0) cyc[0] = (t1 - t0) / 1024;
  // 2. shuffle chain (double, idx)
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) x = __shfl_sync(0xffffffffu, x, (lane + 1) & 31) + 1e-9;
  t1 = clock64();
  if (lane == 0) cyc[1] = (t1 - t0) / 1024;
  // 3. rsqrt chain
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) x = rsqrt(x) + 1.0;
  t1 = clock64();
  if (lane == 0) cyc[2] = (t1 - t0) / 1024;
  // 4. sqrt chain
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) x = sqrt(x) + 1.0;
  t1 = clock64();
  if (lane == 0) cyc[3] = (t1 - t0) / 1024;
  // 5. div chain
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) x = 1.0 / x + 1.0;
  t1 = clock64();
  if (lane == 0) cyc[4] = (t1 - t0) / 1024;
  // 6. 32 independent shuffles of one value per iteration (throughput)
  double acc = 0.0;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 64; ++i) {
#pragma unroll
    for (int c = 0; c < 32; ++c) acc += __shfl_sync(0xffffffffu, x, c) * (double)c;
    x += 1e-9 * acc;
  }
  t1 = clock64();
  if (lane == 0) cyc[5] = (t1 - t0) / 64;
  // 7. DMUL/DADD chain
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) x = x * 0.9999 + 1e-9;
  t1 = clock64();
  if (lane == 0) cyc[6] = (t1 - t0) / 1024;
  // 8. float -> double conversions chain
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) x = (double)((float)x * 0.999f) + 1e-9;
  t1 = clock64();
  if (lane == 0) cyc[7] = (t1 - t0) / 1024;
  out[lane] = x + acc;
}

template <int kCB>
__device__ void fd_unrolled(double* P, int ld, int lane) {
  double rg[kCB];
#pragma unroll
  for (int c = 0; c < kCB; ++c) rg[c] = P[lane + c * ld];
#pragma unroll
  for (int j = 0; j < kCB; ++j) {
    double piv = __shfl_sync(0xffffffffu, rg[j], j);
    const double inv = rsqrt(piv);
    const double l = lane > j ? rg[j] * inv : (lane == j ? piv * inv : 0.0);
    if (lane >= j) rg[j] = l;
#pragma unroll
    for (int c = j + 1; c < kCB; ++c) {
      const double lcj = __shfl_sync(0xffffffffu, l, c);
      if (lane >= c) rg[c] -= l * lcj;
    }
  }
#pragma unroll
  for (int c = 0; c < kCB; ++c) P[lane + c * ld] = rg[c];
}

template <int kCB>
__device__ void fd_rolled(double* P, int ld, int lane) {
  double rg[kCB];
#pragma unroll
  for (int c = 0; c < kCB; ++c) rg[c] = P[lane + c * ld];
#pragma unroll 1
  for (int j = 0; j < kCB; ++j) {
    double mine = 0.0;
#pragma unroll
    for (int c = 0; c < kCB; ++c) mine = c == j ? rg[c] : mine;
    double piv = __shfl_sync(0xffffffffu, mine, j);
    const double inv = rsqrt(piv);
    const double l = lane > j ? mine * inv : (lane == j ? piv * inv : 0.0);
#pragma unroll
    for (int c = 0; c < kCB; ++c) {
      const double lcj = __shfl_sync(0xffffffffu, l, c);
      rg[c] = (c == j && lane >= j) ? l : ((c > j && lane >= c) ? rg[c] - l * lcj : rg[c]);
    }
  }
#pragma unroll
  for (int c = 0; c < kCB; ++c) P[lane + c * ld] = rg[c];
}

// unrolled, pivot chain through the pivot lane's own registers: d_{j} is updated
// and its rsqrt taken before the other lanes' updates are needed
template <int kCB>
__device__ void fd_chain(double* P, int ld, int lane) {
  double rg[kCB];
#pragma unroll
  for (int c = 0; c < kCB; ++c) rg[c] = P[lane + c * ld];
  double inv_mine = rsqrt(rg[0]);
#pragma unroll
  for (int j = 0; j < kCB; ++j) {
    const double inv = __shfl_sync(0xffffffffu, inv_mine, j);
    const double l = lane > j ? rg[j] * inv : (lane == j ? rg[j] * inv : 0.0);
    if (lane >= j) rg[j] = l;
    if (j + 1 < kCB) {
      // next pivot first: lane j+1's own entry
      const double dn = rg[j + 1] - l * l;
      inv_mine = rsqrt(dn);
#pragma unroll
      for (int c = j + 1; c < kCB; ++c) {
        const double lcj = __shfl_sync(0xffffffffu, l, c);
        if (lane >= c) rg[c] -= l * lcj;
      }
    }
  }
#pragma unroll
  for (int c = 0; c < kCB; ++c) P[lane + c * ld] = rg[c];
}

// rolled over columns: the register array shifts down one slot per column, so
// the pivot column is always rg[0] (static register indices, a ~4 KB loop body)
template <int kCB>
__device__ void fd_shift(double* P, int ld, int lane) {
  double rg[kCB];
#pragma unroll
  for (int c = 0; c < kCB; ++c) rg[c] = P[lane + c * ld];
  double out[1];
  double inv_mine = rsqrt(rg[0]);
#pragma unroll 1
  for (int j = 0; j < kCB; ++j) {
    const double inv = __shfl_sync(0xffffffffu, inv_mine, j);
    const double l = lane >= j ? rg[0] * inv : 0.0;
    const double dn = rg[1] - l * l;
    inv_mine = rsqrt(dn);
#pragma unroll
    for (int c = 1; c < kCB; ++c) {
      const double lcj = __shfl_sync(0xffffffffu, l, (j + c) & 31);
      rg[c] = lane >= j + c ? rg[c] - l * lcj : rg[c];
    }
    P[lane + j * ld] = lane >= j ? l : 0.0;
#pragma unroll
    for (int c = 0; c + 1 < kCB; ++c) rg[c] = rg[c + 1];
    rg[kCB - 1] = 0.0;
  }
  (void)out;
}

// left-looking by rows in shared memory: column j, lane i >= j: dot of rows i, j
template <int kCB>
__device__ void fd_smem(double* P, int ld, int lane) {
  for (int j = 0; j < kCB; ++j) {
    double v = P[lane + j * ld];
    if (lane >= j) {
      double a0 = 0.0, a1 = 0.0;
      int q = 0;
      for (; q + 1 < j; q += 2) {
        a0 += P[lane + q * ld] * P[j + q * ld];
        a1 += P[lane + (q + 1) * ld] * P[j + (q + 1) * ld];
      }
      if (q < j) a0 += P[lane + q * ld] * P[j + q * ld];
      v -= a0 + a1;
    }
    const double piv = __shfl_sync(0xffffffffu, v, j);
    const double inv = rsqrt(piv);
    if (lane >= j) P[lane + j * ld] = lane == j ? piv * inv : v * inv;
    __syncwarp();
  }
}

template <int V>
__global__ void fd_kernel(const double* G, double* out, long long* cyc, int reps) {
  __shared__ double P[32 * 33];
  const int lane = threadIdx.x;
  long long best = 1ll << 60;
  for (int r = 0; r < reps; ++r) {
    for (int c = 0; c < 32; ++c) P[lane + c * 33] = G[lane + c * 32];
    __syncwarp();
    const long long t0 = clock64();
    if (V == 0) fd_unrolled<32>(P, 33, lane);
    else if (V == 1) fd_rolled<32>(P, 33, lane);
    else if (V == 3) fd_chain<32>(P, 33, lane);
    else if (V == 4) fd_shift<32>(P, 33, lane);
    else fd_smem<32>(P, 33, lane);
    __syncwarp();
    const long long t1 = clock64();
    best = min(best, t1 - t0);
    if (r == 0 && lane == 0) cyc[16] = t1 - t0;  // cold instruction cache (first run)
  }
  for (int c = 0; c < 32; ++c) out[lane + c * 32] = P[lane + c * 33];
  if (lane == 0) cyc[0] = best;
}

int main() {
  double *d_out, *d_G, *d_o2;
  long long* d_cyc;
  cudaMalloc(&d_out, 32 * 8);
  cudaMalloc(&d_cyc, 64 * 8);
  chains<<<1, 32>>>(d_out, d_cyc, 1.5);
  long long h[16];
  cudaMemcpy(h, d_cyc, 8 * 8, cudaMemcpyDeviceToHost);
  const char* names[] = {"dfma chain", "shfl.f64 chain", "rsqrt chain", "sqrt chain", "div chain",
                         "32 shfl+fma / iter", "dmul+dadd chain", "f64->f32->f64 chain"};
  for (int i = 0; i < 8; ++i) printf("%-22s %lld cycles\n", names[i], h[i]);
  // SPD 32x32: G = I*32 + small
  double hG[1024];
  for (int i = 0; i < 32; ++i)
    for (int j = 0; j < 32; ++j) hG[i + 32 * j] = (i == j ? 40.0 : 0.0) + 1.0 / (1 + i + j);
  cudaMalloc(&d_G, 1024 * 8);
  cudaMalloc(&d_o2, 3 * 1024 * 8);
  cudaMemcpy(d_G, hG, 1024 * 8, cudaMemcpyHostToDevice);
  fd_kernel<0><<<1, 32>>>(d_G, d_o2, d_cyc, 20);
  fd_kernel<1><<<1, 32>>>(d_G, d_o2 + 1024, d_cyc + 1, 20);
  fd_kernel<2><<<1, 32>>>(d_G, d_o2 + 2048, d_cyc + 2, 20);
  long long cold[5];
  for (int v = 0; v < 5; ++v) {
    long long* cp = d_cyc + 8;
    double* o = d_o2 + (v == 0 ? 0 : (v == 1 ? 1024 : 2048));
    switch (v) {
      case 0: fd_kernel<0><<<1, 32>>>(d_G, o, d_cyc + 0 - 0, 20); break;
      case 1: fd_kernel<1><<<1, 32>>>(d_G, o, d_cyc + 1 - 0, 20); break;
      case 2: fd_kernel<2><<<1, 32>>>(d_G, o, d_cyc + 2 - 0, 20); break;
      case 3: fd_kernel<3><<<1, 32>>>(d_G, o, d_cyc + 3 - 0, 20); break;
      case 4: fd_kernel<4><<<1, 32>>>(d_G, o, d_cyc + 4 - 0, 20); break;
    }
    cudaDeviceSynchronize();
    long long c0;
    cudaMemcpy(&c0, d_cyc + v + 16, 8, cudaMemcpyDeviceToHost);
    printf("variant %d: first run %lld cycles\n", v, c0);
    (void)cp;
  }
  cudaMemcpy(h, d_cyc, 5 * 8, cudaMemcpyDeviceToHost);
  (void)cold;
  double o[3072];
  cudaMemcpy(o, d_o2, 3 * 1024 * 8, cudaMemcpyDeviceToHost);
  double d01 = 0, d02 = 0;
  for (int i = 0; i < 32; ++i)
    for (int j = 0; j <= i; ++j) {
      d01 = fmax(d01, fabs(o[i + 32 * j] - o[1024 + i + 32 * j]));
      d02 = fmax(d02, fabs(o[i + 32 * j] - o[2048 + i + 32 * j]));
    }
  printf("factor 32x32 (best of 20): unrolled %lld, rolled %lld, smem %lld, pivot-chain %lld, shift %lld cycles (diffs %.2e %.2e) %s\n",
         h[0], h[1], h[2], h[3], h[4], d01, d02, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
