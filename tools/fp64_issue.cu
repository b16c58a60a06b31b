// DFMA / DMUL issue rate per warp and per SM, and LDS/STS costs.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dfma_k(double* out, long long* cyc, int iters, int nact) {
  const bool work = (threadIdx.x >> 5) < nact;
  double a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double m = 0.999999, c = 1e-9;
  __syncthreads();
  const long long c0 = clock64();
  if (work)
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        a0 = fma(a0, m, c); a1 = fma(a1, m, c); a2 = fma(a2, m, c); a3 = fma(a3, m, c);
        a4 = fma(a4, m, c); a5 = fma(a5, m, c); a6 = fma(a6, m, c); a7 = fma(a7, m, c);
      }
    }
  __syncthreads();
  const long long c1 = clock64();
  if (threadIdx.x == 0) cyc[0] = c1 - c0;
  out[threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}
__global__ void ffma_k(float* out, long long* cyc, int iters, int nact) {
  const bool work = (threadIdx.x >> 5) < nact;
  float a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const float m = 0.999999f, c = 1e-9f;
  __syncthreads();
  const long long c0 = clock64();
  if (work)
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        a0 = fmaf(a0, m, c); a1 = fmaf(a1, m, c); a2 = fmaf(a2, m, c); a3 = fmaf(a3, m, c);
        a4 = fmaf(a4, m, c); a5 = fmaf(a5, m, c); a6 = fmaf(a6, m, c); a7 = fmaf(a7, m, c);
      }
    }
  __syncthreads();
  const long long c1 = clock64();
  if (threadIdx.x == 0) cyc[0] = c1 - c0;
  out[threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}
int main() {
  double* out; float* outf; long long* cyc;
  cudaMalloc(&out, 1024 * 8); cudaMalloc(&outf, 1024 * 4); cudaMallocManaged(&cyc, 8 * 8);
  const int iters = 4096;
  for (int na : {1, 2, 4, 8, 16, 32}) {
    dfma_k<<<1, 1024>>>(out, cyc, iters, na); cudaDeviceSynchronize();
    const double cd = (double)cyc[0] / (iters * 32.0);
    ffma_k<<<1, 1024>>>(outf, cyc, iters, na); cudaDeviceSynchronize();
    const double cf = (double)cyc[0] / (iters * 32.0);
    printf("warps %2d: DFMA cycles per warp-instr (per warp) %.2f -> SM DFMA lanes/clk %.1f | FFMA %.2f -> lanes/clk %.1f\n",
           na, cd, na * 32 / cd, cf, na * 32 / cf);
  }
  return 0;
}
