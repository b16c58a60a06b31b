// Cycles per Jacobi round (jacobi_pair + barrier) for lane-group shapes vs pairs per CTA.
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_1809_10585_b200/csrc/hq_common.cuh"
#include "../paper_1809_10585_b200/csrc/hq_svd_kernel.cuh"
template <int LP, int E, bool XREG>
__global__ void __launch_bounds__(512, 1) k(double* out, long long* cyc, int iters, int npairs, int ld) {
  extern __shared__ __align__(16) double sm[];
  __shared__ double2 trash[32];
  constexpr int GPW = 32 / LP;
  const int lane = threadIdx.x & 31, gl = lane % LP, grp = (threadIdx.x >> 5) * GPW + lane / LP;
  const int ncol = 2 * 64;
  for (int i = threadIdx.x; i < ncol * ld; i += blockDim.x) sm[i] = 1.0 / (i + 3);
  __syncthreads();
  double xp[E];
#pragma unroll
  for (int e = 0; e < E; ++e) xp[e] = 0.5 + e * 1e-3 * lane;
  double a = 3.0;
  const bool act = grp < npairs;
  const bool warp_act = (threadIdx.x >> 5) * GPW < npairs;
  double* cx = sm + (size_t)(2 * (grp % 64)) * ld;
  double* cy = cx + ld;
  const long long c0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (warp_act) {
      double bb = 2.0;
      jacobi_pair<LP, E, XREG>(xp, cx, cy, a, bb, ld, 1e-28, 1e-30, 1e-20, gl, act, trash);
      a = 3.0 + 1e-3 * bb;
    }
    __syncthreads();
  }
  const long long c1 = clock64();
  if (threadIdx.x == 0) *cyc = (c1 - c0) / iters;
  double s = a;
  for (int e = 0; e < E; ++e) s += xp[e];
  out[threadIdx.x] = s;
}
template <int LP, int E, bool XREG>
long long run(double* out, long long* cyc, int np, int ld) {
  auto f = k<LP, E, XREG>;
  const int smem = 128 * ld * 8;
  cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  f<<<1, 512, smem>>>(out, cyc, 1000, np, ld);
  cudaDeviceSynchronize();
  return *cyc;
}
int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 1024 * 8); cudaMallocManaged(&cyc, 8);
  for (int ld : {64, 128, 208}) {
    for (int np : {4, 8, 13, 16, 24, 32, 48, 64}) {
      printf("ld %3d pairs %2d |", ld, np);
      if (ld <= 64) printf(" 8x8 %5lld/%5lld |", run<8, 8, true>(out, cyc, np, ld), run<8, 8, false>(out, cyc, np, ld));
      if (ld <= 128) printf(" 8x16 %5lld/%5lld | 16x8 %5lld/%5lld | 32x4 %5lld/%5lld |",
                            run<8, 16, true>(out, cyc, np, ld), run<8, 16, false>(out, cyc, np, ld),
                            np <= 32 ? run<16, 8, true>(out, cyc, np, ld) : 0LL, np <= 32 ? run<16, 8, false>(out, cyc, np, ld) : 0LL,
                            np <= 16 ? run<32, 4, true>(out, cyc, np, ld) : 0LL, np <= 16 ? run<32, 4, false>(out, cyc, np, ld) : 0LL);
      printf(" 16x16 %5lld/%5lld | 32x8 %5lld/%5lld\n",
             np <= 32 ? run<16, 16, true>(out, cyc, np, ld) : 0LL, np <= 32 ? run<16, 16, false>(out, cyc, np, ld) : 0LL,
             np <= 16 ? run<32, 8, true>(out, cyc, np, ld) : 0LL, np <= 16 ? run<32, 8, false>(out, cyc, np, ld) : 0LL);
    }
  }
  return 0;
}
