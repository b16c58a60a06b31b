// Cycles of the W = Y^T X k-loop pattern (8 loads + 8 loads, 8 dependent DMMAs per 32 rows).
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_1809_10585_b200/csrc/hq_common.cuh"
template <int MODE>
__global__ void k(const double* Yg, const double* Xg, double* out, long long* cyc, int rows, int ld) {
  __shared__ double Ys[384 * 16];
  for (int i = threadIdx.x; i < 384 * 16; i += blockDim.x) Ys[i] = Yg[i % 384 + (i / 384) * ld];
  __syncthreads();
  const int lane = threadIdx.x & 31, gq = lane >> 2, tq = lane & 3;
  const double* Y = MODE == 0 ? Ys : Yg;
  const int ldy = MODE == 0 ? 384 : ld;
  double d0 = 0, d1 = 0;
  const long long c0 = clock64();
  if (MODE <= 1) {
    for (int k0 = 0; k0 < rows; k0 += 32) {
      double av[8], bv[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int ia = k0 + 4 * u + tq;
        av[u] = ia < rows ? Y[ia + gq * ldy] : 0.0;
        bv[u] = ia < rows ? Xg[ia + gq * ld] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) dmma884(d0, d1, av[u], bv[u]);
    }
  } else if (MODE == 2) {
    // DMMA only
    for (int k0 = 0; k0 < rows; k0 += 32) {
#pragma unroll
      for (int u = 0; u < 8; ++u) dmma884(d0, d1, 1.0 + k0, 0.5);
    }
  } else {
    dmma_kloop(d0, d1, 0, rows, [&](int k0, double (&av)[8], double (&bv)[8]) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int ia = k0 + 4 * u + tq;
        av[u] = ia < rows ? Yg[ia + gq * ld] : 0.0;
        bv[u] = ia < rows ? Xg[ia + gq * ld] : 0.0;
      }
    });
  }
  const long long c1 = clock64();
  if (threadIdx.x == 0) *cyc = c1 - c0;
  out[threadIdx.x] = d0 + d1;
}
int main() {
  double *Y, *X, *out; long long* cyc;
  const int ld = 400;
  cudaMalloc(&Y, ld * 16 * 8 + 8192 * 8); cudaMalloc(&X, ld * 16 * 8 + 8192 * 8); cudaMalloc(&out, 1024 * 8);
  cudaMemset(Y, 0, ld * 16 * 8); cudaMemset(X, 0, ld * 16 * 8);
  cudaMallocManaged(&cyc, 8);
  const char* names[] = {"Y smem, X global", "Y global, X global", "DMMA only", "pipelined (global)"};
  for (int rep = 0; rep < 2; ++rep) {
    for (int md = 0; md < 4; ++md) {
      if (md == 0) k<0><<<1, 32>>>(Y, X, out, cyc, 384, ld);
      if (md == 1) k<1><<<1, 32>>>(Y, X, out, cyc, 384, ld);
      if (md == 2) k<2><<<1, 32>>>(Y, X, out, cyc, 384, ld);
      if (md == 3) k<3><<<1, 32>>>(Y, X, out, cyc, 384, ld);
      cudaDeviceSynchronize();
      if (rep) printf("%-22s rows 384: %lld cycles (%lld per 32 rows)\n", names[md], *cyc, *cyc / 12);
    }
  }
  return 0;
}
