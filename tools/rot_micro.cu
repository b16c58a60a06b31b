// Cycle cost of the pieces of one Jacobi pair update (one warp, LP=8, E=24).
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_1809_10585_b200/csrc/hq_common.cuh"
#include "../paper_1809_10585_b200/csrc/hq_svd_kernel.cuh"
#include "../paper_1809_10585_b200/csrc/hq_svd_cluster.cuh"
constexpr int LP = 8, E = 24, LD = 192;
template <int MODE>
__global__ void k(double* out, long long* cyc, int iters, int nact) {
  __shared__ __align__(16) double sm[LD * 32];
  const int lane = threadIdx.x & 31, gl = lane % LP, grp = threadIdx.x / LP; const bool work = (threadIdx.x >> 5) < nact;
  for (int i = threadIdx.x; i < LD * 32; i += blockDim.x) sm[i] = 1.0 / (i + 3);
  __syncthreads();
  double xp[E];
  double* cy = sm + (grp % 32) * LD;
#pragma unroll
  for (int e = 0; e < E; ++e) xp[e] = 0.5 + e * 1e-3 * lane;
  double a = 3.0, b = 2.0, acc = 0.0;
  const long long c0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (MODE == 5) {
      if (work) {
        double bb = b;
        rotate_reg<LP, E>(xp, cy, a, bb, 144, 1e-28, 1e-30, 1e-20, gl, true);
        a = 3.0 + 1e-3 * bb;
      }
    } else if (work) {
    double xq[E];
    double g0 = 0.0, g1 = 0.0;
#pragma unroll
    for (int e = 0; e < E / 2; ++e) {
      const int i = 2 * gl + 2 * LP * e;
      double2 vq = *reinterpret_cast<const double2*>(cy + i);
      xq[2 * e] = vq.x; xq[2 * e + 1] = vq.y;
      g0 = fma(xp[2 * e], vq.x, g0);
      g1 = fma(xp[2 * e + 1], vq.y, g1);
    }
    double g = g0 + g1;
    if (MODE >= 1) {
#pragma unroll
      for (int o = LP / 2; o > 0; o >>= 1) g += __shfl_xor_sync(0xffffffffu, g, o);
    }
    double tt = 0.01, c = 0.99, sn = 0.0099;
    if (MODE >= 2) tt = jacobi_tan(a, b, g);
    if (MODE >= 3) { c = rsqrt(1.0 + tt * tt); sn = c * tt; }
    if (MODE >= 4) {
#pragma unroll
      for (int e = 0; e < E / 2; ++e) {
        const int i = 2 * gl + 2 * LP * e;
        const double x0 = xp[2 * e], x1 = xp[2 * e + 1];
        xp[2 * e] = c * x0 - sn * xq[2 * e];
        xp[2 * e + 1] = c * x1 - sn * xq[2 * e + 1];
        *reinterpret_cast<double2*>(cy + i) = make_double2(sn * x0 + c * xq[2 * e], sn * x1 + c * xq[2 * e + 1]);
      }
    } else {
      acc += g * tt * c * sn;
    }
    a = a + 1e-9 * g; b = b - 1e-9 * g;
    }
    if (blockDim.x > 32) __syncthreads(); else __syncwarp();
  }
  const long long c1 = clock64();
  if (threadIdx.x == 0) cyc[MODE] = (c1 - c0) / iters;
  double s = acc + a;
  for (int e = 0; e < E; ++e) s += xp[e];
  out[threadIdx.x] = s;
}
int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 1024 * 8); cudaMallocManaged(&cyc, 8 * 8);
  int cfg[][2] = {{32, 1}, {512, 1}, {512, 2}, {512, 5}, {512, 8}, {512, 16}};
  for (auto& c : cfg) {
    k<0><<<1, c[0]>>>(out, cyc, 1000, c[1]); k<1><<<1, c[0]>>>(out, cyc, 1000, c[1]); k<2><<<1, c[0]>>>(out, cyc, 1000, c[1]);
    k<3><<<1, c[0]>>>(out, cyc, 1000, c[1]); k<4><<<1, c[0]>>>(out, cyc, 1000, c[1]); k<5><<<1, c[0]>>>(out, cyc, 1000, c[1]);
    cudaDeviceSynchronize();
    printf("threads %d active warps %d cycles/iter: load+dot %lld, +shfl %lld, +tan %lld, +rsqrt %lld, +rotate/store %lld  rotate_reg %lld\n", c[0], c[1], cyc[0], cyc[1], cyc[2], cyc[3], cyc[4], cyc[5]);
  }
  return 0;
}
