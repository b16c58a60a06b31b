// Cycle cost of one Jacobi pair update for several lane-group shapes.
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_1809_10585_b200/csrc/hq_common.cuh"
#include "../paper_1809_10585_b200/csrc/hq_svd_kernel.cuh"
#include "../paper_1809_10585_b200/csrc/hq_svd_cluster.cuh"
__device__ __forceinline__ double rcp_ap(double x) { double r; asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x)); return r; }
__device__ __forceinline__ double rsq_ap(double x) { double r; asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x)); return r; }
__device__ __forceinline__ double tan2(double a, double b, double g) {
  const double d = b - a;
  const double h = fabs(d) * (0.5 * rcp_ap(fabs(g)));
  const double w = fma(h, h, 1.0);
  double t = h < 1e150 ? rcp_ap(fma(w, rsq_ap(w), h)) : 0.5 * rcp_ap(h);
  return ((d >= 0.0) == (g > 0.0)) ? t : -t;
}
template <int LP, int E, bool FAST>
__device__ __forceinline__ bool rot2(double (&xp)[E], double* cy, double& a, double& b, int ld, double tol2,
                                     double tiny2, double thr2, int gl, bool act) {
  double xq[E];
  const bool work = act && !(a + b < thr2) && !(a < tiny2 && b < tiny2);
  double g0 = 0.0, g1 = 0.0, g2 = 0.0, g3 = 0.0;
#pragma unroll
  for (int e = 0; e < E / 2; ++e) {
    const int i = 2 * gl + 2 * LP * e;
    double2 vq = make_double2(0.0, 0.0);
    if (work && i < ld) vq = *reinterpret_cast<const double2*>(cy + i);
    xq[2 * e] = vq.x; xq[2 * e + 1] = vq.y;
    if (e & 1) { g2 = fma(xp[2 * e], vq.x, g2); g3 = fma(xp[2 * e + 1], vq.y, g3); }
    else { g0 = fma(xp[2 * e], vq.x, g0); g1 = fma(xp[2 * e + 1], vq.y, g1); }
  }
  double g = (g0 + g1) + (g2 + g3);
#pragma unroll
  for (int o = LP / 2; o > 0; o >>= 1) g += __shfl_xor_sync(0xffffffffu, g, o);
  const bool rot = work && g != 0.0 && g * g > tol2 * (a * b);
  if (rot) {
    const double tt = FAST ? tan2(a, b, g) : jacobi_tan(a, b, g);
    const double c = rsqrt(fma(tt, tt, 1.0)), sn = c * tt;
#pragma unroll
    for (int e = 0; e < E / 2; ++e) {
      const int i = 2 * gl + 2 * LP * e;
      const double x0 = xp[2 * e], x1 = xp[2 * e + 1];
      xp[2 * e] = c * x0 - sn * xq[2 * e];
      xp[2 * e + 1] = c * x1 - sn * xq[2 * e + 1];
      if (i < ld)
        *reinterpret_cast<double2*>(cy + i) = make_double2(sn * x0 + c * xq[2 * e], sn * x1 + c * xq[2 * e + 1]);
    }
    a = fmax(a - tt * g, 0.0);
    b = b + tt * g;
  }
  return rot;
}
template <int LP, int E>
__device__ __forceinline__ void rot_inst(double (&xp)[E], double* cy, double& a, double& b, int ld, double tol2,
                                     double tiny2, double thr2, int gl, long long* acc) {
  long long t0 = clock64();
  double xq[E];
  const bool work = !(a + b < thr2) && !(a < tiny2 && b < tiny2);
  double g0 = 0.0, g1 = 0.0, g2 = 0.0, g3 = 0.0;
#pragma unroll
  for (int e = 0; e < E / 2; ++e) {
    const int i = 2 * gl + 2 * LP * e;
    double2 vq = make_double2(0.0, 0.0);
    if (work && i < ld) vq = *reinterpret_cast<const double2*>(cy + i);
    xq[2 * e] = vq.x; xq[2 * e + 1] = vq.y;
    if (e & 1) { g2 = fma(xp[2 * e], vq.x, g2); g3 = fma(xp[2 * e + 1], vq.y, g3); }
    else { g0 = fma(xp[2 * e], vq.x, g0); g1 = fma(xp[2 * e + 1], vq.y, g1); }
  }
  double g = (g0 + g1) + (g2 + g3);
  if (g == 12345.0) xp[0] = 1.0;
  long long t1 = clock64();
#pragma unroll
  for (int o = LP / 2; o > 0; o >>= 1) g += __shfl_xor_sync(0xffffffffu, g, o);
  const bool rot = work && g != 0.0 && g * g > tol2 * (a * b);
  if (g == 12345.0) xp[0] = 1.0;
  long long t2 = clock64();
  double tt = tan2(a, b, g);
  if (tt == 12345.0) xp[0] = 1.0;
  long long t3 = clock64();
  const double c = rsqrt(fma(tt, tt, 1.0)), sn = c * tt;
  if (c == 12345.0) xp[0] = 1.0;
  long long t4 = clock64();
  if (rot) {
#pragma unroll
    for (int e = 0; e < E / 2; ++e) {
      const int i = 2 * gl + 2 * LP * e;
      const double x0 = xp[2 * e], x1 = xp[2 * e + 1];
      xp[2 * e] = c * x0 - sn * xq[2 * e];
      xp[2 * e + 1] = c * x1 - sn * xq[2 * e + 1];
      if (i < ld)
        *reinterpret_cast<double2*>(cy + i) = make_double2(sn * x0 + c * xq[2 * e], sn * x1 + c * xq[2 * e + 1]);
    }
    a = fmax(a - tt * g, 0.0);
    b = b + tt * g;
  }
  if (xp[E - 1] == 12345.0) xp[0] = 1.0;
  long long t5 = clock64();
  acc[0] += t1 - t0; acc[1] += t2 - t1; acc[2] += t3 - t2; acc[3] += t4 - t3; acc[4] += t5 - t4; acc[5] += rot;
}
template <int LP, int E, int MODE>
__global__ void k(double* out, long long* cyc, int iters, int nact, int ld) {
  __shared__ __align__(16) double sm[256 * 20];
  const int lane = threadIdx.x & 31, gl = lane % LP, grp = threadIdx.x / LP;
  const bool work = (threadIdx.x >> 5) < nact;
  for (int i = threadIdx.x; i < 256 * 20; i += blockDim.x) sm[i] = 1.0 / (i + 3);
  __syncthreads();
  double xp[E];
  double* cy = sm + (grp % 20) * 256;
#pragma unroll
  for (int e = 0; e < E; ++e) xp[e] = 0.5 + e * 1e-3 * lane;
  double a = 3.0;
  long long acc[6] = {0, 0, 0, 0, 0, 0};
  const long long c0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (work) {
      double bb = 2.0;
      if (MODE == 0) rotate_reg<LP, E>(xp, cy, a, bb, ld, 1e-28, 1e-30, 1e-20, gl, true);
      else if (MODE == 1) rot2<LP, E, false>(xp, cy, a, bb, ld, 1e-28, 1e-30, 1e-20, gl, true);
      else if (MODE == 2) rot2<LP, E, true>(xp, cy, a, bb, ld, 1e-28, 1e-30, 1e-20, gl, true);
      else rot_inst<LP, E>(xp, cy, a, bb, ld, 1e-28, 1e-30, 1e-20, gl, acc);
      a = 3.0 + 1e-3 * bb;
    }
    __syncthreads();
  }
  const long long c1 = clock64();
  if (threadIdx.x == 0) cyc[MODE] = (c1 - c0) / iters;
  if (MODE == 3 && threadIdx.x == 0) for (int q = 0; q < 6; ++q) cyc[4 + q] = acc[q] / iters;
  double s = a;
  for (int e = 0; e < E; ++e) s += xp[e];
  out[threadIdx.x] = s;
}
template <int LP, int E>
void run(double* out, long long* cyc, int ld) {
  for (int na : {1, 4, 8, 16}) {
    k<LP, E, 0><<<1, 512>>>(out, cyc, 2000, na, ld);
    k<LP, E, 1><<<1, 512>>>(out, cyc, 2000, na, ld);
    k<LP, E, 2><<<1, 512>>>(out, cyc, 2000, na, ld);
    k<LP, E, 3><<<1, 512>>>(out, cyc, 2000, na, ld);
    cudaDeviceSynchronize();
    printf("   inst: dot %lld shfl %lld tan %lld rsqrt %lld rot %lld (rot frac %lld/2000) total %lld\n", cyc[4], cyc[5], cyc[6], cyc[7], cyc[8], cyc[9]*1, cyc[3]);
    printf("LP %2d E %2d ld %3d warps %2d (pairs %3d): cur %lld  acc4 %lld  acc4+fasttan %lld\n", LP, E, ld, na, na * 32 / LP,
           cyc[0], cyc[1], cyc[2]);
  }
}
int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 1024 * 8); cudaMallocManaged(&cyc, 16 * 8);
  run<8, 16>(out, cyc, 128); run<16, 16>(out, cyc, 208); run<16, 8>(out, cyc, 128);
  run<32, 8>(out, cyc, 208); run<32, 4>(out, cyc, 128); 
  return 0;
}
