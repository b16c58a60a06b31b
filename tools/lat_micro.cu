// latency of dependent DMMA / DFMA chains (one warp)
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, int iters, long long* cyc) {
  double d0 = threadIdx.x, d1 = 1.0, a = 1.0000001, b = 0.999;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i)
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n" : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
  long long t1 = clock64();
  double x = d0;
  for (int i = 0; i < iters; ++i) x = fma(x, a, b);
  long long t2 = clock64();
  double y = x;
  for (int i = 0; i < iters; ++i) y += __shfl_xor_sync(0xffffffffu, y, 1);
  long long t3 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; }
  out[threadIdx.x] = d0 + d1 + x + y;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 256 * 8); cudaMallocManaged(&c, 3 * 8);
  for (int r = 0; r < 2; ++r) { k<<<1, 32>>>(o, 1000, c); cudaDeviceSynchronize(); }
  printf("DMMA dep latency %.1f cyc, DFMA %.1f cyc, SHFL+DADD %.1f cyc\n", c[0] / 1000.0, c[1] / 1000.0, c[2] / 1000.0);
  return 0;
}
