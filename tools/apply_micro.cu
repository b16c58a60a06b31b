// Cycle breakdown of apply_panel_cols on shared-memory operands (one CTA).
#define HQ_DEBUG_TIMING 1
#include "../paper_1809_10585_b200/csrc/hq_qr.cu"
#include <cstdio>
__global__ void __launch_bounds__(NT) k(int rows, int ncols, long long* cyc) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  QrSmem& S = *reinterpret_cast<QrSmem*>(smem_raw);
  const int ld = pad_ld(rows);
  for (int i = threadIdx.x; i < ld * 16; i += NT) { S.ybuf[i] = 1.0 / (i + 1); S.panel[i] = 1.0 / (i + 2); }
  if (threadIdx.x < 256) S.tp[threadIdx.x] = 0.01;
  __syncthreads();
  const long long c0 = clock64();
  for (int rep = 0; rep < 10; ++rep)
    apply_panel_cols(S.ybuf, ld, rows, 16, S.tp, S.panel, ld, ncols, true, S);
  const long long c1 = clock64();
  if (threadIdx.x == 0) *cyc = (c1 - c0) / 10;
}
int main() {
  long long* dbg; long long* cyc;
  cudaMalloc(&dbg, 4096 * 8); cudaMemset(dbg, 0, 4096 * 8);
  cudaMemcpyToSymbol(hq_dbg, &dbg, sizeof(dbg));
  cudaMallocManaged(&cyc, 8);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(QrSmem));
  for (int rows : {128, 256, 400}) {
    cudaMemset(dbg, 0, 4096 * 8);
    k<<<1, NT, sizeof(QrSmem)>>>(rows, 16, cyc);
    cudaDeviceSynchronize();
    long long h[4096];
    cudaMemcpy(h, dbg, sizeof(h), cudaMemcpyDeviceToHost);
    printf("rows %d cols 16: total %lld cycles/call; W %lld T %lld X %lld (err %s)\n", rows, *cyc,
           h[2048] / max(1LL, h[2064]), h[2049] / max(1LL, h[2065]), h[2050] / max(1LL, h[2066]),
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
