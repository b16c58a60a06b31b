// Shared device helpers for the B200 HODLR-QR kernels (FP64, column-major).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include "../../include/hodlrqr_b200.h"

#define HQ_DEV __device__ __forceinline__

// dimension (d, d_ri): rank[d_ri] clamped to [0, d] when d_ri >= 0, else d
HQ_DEV int hq_dim(const int* rank, int d, int ri) {
  if (ri < 0) return d;
  int v = rank[ri];
  return v < 0 ? 0 : (v > d ? d : v);
}

HQ_DEV double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// block-wide sum; `red` must hold >= 32 doubles; result broadcast to all threads
HQ_DEV double block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  double s = 0.0;
  if (wid == 0) {
    s = lane < nw ? red[lane] : 0.0;
    s = warp_sum(s);
    if (lane == 0) red[0] = s;
  }
  __syncthreads();
  s = red[0];
  return s;
}

// value of a stored matrix element under a triangular mask
HQ_DEV double hq_mask(double v, int r, int c, int mask) {
  if (mask == 1) return r <= c ? v : 0.0;              // upper incl. diagonal
  if (mask == 2) return r > c ? v : (r == c ? 1.0 : 0.0);  // unit lower
  return v;
}

static inline int hq_err(cudaError_t e) { return (int)e; }
