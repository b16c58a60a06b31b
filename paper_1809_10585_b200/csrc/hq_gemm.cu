// Batched multi-term FP64 GEMM with run-time (rank-table) dimensions.
//   C (m x n) = beta*C + sum_t alpha_t * op(A_t) * op(B_t)
// Used for every dense/low-rank product of the hQR recursion: both phases of
// HODLR x dense (arith.py:35-64), the cross/slab updates (hqr.py:156-159),
// the leaf low-rank updates (arith.py:136) and the truncation cores.
// 64x64 output tile per CTA, 256 threads, 4x4 register micro-tile, K-step 16.
#include "hq_common.cuh"

namespace {
constexpr int BM = 64, BN = 64, BK = 16, NT = 256;

__global__ void __launch_bounds__(NT) gemm_kernel(const hq_gemm_prob* __restrict__ probs,
                                                  const hq_gemm_term* __restrict__ terms,
                                                  const int* __restrict__ rank, int ksplit,
                                                  const int* __restrict__ skip) {
  if (skip && *skip) return;
  const hq_gemm_prob P = probs[blockIdx.y];
  const int m = hq_dim(rank, P.m, P.m_ri), n = hq_dim(rank, P.n, P.n_ri);
  if (m <= 0 || n <= 0) return;
  const int ntm = (m + BM - 1) / BM, ntn = (n + BN - 1) / BN;
  const int tile = blockIdx.x;
  if (tile >= ntm * ntn) return;
  const int i0 = (tile % ntm) * BM, j0 = (tile / ntm) * BN;
  // per-problem split: at least 8 k-tiles per slice (short-K problems of a
  // split launch keep one slice; the output was pre-zeroed either way)
  int ks = ksplit;
  if (ksplit > 1) {
    int nkt = 0;
    for (int ti = 0; ti < P.nterm; ++ti) {
      const hq_gemm_term T = terms[P.term0 + ti];
      nkt += (hq_dim(rank, T.k, T.k_ri) + BK - 1) / BK;
    }
    ks = min(ksplit, max(1, nkt / 8));
    if ((int)blockIdx.z >= ks) return;
  }

  __shared__ double As[BK][BM + 1];
  __shared__ double Bs[BK][BN + 1];
  const int t = threadIdx.x, tx = t & 15, ty = t >> 4;
  double acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;

  int gk = 0;  // global k-tile counter across terms (split-K striping)
  for (int ti = 0; ti < P.nterm; ++ti) {
    const hq_gemm_term T = terms[P.term0 + ti];
    const int kd = hq_dim(rank, T.k, T.k_ri);
    for (int k0 = 0; k0 < kd; k0 += BK, ++gk) {
      if (ks > 1 && (gk % ks) != (int)blockIdx.z) continue;
      // ---- A tile: op(A)(i, kk)
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        int ii, kk;
        if (T.ta == 0) { ii = t & 63; kk = (t >> 6) + 4 * r; }
        else { kk = t & 15; ii = (t >> 4) + 16 * r; }
        const int gi = i0 + ii, gkk = k0 + kk;
        double v = 0.0;
        if (gi < m && gkk < kd) {
          if (T.ta == 0) v = hq_mask(T.a[gi + (size_t)gkk * T.lda], gi, gkk, T.mask_a);
          else v = hq_mask(T.a[gkk + (size_t)gi * T.lda], gkk, gi, T.mask_a);
        }
        As[kk][ii] = v;
      }
      // ---- B tile: op(B)(kk, j)
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        int jj, kk;
        if (T.tb == 0) { kk = t & 15; jj = (t >> 4) + 16 * r; }
        else { jj = t & 63; kk = (t >> 6) + 4 * r; }
        const int gj = j0 + jj, gkk = k0 + kk;
        double v = 0.0;
        if (gj < n && gkk < kd) {
          if (T.tb == 0) v = hq_mask(T.b[gkk + (size_t)gj * T.ldb], gkk, gj, T.mask_b);
          else v = hq_mask(T.b[gj + (size_t)gkk * T.ldb], gj, gkk, T.mask_b);
        }
        Bs[kk][jj] = v * T.alpha;
      }
      __syncthreads();
#pragma unroll
      for (int kk = 0; kk < BK; ++kk) {
        double av[4], bv[4];
#pragma unroll
        for (int a = 0; a < 4; ++a) av[a] = As[kk][tx + 16 * a];
#pragma unroll
        for (int b = 0; b < 4; ++b) bv[b] = Bs[kk][ty + 16 * b];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) acc[a][b] = fma(av[a], bv[b], acc[a][b]);
      }
      __syncthreads();
    }
  }
  // ---- epilogue
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const int gi = i0 + tx + 16 * a;
    if (gi >= m) continue;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int gj = j0 + ty + 16 * b;
      if (gj >= n) continue;
      double* cp = P.c + gi + (size_t)gj * P.ldc;
      if (ksplit > 1) atomicAdd(cp, acc[a][b]);
      else *cp = (P.beta == 0.0) ? acc[a][b] : fma(P.beta, *cp, acc[a][b]);
    }
  }
}
}  // namespace

extern "C" int hq_gemm(void* stream, const hq_gemm_prob* probs, int nprob,
                       const hq_gemm_term* terms, int* rank, int tiles, int ksplit,
                       const int* skip) {
  if (nprob <= 0 || tiles <= 0) return 0;
  if (ksplit < 1) ksplit = 1;
  dim3 grid(tiles, nprob, ksplit);
  gemm_kernel<<<grid, NT, 0, (cudaStream_t)stream>>>(probs, terms, rank, ksplit, skip);
  return hq_err(cudaGetLastError());
}
