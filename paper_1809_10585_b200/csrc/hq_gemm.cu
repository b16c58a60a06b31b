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
// Skinny variant for outputs with few columns (n <= NC) and long K (the
// power-iteration products: blocks^T X with 2 vectors, the 2x2 Gram): a
// CTA owns a K-slice of one problem, its threads stride over k and keep an
// MB x NC accumulator chunk in registers; the chunk is reduced over the CTA
// (shuffles + shared memory) and added to C (atomically when K is split).
// A 64x64 tile would waste its shared-memory traffic on 2 live columns.
template <int MB, int NC>
__global__ void __launch_bounds__(NT) gemm_skinny_kernel(const hq_gemm_prob* __restrict__ probs,
                                                         const hq_gemm_term* __restrict__ terms,
                                                         const int* __restrict__ rank, int ksplit,
                                                         const int* __restrict__ skip) {
  if (skip && *skip) return;
  const hq_gemm_prob P = probs[blockIdx.y];
  const int m = hq_dim(rank, P.m, P.m_ri), n = hq_dim(rank, P.n, P.n_ri);
  if (m <= 0 || n <= 0) return;
  const int z = blockIdx.x, ks = ksplit;
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  __shared__ double red[NT / 32][MB * NC];
  for (int i0 = 0; i0 < m; i0 += MB) {
    for (int j0 = 0; j0 < n; j0 += NC) {
      double acc[MB][NC];
#pragma unroll
      for (int ii = 0; ii < MB; ++ii)
#pragma unroll
        for (int jj = 0; jj < NC; ++jj) acc[ii][jj] = 0.0;
      for (int ti = 0; ti < P.nterm; ++ti) {
        const hq_gemm_term T = terms[P.term0 + ti];
        const int kd = hq_dim(rank, T.k, T.k_ri);
        const int kb = (int)(((long long)kd * z) / ks), ke = (int)(((long long)kd * (z + 1)) / ks);
        for (int k = kb + t; k < ke; k += NT) {
          double bv[NC];
#pragma unroll
          for (int jj = 0; jj < NC; ++jj) {
            const int j = j0 + jj;
            double v = 0.0;
            if (j < n) v = T.tb == 0 ? hq_mask(T.b[k + (size_t)j * T.ldb], k, j, T.mask_b)
                                     : hq_mask(T.b[j + (size_t)k * T.ldb], j, k, T.mask_b);
            bv[jj] = v * T.alpha;
          }
#pragma unroll
          for (int ii = 0; ii < MB; ++ii) {
            const int i = i0 + ii;
            double a = 0.0;
            if (i < m) a = T.ta == 0 ? hq_mask(T.a[i + (size_t)k * T.lda], i, k, T.mask_a)
                                     : hq_mask(T.a[k + (size_t)i * T.lda], k, i, T.mask_a);
#pragma unroll
            for (int jj = 0; jj < NC; ++jj) acc[ii][jj] = fma(a, bv[jj], acc[ii][jj]);
          }
        }
      }
#pragma unroll
      for (int ii = 0; ii < MB; ++ii)
#pragma unroll
        for (int jj = 0; jj < NC; ++jj) {
          const double v = warp_sum(acc[ii][jj]);
          if (lane == 0) red[wid][ii * NC + jj] = v;
        }
      __syncthreads();
      if (t < MB * NC) {
        double v = 0.0;
#pragma unroll
        for (int w = 0; w < NT / 32; ++w) v += red[w][t];
        const int i = i0 + t / NC, j = j0 + t % NC;
        if (i < m && j < n) {
          double* cp = P.c + i + (size_t)j * P.ldc;
          if (ks > 1) atomicAdd(cp, v);
          else *cp = (P.beta == 0.0) ? v : fma(P.beta, *cp, v);
        }
      }
      __syncthreads();
    }
  }
}
// Row variant of the skinny product for tall outputs (m rows, n <= NC
// columns, moderate K): a CTA owns 32 output rows (one per lane) and its 8
// warps split K; each lane keeps NC accumulators, the warps' partials are
// summed through shared memory.  A's columns are read 256 B per warp load.
template <int NC>
__global__ void __launch_bounds__(NT) gemm_rows_kernel(const hq_gemm_prob* __restrict__ probs,
                                                       const hq_gemm_term* __restrict__ terms,
                                                       const int* __restrict__ rank,
                                                       const int* __restrict__ skip) {
  if (skip && *skip) return;
  const hq_gemm_prob P = probs[blockIdx.y];
  const int m = hq_dim(rank, P.m, P.m_ri), n = hq_dim(rank, P.n, P.n_ri);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int i = blockIdx.x * 32 + lane;
  if (n <= 0 || blockIdx.x * 32 >= m) return;
  __shared__ double red[NT / 32][32 * NC];
  for (int j0 = 0; j0 < n; j0 += NC) {
    double acc[NC];
#pragma unroll
    for (int jj = 0; jj < NC; ++jj) acc[jj] = 0.0;
    for (int ti = 0; ti < P.nterm; ++ti) {
      const hq_gemm_term T = terms[P.term0 + ti];
      const int kd = hq_dim(rank, T.k, T.k_ri);
      const int ic = i < m ? i : 0;
#pragma unroll 4
      for (int k = wid; k < kd; k += NT / 32) {
        double a = T.ta == 0 ? hq_mask(T.a[ic + (size_t)k * T.lda], ic, k, T.mask_a)
                             : hq_mask(T.a[k + (size_t)ic * T.lda], k, ic, T.mask_a);
        a *= T.alpha;
#pragma unroll
        for (int jj = 0; jj < NC; ++jj) {
          const int j = j0 + jj < n ? j0 + jj : n - 1;
          const double b = T.tb == 0 ? hq_mask(T.b[k + (size_t)j * T.ldb], k, j, T.mask_b)
                                     : hq_mask(T.b[j + (size_t)k * T.ldb], j, k, T.mask_b);
          acc[jj] = fma(a, b, acc[jj]);
        }
      }
    }
#pragma unroll
    for (int jj = 0; jj < NC; ++jj) red[wid][lane * NC + jj] = acc[jj];
    __syncthreads();
    if (threadIdx.x < 32 * NC) {
      const int l = threadIdx.x / NC, jj = threadIdx.x % NC;
      double v = 0.0;
#pragma unroll
      for (int w = 0; w < NT / 32; ++w) v += red[w][threadIdx.x];
      const int ii = blockIdx.x * 32 + l, j = j0 + jj;
      if (ii < m && j < n) {
        double* cp = P.c + ii + (size_t)j * P.ldc;
        *cp = (P.beta == 0.0) ? v : fma(P.beta, *cp, v);
      }
    }
    __syncthreads();
  }
}
}  // namespace

// skinny products (n <= 4 output columns).  mode 0: grid (ksplit, nprob),
// threads split K; mode 1: grid (ceil(m/256), nprob), one thread per row
// (ksplit ignored)
extern "C" int hq_gemm_skinny(void* stream, const hq_gemm_prob* probs, int nprob,
                              const hq_gemm_term* terms, int* rank, int ksplit, int ncmax, int mode,
                              int max_rows, const int* skip) {
  if (nprob <= 0) return 0;
  if (ksplit < 1) ksplit = 1;
  cudaStream_t st = (cudaStream_t)stream;
  if (mode == 1) {
    dim3 grid((max_rows + 31) / 32, nprob);
    if (ncmax <= 2) gemm_rows_kernel<2><<<grid, NT, 0, st>>>(probs, terms, rank, skip);
    else gemm_rows_kernel<4><<<grid, NT, 0, st>>>(probs, terms, rank, skip);
    return hq_err(cudaGetLastError());
  }
  dim3 grid(ksplit, nprob);
  if (ncmax <= 2) gemm_skinny_kernel<16, 2><<<grid, NT, 0, st>>>(probs, terms, rank, ksplit, skip);
  else gemm_skinny_kernel<8, 4><<<grid, NT, 0, st>>>(probs, terms, rank, ksplit, skip);
  return hq_err(cudaGetLastError());
}

extern "C" int hq_gemm(void* stream, const hq_gemm_prob* probs, int nprob,
                       const hq_gemm_term* terms, int* rank, int tiles, int ksplit,
                       const int* skip) {
  if (nprob <= 0 || tiles <= 0) return 0;
  if (ksplit < 1) ksplit = 1;
  dim3 grid(tiles, nprob, ksplit);
  gemm_kernel<<<grid, NT, 0, (cudaStream_t)stream>>>(probs, terms, rank, ksplit, skip);
  return hq_err(cudaGetLastError());
}
