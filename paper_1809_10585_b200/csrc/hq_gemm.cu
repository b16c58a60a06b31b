// Batched multi-term FP64 GEMM with run-time (rank-table) dimensions.
//   C (m x n) = beta*C + sum_t alpha_t * op(A_t) * op(B_t)
// Used for every dense/low-rank product of the hQR recursion: both phases of
// HODLR x dense (arith.py:35-64), the cross/slab updates (hqr.py:156-159),
// the leaf low-rank updates (arith.py:136) and the truncation cores.
// 64x64 output tile per CTA, 256 threads, 4x4 register micro-tile, K-step 16.
#include "hq_common.cuh"

namespace {
#ifndef HQ_GEMM_BK
#define HQ_GEMM_BK 16
#endif
constexpr int NT = 256, BK = HQ_GEMM_BK;

// async 8-byte copy with zero fill when !valid (src-size 0)
__device__ __forceinline__ void cp_async8_zfill(void* smem, const void* gmem, bool valid) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  const int sz = valid ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(gmem), "r"(sz) : "memory");
}
// 16-byte copy of which the first `bytes` (0, 8 or 16) come from global
// memory, the rest zero; both addresses 16-byte aligned
__device__ __forceinline__ void cp_async16_zfill(void* smem, const void* gmem, int bytes) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gmem), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// FP64 tensor-core GEMM, BM x BN output tile per CTA, WM x WN warps (each a
// (BM/WM) x (BN/WN) block of m8n8 tiles), k-tiles of BK staged in shared
// memory with asynchronous copies, STAGES deep (the next STAGES-1 k-tiles are
// in flight while the current one runs on mma.sync.m8n8k4).  Operands are staged in
// their raw layout as op(A)[k][i], op(B)[k][j] with leading dims == 4 mod 16
// (bank-conflict-free fragment fetches); masks and alpha are applied by the
// thread that copied the element, before the barrier that publishes the tile.
template <int BM, int BN, int WM, int WN, int STAGES>
__global__ void __launch_bounds__(WM * WN * 32, BM == 64 ? 3 : 4) gemm_kernel(const hq_gemm_prob* __restrict__ probs,
                                                            const hq_gemm_term* __restrict__ terms,
                                                            const int* __restrict__ rank, int ksplit,
                                                            const int* __restrict__ skip) {
  constexpr int NTH = WM * WN * 32;
  constexpr int LDA = BM + 4, LDB = BN + 4;
  constexpr int TM = BM / WM / 8, TN = BN / WN / 8;   // m8n8 tiles per warp
  constexpr int EA = BM * BK / NTH, EB = BN * BK / NTH;  // staged elements per thread
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
  int ks = 1, ks_cap = 1;
  if (ksplit > 1) {
    int nkt = 0, nkt_cap = 0;
    for (int ti = 0; ti < P.nterm; ++ti) {
      const hq_gemm_term& T = terms[P.term0 + ti];
      nkt += (hq_dim(rank, T.k, T.k_ri) + BK - 1) / BK;
      nkt_cap += (T.k + BK - 1) / BK;
    }
    ks = min(ksplit, max(1, nkt / 8));
    ks_cap = min(ksplit, max(1, nkt_cap / 8));
    if ((int)blockIdx.z >= ks) return;
  }

  // staged tile of op(A): layout 0 = [k][i] (ld LDA), layout 1 = [i][k] (ld
  // LDT) for operands whose k runs contiguously in memory (A with ta = 1, B
  // with tb = 0), so that those too are copied 16 bytes at a time.  LDT = 20:
  // the m8n8k4 fragment fetch (8 rows x 4 k) touches 8-byte banks 4 gq + tq
  // (mod 16): two wavefronts per warp, the minimum for 256 bytes
  extern __shared__ __align__(16) double gsm[];
  constexpr int LDT = BK + 4;
  constexpr int ASZ = BK * LDA > BM * LDT ? BK * LDA : BM * LDT;
  constexpr int BSZ = BK * LDB > BN * LDT ? BK * LDB : BN * LDT;
  double* const Asf = gsm;
  double* const Bsf = gsm + STAGES * ASZ;
  auto aidx = [&](int buf, bool tr, int kk, int ii) { return buf * ASZ + (tr ? ii * LDT + kk : kk * LDA + ii); };
  auto bidx = [&](int buf, bool tr, int kk, int jj) { return buf * BSZ + (tr ? jj * LDT + kk : kk * LDB + jj); };
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  const int gq = lane >> 2, tq = lane & 3;
  const int wm = wid % WM, wn = wid / WM;
  double acc[TM][TN][2];
#pragma unroll
  for (int a = 0; a < TM; ++a)
#pragma unroll
    for (int b = 0; b < TN; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

  // flat sequence of this CTA's k-tiles: (term, k0)
  int ti = 0, k0 = 0, gk = 0;
  auto advance = [&](int& ti_, int& k0_, int& gk_) {
    // move to the next k-tile of this slice (ti_ == nterm: none left)
    for (;;) {
      k0_ += BK;
      if (ti_ >= P.nterm) return;
      const int kd = hq_dim(rank, terms[P.term0 + ti_].k, terms[P.term0 + ti_].k_ri);
      if (k0_ >= kd) { ++ti_; k0_ = -BK; continue; }
      ++gk_;   // a real k-tile of the problem (split-K striping counter)
      if (ks > 1 && (gk_ % ks) != (int)blockIdx.z) continue;
      return;
    }
  };
  // position on the first k-tile of the slice
  {
    ti = 0; k0 = -BK; gk = -1;
    advance(ti, k0, gk);
  }
  // element e of this thread's share of a staged k-tile -> (row/col, k).
  // Copy modes: 0 / 1 element by element (ta or tb = 0 / 1), 2 / 3 in pairs by
  // one 16-byte cp.async when the operand is 16-byte aligned with an even
  // leading dimension: 2 = pairs along the row index (A with ta = 0, B with
  // tb = 1; layout [k][row]), 3 = pairs along k (A with ta = 1, B with
  // tb = 0; layout [row][k]).
  auto a_elem = [&](int e, int mode, int& ii, int& kk) {
    if (mode == 2) { const int p = t + (e >> 1) * NTH; ii = 2 * (p % (BM / 2)) + (e & 1); kk = p / (BM / 2); }
    else if (mode == 3) { const int p = t + (e >> 1) * NTH; kk = 2 * (p % (BK / 2)) + (e & 1); ii = p / (BK / 2); }
    else if (mode == 0) { const int idx = t + e * NTH; ii = idx % BM; kk = idx / BM; }
    else { const int idx = t + e * NTH; kk = idx % BK; ii = idx / BK; }
  };
  auto b_elem = [&](int e, int mode, int& jj, int& kk) {
    if (mode == 2) { const int p = t + (e >> 1) * NTH; jj = 2 * (p % (BN / 2)) + (e & 1); kk = p / (BN / 2); }
    else if (mode == 3) { const int p = t + (e >> 1) * NTH; kk = 2 * (p % (BK / 2)) + (e & 1); jj = p / (BK / 2); }
    else if (mode == 0) { const int idx = t + e * NTH; kk = idx % BK; jj = idx / BK; }
    else { const int idx = t + e * NTH; jj = idx % BN; kk = idx / BN; }
  };
  auto mode_a = [&](const hq_gemm_term& T) {
    const bool al = (((uintptr_t)T.a & 15) == 0) && (T.lda & 1) == 0;
    return T.ta == 0 ? (al ? 2 : 0) : (al ? 3 : 1);
  };
  auto mode_b = [&](const hq_gemm_term& T) {
    const bool al = (((uintptr_t)T.b & 15) == 0) && (T.ldb & 1) == 0;
    return T.tb != 0 ? (al ? 2 : 1) : (al ? 3 : 0);
  };
  bool la[STAGES], lb[STAGES];   // layout of the tile in each ring buffer
  auto stage = [&](int buf, int ti_, int k0_) {
    const hq_gemm_term T = terms[P.term0 + ti_];
    const int kd = hq_dim(rank, T.k, T.k_ri);
    const int ma = mode_a(T), mb = mode_b(T);
    la[buf] = ma == 3;
    lb[buf] = mb == 3;
    if (ma == 2) {
#pragma unroll
      for (int e = 0; e < EA; e += 2) {
        int ii, kk;
        a_elem(e, 2, ii, kk);
        const int gi = i0 + ii, gkk = k0_ + kk;
        const int nv = gkk < kd ? min(max(m - gi, 0), 2) : 0;
        cp_async16_zfill(Asf + aidx(buf, false, kk, ii), T.a + (nv ? gi + (size_t)gkk * T.lda : 0), 8 * nv);
      }
    } else if (ma == 3) {
#pragma unroll
      for (int e = 0; e < EA; e += 2) {
        int ii, kk;
        a_elem(e, 3, ii, kk);
        const int gi = i0 + ii, gkk = k0_ + kk;
        const int nv = gi < m ? min(max(kd - gkk, 0), 2) : 0;
        cp_async16_zfill(Asf + aidx(buf, true, kk, ii), T.a + (nv ? gkk + (size_t)gi * T.lda : 0), 8 * nv);
      }
    } else {
#pragma unroll
      for (int e = 0; e < EA; ++e) {
        int ii, kk;
        a_elem(e, ma, ii, kk);
        const int gi = i0 + ii, gkk = k0_ + kk;
        const bool ok = gi < m && gkk < kd;
        const double* src = T.ta == 0 ? T.a + (ok ? gi + (size_t)gkk * T.lda : 0)
                                      : T.a + (ok ? gkk + (size_t)gi * T.lda : 0);
        cp_async8_zfill(Asf + aidx(buf, false, kk, ii), src, ok);
      }
    }
    if (mb == 2) {
#pragma unroll
      for (int e = 0; e < EB; e += 2) {
        int jj, kk;
        b_elem(e, 2, jj, kk);
        const int gj = j0 + jj, gkk = k0_ + kk;
        const int nv = gkk < kd ? min(max(n - gj, 0), 2) : 0;
        cp_async16_zfill(Bsf + bidx(buf, false, kk, jj), T.b + (nv ? gj + (size_t)gkk * T.ldb : 0), 8 * nv);
      }
    } else if (mb == 3) {
#pragma unroll
      for (int e = 0; e < EB; e += 2) {
        int jj, kk;
        b_elem(e, 3, jj, kk);
        const int gj = j0 + jj, gkk = k0_ + kk;
        const int nv = gj < n ? min(max(kd - gkk, 0), 2) : 0;
        cp_async16_zfill(Bsf + bidx(buf, true, kk, jj), T.b + (nv ? gkk + (size_t)gj * T.ldb : 0), 8 * nv);
      }
    } else {
#pragma unroll
      for (int e = 0; e < EB; ++e) {
        int jj, kk;
        b_elem(e, mb, jj, kk);
        const int gj = j0 + jj, gkk = k0_ + kk;
        const bool ok = gj < n && gkk < kd;
        const double* src = T.tb == 0 ? T.b + (ok ? gkk + (size_t)gj * T.ldb : 0)
                                      : T.b + (ok ? gj + (size_t)gkk * T.ldb : 0);
        cp_async8_zfill(Bsf + bidx(buf, false, kk, jj), src, ok);
      }
    }
  };
  // masks / alpha on the elements this thread staged (after they landed)
  auto fixup = [&](int buf, int ti_, int k0_) {
    const hq_gemm_term T = terms[P.term0 + ti_];
    if (T.mask_a != 0) {
      const int ma = mode_a(T);
#pragma unroll
      for (int e = 0; e < EA; ++e) {
        int ii, kk;
        a_elem(e, ma, ii, kk);
        const int gi = i0 + ii, gkk = k0_ + kk;
        double& v = Asf[aidx(buf, ma == 3, kk, ii)];
        v = T.ta == 0 ? hq_mask(v, gi, gkk, T.mask_a) : hq_mask(v, gkk, gi, T.mask_a);
      }
    }
    if (T.mask_b != 0 || T.alpha != 1.0) {
      const int mb = mode_b(T);
#pragma unroll
      for (int e = 0; e < EB; ++e) {
        int jj, kk;
        b_elem(e, mb, jj, kk);
        const int gj = j0 + jj, gkk = k0_ + kk;
        double& v = Bsf[bidx(buf, mb == 3, kk, jj)];
        const double w = T.tb == 0 ? hq_mask(v, gkk, gj, T.mask_b) : hq_mask(v, gj, gkk, T.mask_b);
        v = w * T.alpha;
      }
    }
  };

  // ring of STAGES buffers: tile s of the slice lives in buffer s % STAGES
  int sti[STAGES], sk0[STAGES];
  int pti = ti, pk0 = k0, pgk = gk;   // next tile to stage
#pragma unroll
  for (int q = 0; q < STAGES - 1; ++q) {
    sti[q] = pti; sk0[q] = pk0;
    if (pti < P.nterm) { stage(q, pti, pk0); advance(pti, pk0, pgk); }
    cp_async_commit();
  }
  int buf = 0;
  while (sti[buf] < P.nterm) {
    // stage tile (current + STAGES-1) into the buffer freed last iteration
    const int nb = (buf + STAGES - 1) % STAGES;
    sti[nb] = pti; sk0[nb] = pk0;
    if (pti < P.nterm) { stage(nb, pti, pk0); advance(pti, pk0, pgk); }
    cp_async_commit();
    cp_async_wait<STAGES - 1>();
    fixup(buf, sti[buf], sk0[buf]);
    __syncthreads();
    const bool tra = la[buf], trb = lb[buf];
    const double* Ab = Asf + buf * ASZ;
    const double* Bb = Bsf + buf * BSZ;
#pragma unroll
    for (int kq = 0; kq < BK; kq += 4) {
      double av[TM], bv[TN];
#pragma unroll
      for (int a = 0; a < TM; ++a) av[a] = Ab[tra ? ((wm * TM + a) * 8 + gq) * LDT + kq + tq : (kq + tq) * LDA + (wm * TM + a) * 8 + gq];
#pragma unroll
      for (int b = 0; b < TN; ++b) bv[b] = Bb[trb ? ((wn * TN + b) * 8 + gq) * LDT + kq + tq : (kq + tq) * LDB + (wn * TN + b) * 8 + gq];
#pragma unroll
      for (int a = 0; a < TM; ++a)
#pragma unroll
        for (int b = 0; b < TN; ++b) dmma884(acc[a][b][0], acc[a][b][1], av[a], bv[b]);
    }
    __syncthreads();   // this buffer is restaged next iteration
    buf = (buf + 1) % STAGES;
  }
  cp_async_wait<0>();
  // ---- epilogue: lane holds D[gq][2tq + {0,1}] of each m8n8 tile
  if (ks > 1) {
    // K-split: partial tile into this slice's slot; the last slice to arrive
    // sums the slots in slice order (deterministic)
    double* slot0 = P.ws + (size_t)tile * ks_cap * (BM * BN);
    double* mine = slot0 + (size_t)blockIdx.z * (BM * BN);
#pragma unroll
    for (int a = 0; a < TM; ++a)
#pragma unroll
      for (int b = 0; b < TN; ++b)
#pragma unroll
        for (int h = 0; h < 2; ++h)
          mine[(wm * TM + a) * 8 + gq + ((wn * TN + b) * 8 + 2 * tq + h) * BM] = acc[a][b][h];
    if (!hq_split_last(P.cnt + tile, ks)) return;
#pragma unroll
    for (int a = 0; a < TM; ++a)
#pragma unroll
      for (int b = 0; b < TN; ++b)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int e = (wm * TM + a) * 8 + gq + ((wn * TN + b) * 8 + 2 * tq + h) * BM;
          double v = 0.0;
          for (int z = 0; z < ks; ++z) v += __ldcg(slot0 + (size_t)z * (BM * BN) + e);
          acc[a][b][h] = v;
        }
  }
#pragma unroll
  for (int a = 0; a < TM; ++a) {
    const int gi = i0 + (wm * TM + a) * 8 + gq;
    if (gi >= m) continue;
#pragma unroll
    for (int b = 0; b < TN; ++b) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int gj = j0 + (wn * TN + b) * 8 + 2 * tq + h;
        if (gj >= n) continue;
        double* cp = P.c + gi + (size_t)gj * P.ldc;
        *cp = (P.beta == 0.0) ? acc[a][b][h] : fma(P.beta, *cp, acc[a][b][h]);
      }
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
          if (ks > 1) {
            P.ws[(size_t)z * P.m * P.n + i + (size_t)j * P.m] = v;
          } else {
            double* cp = P.c + i + (size_t)j * P.ldc;
            *cp = (P.beta == 0.0) ? v : fma(P.beta, *cp, v);
          }
        }
      }
      __syncthreads();
    }
  }
  // K-split: slot z = ws + z * m_cap * n_cap; the last slice sums in order
  if (ks > 1 && hq_split_last(P.cnt, ks)) {
    for (int e = t; e < m * n; e += NT) {
      const int i = e % m, j = e / m;
      double v = 0.0;
      for (int zz = 0; zz < ks; ++zz) v += __ldcg(P.ws + (size_t)zz * P.m * P.n + i + (size_t)j * P.m);
      double* cp = P.c + i + (size_t)j * P.ldc;
      *cp = (P.beta == 0.0) ? v : fma(P.beta, *cp, v);
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
// Streaming product for outputs of at most NC columns (the power iteration's
// HODLR x 2 vectors, arith.py:35-64 on a 2-column block): HBM-bound, so each
// term is read in its own coalesced pattern.  A CTA owns GV_ROWS output rows
// of one problem (blockIdx.x) and a K-slice (blockIdx.z):
//   op(A) = A   (ta = 0, column-major m x k): thread (row r, slice s) walks
//               k = s, s + 4, ...; a warp load covers 32 consecutive rows;
//   op(A) = A^T (ta = 1): row r of op(A) is a contiguous column of A: work
//               items (row, k-lane-group) spread over the 8 warps, lanes along
//               k, warp-shuffle reduction, shared-memory accumulation.
// B (k x NC) is tiny and read through the cache.  K-split slices add into C
// atomically (the caller zeroed C).
constexpr int GV_U = 8, GV_RQH = 4;
// output rows per CTA from the launch's tallest problem (plan.py gv_rows is
// the same rule): a 256-row leaf as ONE band reads whole 2 KB columns -- 64-row
// bands (512-byte pieces at a 2 KB stride, the four bands of a leaf on
// different SMs at different times) reached 4.4 TB/s, 128-row bands 5.4
__host__ __device__ constexpr int gv_rows(int max_rows) { return max_rows >= 256 ? 256 : (max_rows >= 128 ? 128 : 64); }
// KIND 0: terms of both layouts; 1: only op(A) = A; 2: only op(A) = A^T
// (the planner knows each launch's layouts; the lean variants keep fewer
// registers live and run more warps per SM)
template <int NC, int KIND, int GV_ROWS>
__global__ void __launch_bounds__(NT, NC == 2 ? 3 : 2) gemv_kernel(const hq_gemm_prob* __restrict__ probs,
                                                  const hq_gemm_term* __restrict__ terms,
                                                  const int* __restrict__ rank, int ksplit,
                                                  const int* __restrict__ skip) {
  if (skip && *skip) return;
  const hq_gemm_prob P = probs[blockIdx.y];
  const int m = hq_dim(rank, P.m, P.m_ri), n = hq_dim(rank, P.n, P.n_ri);
  const int i0 = blockIdx.x * GV_ROWS;
  if (m <= 0 || n <= 0 || i0 >= m) return;
  const int nr = min(GV_ROWS, m - i0);
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  const int z = blockIdx.z;
  __shared__ double part[NT / GV_ROWS][GV_ROWS][NC];
  // A^T-layout sums per k-lane group (a row is shared by up to 8 warps:
  // separate slots, added in a fixed order -- no shared-memory atomics)
  constexpr int DQ = GV_ROWS >= 256 ? 2 : 8;   // k-lane groups per row (few-row blocks only)
  __shared__ double dotr[DQ][GV_ROWS][NC];
  for (int e = t; e < DQ * GV_ROWS * NC; e += NT) (&dotr[0][0][0])[e] = 0.0;
  __syncthreads();
  const int r = t % GV_ROWS, sl = t / GV_ROWS;
  constexpr int NSL = NT / GV_ROWS;
  double acc[NC];
#pragma unroll
  for (int j = 0; j < NC; ++j) acc[j] = 0.0;
  // per-problem K split: slices of >= 512 k (the launch's ksplit bounds it)
  int ktot = 0, ktot_cap = 0;
  for (int ti = 0; ti < P.nterm; ++ti) {
    ktot += hq_dim(rank, terms[P.term0 + ti].k, terms[P.term0 + ti].k_ri);
    ktot_cap += terms[P.term0 + ti].k;
  }
  const int ks = min(ksplit, max(1, ktot / 512));
  const int ks_cap = min(ksplit, max(1, ktot_cap / 512));
  if (z >= ks) return;
  // warps per A^T row: spread few rows over all warps
  int wpr = 1;
  while (wpr < DQ && nr * wpr * 2 <= 8) wpr *= 2;
  for (int ti = 0; ti < P.nterm; ++ti) {
    const hq_gemm_term T = terms[P.term0 + ti];
    const int kd = hq_dim(rank, T.k, T.k_ri);
    const int kb = (int)(((long long)kd * z) / ks), ke = (int)(((long long)kd * (z + 1)) / ks);
    if (kb >= ke) continue;
    // B element (k, j) = T.b[k * sbk + j * sbj]; columns past n read column 0
    // (their sums are never stored)
    const size_t sbk = T.tb == 0 ? 1 : (size_t)T.ldb, sbj = T.tb == 0 ? (size_t)T.ldb : 1;
    size_t bj[NC];
#pragma unroll
    for (int j = 0; j < NC; ++j) bj[j] = (j < n ? j : 0) * sbj;
    const bool plain = T.mask_a == 0 && T.mask_b == 0;
    auto bval = [&](int k, int j) -> double {
      const int jj = j < n ? j : 0;
      return hq_mask(T.b[(size_t)k * sbk + bj[j]], T.tb == 0 ? k : jj, T.tb == 0 ? jj : k, T.mask_b);
    };
    if (KIND != 2 && (KIND == 1 || T.ta == 0)) {
      if (r < nr) {
        const int gi = i0 + r;
        const double* ap = T.a + gi;
        double tacc[NC];
#pragma unroll
        for (int j = 0; j < NC; ++j) tacc[j] = 0.0;
        if (plain) {
          // branch-free body: GV_U loads of A (and of B) issued before use
          int k = kb + sl;
          for (; k + (GV_U - 1) * NSL < ke; k += GV_U * NSL) {
            double a[GV_U], b[GV_U][NC];
#pragma unroll
            for (int u = 0; u < GV_U; ++u) {
              a[u] = __ldg(ap + (size_t)(k + u * NSL) * T.lda);
#pragma unroll
              for (int j = 0; j < NC; ++j) b[u][j] = __ldg(T.b + (size_t)(k + u * NSL) * sbk + bj[j]);
            }
#pragma unroll
            for (int u = 0; u < GV_U; ++u)
#pragma unroll
              for (int j = 0; j < NC; ++j) tacc[j] = fma(a[u], b[u][j], tacc[j]);
          }
          for (; k < ke; k += NSL) {
            const double a = __ldg(ap + (size_t)k * T.lda);
#pragma unroll
            for (int j = 0; j < NC; ++j) tacc[j] = fma(a, __ldg(T.b + (size_t)k * sbk + bj[j]), tacc[j]);
          }
        } else {
          for (int k = kb + sl; k < ke; k += NSL) {
            const double a = hq_mask(ap[(size_t)k * T.lda], gi, k, T.mask_a);
#pragma unroll
            for (int j = 0; j < NC; ++j) tacc[j] = fma(a, bval(k, j), tacc[j]);
          }
        }
#pragma unroll
        for (int j = 0; j < NC; ++j) acc[j] = fma(T.alpha, tacc[j], acc[j]);
      }
    } else if (KIND != 1) {
      // warp w owns rows rr = w / wpr + (8 / wpr) q of this block and the
      // k-lane-group w % wpr: all its rows advance together, so every k
      // step issues one load per row (independent) plus the B loads
      const int sub = wid % wpr, ngrp = (NT / 32) / wpr, r0 = wid / wpr;
      const int st = 32 * wpr;
      // rows past nr re-read row r0 (their sums are dropped)
      const double* ap0 = T.a + (size_t)(i0 + r0) * T.lda;
      const size_t rstep = (size_t)ngrp * T.lda;
      const int nq = r0 < nr ? (nr - 1 - r0) / ngrp + 1 : 0;   // valid rows of this warp
      // the rows go in chunks of GV_RQH (fewer live registers: more warps per SM)
      for (int qc = 0; qc < nq; qc += GV_RQH) {
        double d[GV_RQH][NC];
#pragma unroll
        for (int q = 0; q < GV_RQH; ++q)
#pragma unroll
          for (int j = 0; j < NC; ++j) d[q][j] = 0.0;
        bool rv[GV_RQH];
#pragma unroll
        for (int q = 0; q < GV_RQH; ++q) rv[q] = qc + q < nq;
        const double* apc = ap0 + (size_t)qc * rstep;
        if (plain) {
          // 16-byte loads along k, two 64-wide steps in flight (even leading
          // dims, 16-byte aligned bases, even slice start); the k-lane groups
          // of a row interleave whole steps; the rest of the slice goes by
          // the element loop below
          const bool vec = T.tb == 0 && ((T.lda | T.ldb) & 1) == 0 && (kb & 1) == 0 &&
                           (((uintptr_t)T.a | (uintptr_t)T.b) & 15) == 0;
          const int stv = 64 * wpr;
          const int kvend = vec ? kb + ((ke - kb) / stv) * stv : kb;
          if (vec) {
            auto step = [&](int kr, double2 (&a2)[GV_RQH], double2 (&b2)[NC]) {
#pragma unroll
              for (int j = 0; j < NC; ++j) b2[j] = __ldg(reinterpret_cast<const double2*>(T.b + bj[j] + kr) + lane);
#pragma unroll
              for (int q = 0; q < GV_RQH; ++q)
                a2[q] = __ldg(reinterpret_cast<const double2*>(apc + (rv[q] ? q * rstep : 0) + kr) + lane);
            };
            auto fmas = [&](const double2 (&a2)[GV_RQH], const double2 (&b2)[NC]) {
#pragma unroll
              for (int q = 0; q < GV_RQH; ++q)
#pragma unroll
                for (int j = 0; j < NC; ++j) d[q][j] = fma(a2[q].y, b2[j].y, fma(a2[q].x, b2[j].x, d[q][j]));
            };
            int kr = kb + sub * 64;
            for (; kr + stv < kvend; kr += 2 * stv) {
              double2 a0[GV_RQH], b0[NC], a1[GV_RQH], b1[NC];
              step(kr, a0, b0);
              step(kr + stv, a1, b1);
              fmas(a0, b0);
              fmas(a1, b1);
            }
            if (kr < kvend) {
              double2 a0[GV_RQH], b0[NC];
              step(kr, a0, b0);
              fmas(a0, b0);
            }
          }
          for (int k = kvend + sub * 32 + lane; k < ke; k += st) {
            double b[NC], a[GV_RQH];
#pragma unroll
            for (int j = 0; j < NC; ++j) b[j] = __ldg(T.b + (size_t)k * sbk + bj[j]);
#pragma unroll
            for (int q = 0; q < GV_RQH; ++q) a[q] = __ldg(apc + (rv[q] ? q * rstep : 0) + k);
#pragma unroll
            for (int q = 0; q < GV_RQH; ++q)
#pragma unroll
              for (int j = 0; j < NC; ++j) d[q][j] = fma(a[q], b[j], d[q][j]);
          }
        } else {
          for (int k = kb + sub * 32 + lane; k < ke; k += st) {
#pragma unroll
            for (int q = 0; q < GV_RQH; ++q) {
              if (!rv[q]) continue;
              const double a = hq_mask(apc[q * rstep + k], k, i0 + r0 + ngrp * (qc + q), T.mask_a);
#pragma unroll
              for (int j = 0; j < NC; ++j) d[q][j] = fma(a, bval(k, j), d[q][j]);
            }
          }
        }
#pragma unroll
        for (int q = 0; q < GV_RQH; ++q) {
          if (!rv[q]) continue;   // warp-uniform
#pragma unroll
          for (int j = 0; j < NC; ++j) {
            const double v = warp_sum(d[q][j]);
            if (lane == 0) dotr[sub][r0 + ngrp * (qc + q)][j] += T.alpha * v;
          }
        }
      }
    }
  }
#pragma unroll
  for (int j = 0; j < NC; ++j) part[sl][r][j] = acc[j];
  __syncthreads();
  // K-split slot of this (row block, slice): 64 x NC doubles
  double* slot0 = ks > 1 ? P.ws + (size_t)blockIdx.x * ks_cap * (GV_ROWS * NC) : nullptr;
  for (int e = t; e < nr * NC; e += NT) {
    const int rr = e / NC, j = e % NC;
    if (j >= n) continue;
    double v = 0.0;
#pragma unroll
    for (int q = 0; q < DQ; ++q) v += dotr[q][rr][j];
#pragma unroll
    for (int q = 0; q < NSL; ++q) v += part[q][rr][j];
    if (ks > 1) {
      slot0[(size_t)z * (GV_ROWS * NC) + e] = v;
      continue;
    }
    double* cp = P.c + (i0 + rr) + (size_t)j * P.ldc;
    *cp = (P.beta == 0.0) ? v : fma(P.beta, *cp, v);
  }
  if (ks > 1 && hq_split_last(P.cnt + blockIdx.x, ks)) {
    for (int e = t; e < nr * NC; e += NT) {
      const int rr = e / NC, j = e % NC;
      if (j >= n) continue;
      double v = 0.0;
      for (int zz = 0; zz < ks; ++zz) v += __ldcg(slot0 + (size_t)zz * (GV_ROWS * NC) + e);
      double* cp = P.c + (i0 + rr) + (size_t)j * P.ldc;
      *cp = (P.beta == 0.0) ? v : fma(P.beta, *cp, v);
    }
  }
}
// Mode 5: the power iteration's V^T X products of every tree level in ONE
// launch.  Problem i owns the work items [item0_i, item0_{i+1}) (its K
// slices, sized on the host from the static block sizes), so the grid has no
// empty CTAs; a CTA finds its problem by binary search, then covers all output
// rows of that problem for its K slice: warp w takes rows w, w+8, ... (RQ at a
// time, one independent 16-byte load per row per lane and k step), lanes
// along k, shuffle reduction.  A problem with one item writes C directly; the
// slices of a split problem write their own workspace slots and the last to
// arrive sums them in slice order (deterministic).
template <int NC>
__global__ void __launch_bounds__(NT, NC == 2 ? 3 : 2) gemv_flat_kernel(const hq_gemm_prob* __restrict__ probs,
                                                       const hq_gemm_term* __restrict__ terms,
                                                       const int* __restrict__ rank, int nprob, int nitems,
                                                       const int* __restrict__ skip) {
  if (skip && *skip) return;
  constexpr int RQ = 4;
  const int bid = blockIdx.x;
  // last problem with item0 <= bid: 32-ary search by every warp (3 dependent
  // loads for 32768 problems instead of 15 for the binary search -- the
  // descriptor fetches were most of a CTA's life on ~50 KB work items)
  int lo = 0, hi = nprob - 1;
  {
    const int ln = threadIdx.x & 31;
    while (lo < hi) {
      const int span = hi - lo;                 // candidates lo+1 .. hi
      const int step = (span + 31) / 32;        // probe lo + step * (ln + 1), clamped
      const int idx = min(lo + step * (ln + 1), hi);
      const bool le = probs[idx].item0 <= bid;
      const unsigned bal = __ballot_sync(0xffffffffu, le);
      const int cnt = __popc(bal);              // probes are monotone: the first cnt are <= bid
      const int nlo = cnt == 0 ? lo : min(lo + step * cnt, hi);
      const int nhi = cnt == 32 ? hi : min(lo + step * (cnt + 1), hi) - 1;
      lo = nlo;
      hi = max(nhi, nlo);
    }
  }
  const hq_gemm_prob P = probs[lo];
  const int ks = (lo + 1 < nprob ? probs[lo + 1].item0 : nitems) - P.item0;
  const int z = bid - P.item0;
  const int m = hq_dim(rank, P.m, P.m_ri), n = hq_dim(rank, P.n, P.n_ri);
  if (m <= 0 || n <= 0 || z < 0 || z >= ks) return;
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  // destination of this slice: C (one slice) or its slot (row-major NC)
  double* slot0 = P.ws;
  double* mine = ks > 1 ? P.ws + (size_t)z * P.m * NC : nullptr;
  // out(i, j) op= v: first term stores (C: with beta), later terms add; a
  // barrier separates the terms (row ownership differs between layouts)
  auto emit = [&](int i, int j, double v, bool first) {
    if (ks > 1) {
      double& d = mine[(size_t)i * NC + j];
      d = first ? v : d + v;
    } else {
      double* cp = P.c + i + (size_t)j * P.ldc;
      *cp = first ? (P.beta == 0.0 ? v : fma(P.beta, *cp, v)) : *cp + v;
    }
  };
  for (int ti = 0; ti < P.nterm; ++ti) {
    const bool first = ti == 0;
    if (ti > 0) __syncthreads();
    const hq_gemm_term T = terms[P.term0 + ti];
    const int kd = hq_dim(rank, T.k, T.k_ri);
    // slice bounds on multiples of 4 (16-byte aligned vector loads)
    int kb = (int)(((long long)kd * z) / ks) & ~3, ke = z + 1 == ks ? kd : (int)(((long long)kd * (z + 1)) / ks) & ~3;
    if (kb > ke) kb = ke;
    const size_t sbk = T.tb == 0 ? 1 : (size_t)T.ldb, sbj = T.tb == 0 ? (size_t)T.ldb : 1;
    if (T.ta == 0) {
      // rows across threads (coalesced columns of A)
      for (int i = t; i < m; i += NT) {
        double d[NC];
#pragma unroll
        for (int j = 0; j < NC; ++j) d[j] = 0.0;
        for (int k = kb; k < ke; ++k) {
          const double a = hq_mask(T.a[i + (size_t)k * T.lda], i, k, T.mask_a);
#pragma unroll
          for (int j = 0; j < NC; ++j) {
            const int jj = j < n ? j : 0;
            d[j] = fma(a, hq_mask(T.b[(size_t)k * sbk + jj * sbj], T.tb == 0 ? k : jj, T.tb == 0 ? jj : k,
                                  T.mask_b), d[j]);
          }
        }
#pragma unroll
        for (int j = 0; j < NC; ++j)
          if (j < n) emit(i, j, T.alpha * d[j], first);
      }
      continue;
    }
    const bool plain = T.mask_a == 0 && T.mask_b == 0;
    // 16-byte loads need even leading dims and 16-byte aligned bases
    const bool vec = plain && T.tb == 0 && ((T.lda | T.ldb) & 1) == 0 &&
                     (((uintptr_t)T.a | (uintptr_t)T.b) & 15) == 0;
    for (int r0 = wid; r0 < m; r0 += (NT / 32) * RQ) {
      double d[RQ][NC];
#pragma unroll
      for (int q = 0; q < RQ; ++q)
#pragma unroll
        for (int j = 0; j < NC; ++j) d[q][j] = 0.0;
      const double* ap0 = T.a + (size_t)r0 * T.lda;
      const size_t rstep = (size_t)(NT / 32) * T.lda;
      const int nq = min(RQ, (m - 1 - r0) / (NT / 32) + 1);
      int k = kb;
      if (vec) {
        // lane covers k = 2 lane + {0, 1} of every 64-wide step; two steps in
        // flight: 2 x (RQ + NC) independent 16-byte loads
        const double2* bcol[NC];
#pragma unroll
        for (int j = 0; j < NC; ++j) bcol[j] = reinterpret_cast<const double2*>(T.b + (size_t)(j < n ? j : 0) * T.ldb);
        // rank-16 inputs leave a warp 2 rows: four steps in flight instead
        // (the same 8 independent 16-byte loads of A per lane)
        if (nq <= 2) {
          for (; k + 256 <= ke; k += 256) {
            double2 b[4][NC], av[4][2];
#pragma unroll
            for (int h = 0; h < 4; ++h) {
              const int kk = (k + 64 * h) / 2 + lane;
#pragma unroll
              for (int j = 0; j < NC; ++j) b[h][j] = __ldg(bcol[j] + kk);
#pragma unroll
              for (int q = 0; q < 2; ++q)
                av[h][q] = __ldg(reinterpret_cast<const double2*>(ap0 + (q < nq ? q * rstep : 0)) + kk);
            }
#pragma unroll
            for (int h = 0; h < 4; ++h)
#pragma unroll
              for (int q = 0; q < 2; ++q)
#pragma unroll
                for (int j = 0; j < NC; ++j) d[q][j] = fma(av[h][q].y, b[h][j].y, fma(av[h][q].x, b[h][j].x, d[q][j]));
          }
        }
        for (; k + 128 <= ke; k += 128) {
          double2 b[2][NC], av[2][RQ];
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int kk = (k + 64 * h) / 2 + lane;
#pragma unroll
            for (int j = 0; j < NC; ++j) b[h][j] = __ldg(bcol[j] + kk);
#pragma unroll
            for (int q = 0; q < RQ; ++q)
              av[h][q] = __ldg(reinterpret_cast<const double2*>(ap0 + (q < nq ? q * rstep : 0)) + kk);
          }
#pragma unroll
          for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int q = 0; q < RQ; ++q)
#pragma unroll
              for (int j = 0; j < NC; ++j) d[q][j] = fma(av[h][q].y, b[h][j].y, fma(av[h][q].x, b[h][j].x, d[q][j]));
        }
      }
      // scalar remainder (and the masked / unaligned case)
      for (k += lane; k < ke; k += 32) {
        double b[NC];
#pragma unroll
        for (int j = 0; j < NC; ++j) {
          const int jj = j < n ? j : 0;
          const double v = __ldg(T.b + (size_t)k * sbk + jj * sbj);
          b[j] = plain ? v : hq_mask(v, T.tb == 0 ? k : jj, T.tb == 0 ? jj : k, T.mask_b);
        }
#pragma unroll
        for (int q = 0; q < RQ; ++q) {
          const double v = __ldg(ap0 + (q < nq ? q * rstep : 0) + k);
          const double a = plain ? v : hq_mask(v, k, r0 + (NT / 32) * q, T.mask_a);
#pragma unroll
          for (int j = 0; j < NC; ++j) d[q][j] = fma(a, b[j], d[q][j]);
        }
      }
#pragma unroll
      for (int q = 0; q < RQ; ++q) {
        if (q >= nq) break;   // warp-uniform
#pragma unroll
        for (int j = 0; j < NC; ++j) {
          const double v = warp_sum(d[q][j]);
          if (lane == 0 && j < n) emit(r0 + (NT / 32) * q, j, T.alpha * v, first);
        }
      }
    }
  }
  if (ks > 1 && hq_split_last(P.cnt, ks)) {
    for (int e = t; e < m * n; e += NT) {
      const int i = e % m, j = e / m;
      double v = 0.0;
      for (int zz = 0; zz < ks; ++zz) v += __ldcg(slot0 + (size_t)zz * P.m * NC + (size_t)i * NC + j);
      double* cp = P.c + i + (size_t)j * P.ldc;
      *cp = (P.beta == 0.0) ? v : fma(P.beta, *cp, v);
    }
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
  if (mode == 5) {
    // ksplit carries the total work-item count of the launch
    if (ncmax <= 2) gemv_flat_kernel<2><<<ksplit, NT, 0, st>>>(probs, terms, rank, nprob, ksplit, skip);
    else gemv_flat_kernel<4><<<ksplit, NT, 0, st>>>(probs, terms, rank, nprob, ksplit, skip);
    return hq_err(cudaGetLastError());
  }
  if (mode >= 2 && mode <= 4) {
    const int R = gv_rows(max_rows);
    dim3 grid((max_rows + R - 1) / R, nprob, ksplit);
    const int kind = mode - 2;
#define HQ_GEMV_LAUNCH(NC_, KIND_)                                                                          \
  do {                                                                                                      \
    if (R == 256) gemv_kernel<NC_, KIND_, 256><<<grid, NT, 0, st>>>(probs, terms, rank, ksplit, skip);      \
    else if (R == 128) gemv_kernel<NC_, KIND_, 128><<<grid, NT, 0, st>>>(probs, terms, rank, ksplit, skip); \
    else gemv_kernel<NC_, KIND_, 64><<<grid, NT, 0, st>>>(probs, terms, rank, ksplit, skip);                \
  } while (0)
    if (ncmax <= 2) {
      if (kind == 1) HQ_GEMV_LAUNCH(2, 1);
      else if (kind == 2) HQ_GEMV_LAUNCH(2, 2);
      else HQ_GEMV_LAUNCH(2, 0);
    } else {
      HQ_GEMV_LAUNCH(4, 0);
    }
#undef HQ_GEMV_LAUNCH
    return hq_err(cudaGetLastError());
  }
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

extern "C" int hq_gemm_tiled(void* stream, const hq_gemm_prob* probs, int nprob,
                             const hq_gemm_term* terms, int* rank, int tiles, int ksplit, int tile,
                             const int* skip) {
  if (nprob <= 0 || tiles <= 0) return 0;
  if (ksplit < 1) ksplit = 1;
  dim3 grid(tiles, nprob, ksplit);
  cudaStream_t st = (cudaStream_t)stream;
  if (tile == 32) {
    constexpr int S = 4, smem = S * 2 * (32 * (BK + 4) > BK * 36 ? 32 * (BK + 4) : BK * 36) * 8;
    static bool attr32 = false;
    if (!attr32) {
      cudaError_t e = cudaFuncSetAttribute(gemm_kernel<32, 32, 2, 2, S>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      if (e != cudaSuccess) return hq_err(e);
      attr32 = true;
    }
    gemm_kernel<32, 32, 2, 2, S><<<grid, 128, smem, st>>>(probs, terms, rank, ksplit, skip);
  } else {
    constexpr int S = 3, smem = S * 2 * (64 * (BK + 4) > BK * 68 ? 64 * (BK + 4) : BK * 68) * 8;
    static bool attr = false;
    if (!attr) {
      cudaError_t e = cudaFuncSetAttribute(gemm_kernel<64, 64, 2, 4, S>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      if (e != cudaSuccess) return hq_err(e);
      attr = true;
    }
    gemm_kernel<64, 64, 2, 4, S><<<grid, 256, smem, st>>>(probs, terms, rank, ksplit, skip);
  }
  return hq_err(cudaGetLastError());
}

extern "C" int hq_gemm(void* stream, const hq_gemm_prob* probs, int nprob,
                       const hq_gemm_term* terms, int* rank, int tiles, int ksplit,
                       const int* skip) {
  return hq_gemm_tiled(stream, probs, nprob, terms, rank, tiles, ksplit, 64, skip);
}
