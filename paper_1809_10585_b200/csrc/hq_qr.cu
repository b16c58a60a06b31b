// Householder QR with compact-WY panels, Q application, and the gathers that
// build the compressed columns / factor stacks.
//   QR      reference wy.py:17-72 (+ dense.py:45-68 sign convention)
//   applyQ  reference wy.py:91-95 / hqr.py:197-216 (Q^T M = M - Y T^T Y^T M)
//   leaf    reference hqr.py:110-119 (compressed column [A; B_R; C])
//   concat  reference hqr.py:145,154 / arith.py:107 (stacked low-rank factors)
// One CTA per problem; panels of NB columns are staged in shared memory when
// they fit, otherwise reduced in place in (L2-resident) global memory.
#include "hq_common.cuh"
#include <cstdlib>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

#ifdef HQ_DEBUG_TIMING
__device__ long long* hq_dbg = nullptr;
#define HQ_T0 long long hq_t_ = clock64();
#define HQ_TMARK(k) do { if (threadIdx.x == 0 && hq_dbg) { const long long c_ = clock64(); atomicAdd((unsigned long long*)(hq_dbg + 2048 + (k)), (unsigned long long)(c_ - hq_t_)); atomicAdd((unsigned long long*)(hq_dbg + 2064 + (k)), 1ull); hq_t_ = c_; } } while (0)
#else
#define HQ_T0
#define HQ_TMARK(k) do { } while (0)
#endif
#ifdef HQ_DEBUG_TIMING
extern "C" int hq_debug_set(void* p) {
  return (int)cudaMemcpyToSymbol(hq_dbg, &p, sizeof(p));
}
#endif
namespace {
constexpr int NT = 256, NW = NT / 32, NB = 16;
constexpr int STAGE_ROWS = 1024;  // panel staged in smem when rows <= STAGE_ROWS
constexpr int CW = 32;            // trailing-update column chunk
constexpr int YBUF = 528 * NB;    // staged Y / X chunk / merge scratch (doubles)
constexpr int XS_LD = 388;        // merge scratch leading dim (== 4 mod 16)
// W = Y^T X is kept transposed (wc[col + refl * WLD]) and T^op W as
// wc2[refl + col * W2LD]: both padded so the m8n8k4 fragment fetches and the
// per-thread triangular products are bank-conflict free
constexpr int WLD = CW + 4, W2LD = NB + 4;
constexpr int WC_OFF = 0, WC2_OFF = NB * WLD, WPART_OFF = WC2_OFF + CW * W2LD;
constexpr int WSP = WPART_OFF + (NW - 1) * NB * 8;   // k-split partial tiles (16 x 8 each)

// shared-memory leading dimension for staged columns: >= rows and == 4 (mod
// 16 doubles), so the 8-column x 4-row operand fetches of the m8n8k4 tiles
// hit 32 distinct banks (a multiple of 16 puts all 8 columns in one bank)
__host__ __device__ __forceinline__ int pad_ld(int rows) { return ((rows + 11) & ~15) + 4; }

struct QrSmem {
  double panel[(STAGE_ROWS + 4) * NB];  // staged panel being factored / staged X block
  double ybuf[YBUF];              // staged Y of the previous panel (cluster), X chunks
                                  // (single-CTA trailing update), X of the T merge
  double bcast[STAGE_ROWS];       // y_j broadcast of the register-cached panel factorization
  double tp[NB * NB];
  double dmat[NB * NB];   // dmat[c*NB + j] = y_c^T y_j (panel T recurrence)
  double dv[NB];
  double tcol[NB];
  double wsp[WSP];      // W = Y^T X (wc), T^op W (wc2), k-split partials; 2nd y_j broadcast buffer
  double red[32];
  double scal[4];
};

// column j's reflector, formed by the warp that caches column j in `c`
// (the diagonal entry x0 comes from its owning lane with one shuffle)
template <int E>
__device__ __forceinline__ void own_column(double (&c)[E], int j, int rows, int lane, unsigned ybuf,
                                           double* tau, QrSmem& S) {
  // four partial sums: the FP64 FMA chain of one accumulator would be the
  // longest dependency of the column step
  double sp[4] = {0.0, 0.0, 0.0, 0.0}, x0 = 0.0;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int i = lane + 32 * e;
    const double v = c[e];
    if (i > j && i < rows) sp[e & 3] = fma(v, v, sp[e & 3]);
    if (e == (j >> 5)) x0 = v;
  }
  double ss = (sp[0] + sp[1]) + (sp[2] + sp[3]);
  x0 = __shfl_sync(0xffffffffu, x0, j & 31);
  ss = warp_sum(ss);
  double sc = 1.0, isc = 1.0;
  const bool safe = refl_safe(x0, ss);
  if (!safe) {   // warp-uniform, rare: rescale by max|x|
    double amax = 0.0;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int i = lane + 32 * e;
      if (i >= j && i < rows) amax = fmax(amax, fabs(c[e]));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    sc = refl_scale(amax);
    isc = sc == 1.0 ? 1.0 : (sc > 1.0 ? 0x1p-600 : 0x1p600);
    ss = 0.0;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int i = lane + 32 * e;
      const double v = c[e] * sc;
      if (i > j && i < rows) ss = fma(v, v, ss);
    }
    ss = warp_sum(ss);
  }
  // common case (no rescaling): norm, 1 / u1 and gamma from the hardware
  // rsqrt / rcp refined by Newton steps instead of a software sqrt and two
  // divisions on the column step's critical path
  const Refl R = safe ? make_refl_fast(x0, ss) : make_refl(x0, ss, sc, isc);
  const double gamma = R.gamma, rho = R.rho, inv = R.inv;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int i = lane + 32 * e;
    if (i > j && i < rows) c[e] *= inv;
    if (i == j) c[e] = rho;
    hq_sts(ybuf + 8u * i, i > j ? c[e] : (i == j ? 1.0 : 0.0));
  }
  if (lane == 0) { S.dv[j] = gamma; tau[j] = gamma; }
}

// Register-cached variant: warp w holds columns w and w+NW of the panel in
// registers (lane l owns rows l, l+32, ...; E rows per lane), so a column
// step is register arithmetic plus one shared-memory broadcast of y_j.  The
// broadcast buffer alternates between two arrays, so one barrier per column
// suffices (the next owner writes the other buffer while y_j is still read).
template <int E>
__device__ __noinline__ void panel_factor_reg(double* P, int ldp, int rows, int pw, double* tau, QrSmem& S) {
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  HQ_T0
  double col[2][E];
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int c = wid + q * NW;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int i = lane + 32 * e;
      col[q][e] = (c < pw && i < rows) ? P[i + (size_t)c * ldp] : 0.0;
    }
  }
  const unsigned wsp_a = hq_smem_addr(S.wsp), bcast_a = hq_smem_addr(S.bcast), dv_a = hq_smem_addr(S.dv);
  for (int j = 0; j < pw; ++j) {
    // y_j broadcast (rows <= 32 E), as a shared-space address: LDS / STS
    const unsigned ybuf = (j & 1) ? wsp_a : bcast_a;
    if (wid == (j % NW)) {
      if (j < NW) own_column<E>(col[0], j, rows, lane, ybuf, tau, S);
      else own_column<E>(col[1], j, rows, lane, ybuf, tau, S);
    }
    __syncthreads();
    const double gamma = hq_lds(dv_a + 8u * j);
    // the tallest panels (E = 32) re-read y_j for the update instead of keeping it:
    // 2 E column values + E of y would exceed the register file and spill
    constexpr bool KEEPY = E <= 24;
    constexpr int EY = KEEPY ? E : 1;
    double y[EY];
    // both cached columns: dots first, then the two reductions interleaved
    double d[2];
    {
      double dp[2][4] = {{0.0, 0.0, 0.0, 0.0}, {0.0, 0.0, 0.0, 0.0}};
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const double ye = hq_lds(ybuf + 8u * (lane + 32 * e));
        if (KEEPY) y[e] = ye;
        dp[0][e & 3] = fma(ye, col[0][e], dp[0][e & 3]);
        dp[1][e & 3] = fma(ye, col[1][e], dp[1][e & 3]);
      }
      d[0] = (dp[0][0] + dp[0][1]) + (dp[0][2] + dp[0][3]);
      d[1] = (dp[1][0] + dp[1][1]) + (dp[1][2] + dp[1][3]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      d[0] += __shfl_xor_sync(0xffffffffu, d[0], o);
      d[1] += __shfl_xor_sync(0xffffffffu, d[1], o);
    }
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int c = wid + q * NW;
      if (c >= pw || c == j) continue;
      if (c > j) {
        const double gd = gamma * d[q];
#pragma unroll
        for (int e = 0; e < E; ++e)
          col[q][e] = fma(-gd, KEEPY ? y[e] : hq_lds(ybuf + 8u * (lane + 32 * e)), col[q][e]);
      } else if (lane == 0) {
        S.dmat[c * NB + j] = d[q];   // y_c^T y_j  (c < j)
      }
    }
  }
  __syncthreads();
  HQ_TMARK(8);
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int c = wid + q * NW;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int i = lane + 32 * e;
      if (c < pw && i < rows) P[i + (size_t)c * ldp] = col[q][e];
    }
  }
  // T (pw x pw): T[j][j] = gamma_j, T[0:j, j] = -gamma_j T[0:j,0:j] d[0:j, j]
  // (wy.py:37-39); lane i keeps row i of T in registers
  if (wid == 0) {
    double trow[NB];
#pragma unroll
    for (int j = 0; j < NB; ++j) {
      double v0 = 0.0, v1 = 0.0;
#pragma unroll
      for (int l = 0; l < j; ++l) {
        const double dl = S.dmat[l * NB + j];
        if (l & 1) v1 = fma(trow[l], dl, v1); else v0 = fma(trow[l], dl, v0);
      }
      const double gj = j < pw ? S.dv[j] : 0.0;
      trow[j] = j < pw ? (lane < j ? -gj * (v0 + v1) : (lane == j ? gj : 0.0)) : 0.0;
    }
    if (lane < NB) {
#pragma unroll
      for (int j = 0; j < NB; ++j) S.tp[lane + j * NB] = trow[j];
    }
  }
  __syncthreads();
  HQ_TMARK(9);
}

// Block-wide variant for tall panels left in global memory: every warp
// streams a slice of the rows (the warp-owned variant would serialize a tall
// column on one warp).
__device__ void panel_factor_block(double* P, int ldp, int rows, int pw, double* tau, QrSmem& S) {
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  for (int j = 0; j < pw; ++j) {
    double ss = 0.0;
    for (int i = j + 1 + t; i < rows; i += NT) { const double v = P[i + (size_t)j * ldp]; ss = fma(v, v, ss); }
    ss = block_sum(ss, S.red);
    const double x0 = P[j + (size_t)j * ldp];
    double sc = 1.0, isc = 1.0;
    if (!refl_safe(x0, ss)) {   // block-uniform, rare: rescale by max|x|
      double amax = 0.0;
      for (int i = j + t; i < rows; i += NT) amax = fmax(amax, fabs(P[i + (size_t)j * ldp]));
      amax = block_max_nonneg(amax, S.red);
      sc = refl_scale(amax);
      isc = sc == 1.0 ? 1.0 : (sc > 1.0 ? 0x1p-600 : 0x1p600);
      ss = 0.0;
      for (int i = j + 1 + t; i < rows; i += NT) { const double v = P[i + (size_t)j * ldp] * sc; ss = fma(v, v, ss); }
      ss = block_sum(ss, S.red);
    }
    if (t == 0) {
      const Refl R = make_refl(x0, ss, sc, isc);
      P[j + (size_t)j * ldp] = R.rho;
      S.scal[0] = R.gamma; S.scal[1] = R.inv;
      tau[j] = R.gamma;
    }
    __syncthreads();
    const double gamma = S.scal[0], inv = S.scal[1];
    for (int i = j + 1 + t; i < rows; i += NT) P[i + (size_t)j * ldp] *= inv;
    __syncthreads();
    // d_c = y_j^T P[:, c] for every panel column c != j (rows >= j).  For c < j
    // these are Y_c^T y_j (T recurrence), for c > j the reflector application.
    double acc[NB];
#pragma unroll
    for (int c = 0; c < NB; ++c) acc[c] = 0.0;
    for (int i = j + t; i < rows; i += NT) {
      const double yi = (i == j) ? 1.0 : P[i + (size_t)j * ldp];
#pragma unroll
      for (int c = 0; c < NB; ++c)
        if (c < pw && c != j) acc[c] = fma(yi, P[i + (size_t)c * ldp], acc[c]);
    }
#pragma unroll
    for (int c = 0; c < NB; ++c) {
      const double v = warp_sum(acc[c]);
      if (lane == 0) S.dmat[wid * NB + c] = v;
    }
    __syncthreads();
    if (t < NB) {
      double v = 0.0;
      for (int w = 0; w < NW; ++w) v += S.dmat[w * NB + t];
      S.dv[t] = v;
    }
    __syncthreads();
    // T[0:j, j] = -gamma * T[0:j, 0:j] d[0:j];  T[j, j] = gamma   (wy.py:37-39)
    if (t < j) {
      double v = 0.0;
      for (int a = t; a < j; ++a) v = fma(S.tp[t + a * NB], S.dv[a], v);
      S.tcol[t] = -gamma * v;
    }
    __syncthreads();
    if (t < j) S.tp[t + j * NB] = S.tcol[t];
    if (t == j) S.tp[j + j * NB] = gamma;
    for (int i = j + t; i < rows; i += NT) {
      const double yi = (i == j) ? 1.0 : P[i + (size_t)j * ldp];
      for (int c = j + 1; c < pw; ++c) P[i + (size_t)c * ldp] -= gamma * S.dv[c] * yi;
    }
    __syncthreads();
  }
}

// y_a(i) of panel reflector a (unit diagonal, zero above): the load is
// unconditional (rows above the diagonal hold R, harmless) so a warp does
// not diverge around it
__device__ __forceinline__ double yval(const double* P, int ldp, int i, int a) {
  const double v = P[i + (size_t)a * ldp];
  return i > a ? v : (i == a ? 1.0 : 0.0);
}
// the same from a shared-space address (LDS instead of a generic load)
__device__ __forceinline__ double yval_s(unsigned pa, int ldp, int i, int a) {
  const double v = hq_lds(pa + 8u * (unsigned)(i + a * ldp));
  return i > a ? v : (i == a ? 1.0 : 0.0);
}

// stage cols columns of rows rows (global, ld lds) into shared dst (ld ldd)
// with asynchronous copies; ends with a barrier
__device__ __forceinline__ void stage_cols(double* dst, int ldd, const double* src, int lds, int rows, int cols) {
  // 16-byte copies when every column start is 16-byte aligned on both sides
  // (ldd is a multiple of 4 by construction): half the copy instructions
  const bool vec = ((((uintptr_t)src | (uintptr_t)dst) & 15) == 0) && ((lds | ldd) & 1) == 0;
  if (vec) {
    // warp w copies columns w, w + NW, ...; lanes along the rows (no divisions)
    const int pairs = rows >> 1, lane = threadIdx.x & 31;
    for (int c = threadIdx.x >> 5; c < cols; c += NW) {
      const double* sc = src + (size_t)c * lds;
      double* dc = dst + (size_t)c * ldd;
      for (int pi = lane; pi < pairs; pi += 32) cp_async16(dc + 2 * pi, sc + 2 * pi);
    }
    if (rows & 1)
      for (int c = threadIdx.x; c < cols; c += NT)
        cp_async8(dst + rows - 1 + (size_t)c * ldd, src + rows - 1 + (size_t)c * lds);
  } else {
    for (int c = 0; c < cols; ++c)
      for (int i = threadIdx.x; i < rows; i += NT) cp_async8(dst + i + (size_t)c * ldd, src + i + (size_t)c * lds);
  }
  cp_async_wait_all();
  __syncthreads();
}

// stage_cols with the columns moved by the TMA engine: one cp.async.bulk per
// column (the even part of the rows; an odd last row by a plain copy),
// completion on the mbarrier `bar` whose phase parity the caller carries in
// `parity`.  Falls back to stage_cols when a column start is not 16-byte
// aligned.  Block-uniform; ends with a barrier.
__device__ __forceinline__ void stage_cols_bulk(double* dst, int ldd, const double* src, int lds, int rows, int cols,
                                                unsigned long long* bar, unsigned& parity) {
  const int re = rows & ~1;
  const bool ok = ((((uintptr_t)src | (uintptr_t)dst) & 15) == 0) && ((lds | ldd) & 1) == 0 && re > 0 && cols > 0;
  if (!ok) { stage_cols(dst, ldd, src, lds, rows, cols); return; }
  const int t = threadIdx.x;
  if (t < 32) {
    if (t == 0) mbar_expect_tx(bar, (unsigned)cols * (unsigned)re * 8u);
    __syncwarp();
    for (int c = t; c < cols; c += 32) bulk_g2s(dst + (size_t)c * ldd, src + (size_t)c * lds, (unsigned)re * 8u, bar);
  } else if (rows & 1) {
    for (int c = t - 32; c < cols; c += NT - 32) dst[re + (size_t)c * ldd] = src[re + (size_t)c * lds];
  }
  mbar_wait(bar, parity);
  parity ^= 1u;
  __syncthreads();
}

// shared -> global write-back of cols columns by bulk copies (same alignment
// rule; plain stores otherwise).  The caller's last writes to src must be
// separated from this call by a barrier only (the proxy fence is here).
__device__ __forceinline__ void store_cols_bulk(double* dst, int ldd, const double* src, int lds, int rows, int cols) {
  const int re = rows & ~1;
  const bool ok = ((((uintptr_t)src | (uintptr_t)dst) & 15) == 0) && ((lds | ldd) & 1) == 0 && re > 0;
  const int t = threadIdx.x;
  if (!ok) {
    for (int j = 0; j < cols; ++j)
      for (int i = t; i < rows; i += NT) dst[i + (size_t)j * ldd] = src[i + (size_t)j * lds];
    return;
  }
  fence_proxy_async_smem();
  __syncthreads();
  if (t < 32) {
    for (int c = t; c < cols; c += 32) bulk_s2g(dst + (size_t)c * ldd, src + (size_t)c * lds, (unsigned)re * 8u);
    bulk_commit();
    bulk_wait_all();
  } else if (rows & 1) {
    for (int c = t - 32; c < cols; c += NT - 32) dst[re + (size_t)c * ldd] = src[re + (size_t)c * lds];
  }
}

// X (rows x ncols) := (I - Y T^op Y^T) X for panel reflectors Y (rows x pw,
// unit diagonal at local row a; smem or global) with T factor tp (NB x NB).
// trans_t: T^T (applies Q^T) else T (applies Q).  Both products run on the
// FP64 tensor pipe (mma.sync m8n8k4): W = Y^T X (16 x cw), W2 = T^op W,
// X -= Y W2, column chunks of cw.  When X is in global memory and a staging
// buffer xs (xs_cap doubles) is given, each chunk is first staged into shared
// memory with asynchronous copies (one round trip to L2 instead of one per
// k-block); the result goes back to X.
// YSH: Y lives in shared memory, XSH: the chunk of X is read from shared
// memory (staged, or X itself) -- then both are fetched with LDS.
template <bool YSH, bool XSH, class SM>
__device__ __noinline__ void apply_panel_cols_impl(const double* Y, int ldy, int rows, int pw, const double* tp,
                                                   double* X, int ldx, int ncols, bool trans_t, SM& S,
                                                   double* xs, int xs_cap) {
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  const unsigned ya = YSH ? hq_smem_addr(Y) : 0u;
  auto yv = [&](int i, int a) { return YSH ? yval_s(ya, ldy, i, a) : yval(Y, ldy, i, a); };
  const int gq = lane >> 2, tq = lane & 3;
  int cwmax = CW;
  const int ldxs = pad_ld(rows);
  if (xs) {
    cwmax = min(CW, (xs_cap / ldxs) & ~7);
    if (cwmax < 8) { xs = nullptr; cwmax = CW; }
  }
  HQ_T0
  for (int c0 = 0; c0 < ncols; c0 += cwmax) {
    const int cw = min(cwmax, ncols - c0);
    const double* Xr = X + (size_t)c0 * ldx;
    int ldr = ldx;
    if (xs) {
      stage_cols(xs, ldxs, Xr, ldx, rows, cw);
      Xr = xs;
      ldr = ldxs;
    }
    // ---- W = Y^T X_chunk (16 x cw): item (nt, kp) = both 8-reflector halves
    // against column tile nt over row range kp (the rows are split so that
    // every warp has an item); two accumulator sets halve the mma chain
    const int ntn = (cw + 7) / 8;
    const int kparts = max(1, NW / ntn);
    const int kchunk = ((rows + kparts - 1) / kparts + 31) & ~31;
    double* wc = S.wsp + WC_OFF;
    double* wc2 = S.wsp + WC2_OFF;
    double* wpart = S.wsp + WPART_OFF;
    for (int item = wid; item < ntn * kparts; item += NW) {
      const int nt = item % ntn, kp = item / ntn;
      double d00 = 0.0, d01 = 0.0, d10 = 0.0, d11 = 0.0;
      double e00 = 0.0, e01 = 0.0, e10 = 0.0, e11 = 0.0;
      const int j = nt * 8 + gq;          // B col  (chunk column)
      const double* xc = Xr + (size_t)(j < cw ? j : 0) * ldr;
      const unsigned xca = XSH ? hq_smem_addr(xc) : 0u;
      const int kb = kp * kchunk, ke = min(rows, kb + kchunk);
      for (int k0 = kb; k0 < ke; k0 += 32) {
        double a0[8], a1[8], bv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int ia = k0 + 4 * u + tq;
          const bool in = ia < ke;
          a0[u] = (in && gq < pw) ? yv(ia, gq) : 0.0;
          a1[u] = (in && 8 + gq < pw) ? yv(ia, 8 + gq) : 0.0;
          bv[u] = (in && j < cw) ? (XSH ? hq_lds(xca + 8u * ia) : xc[ia]) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; u += 2) {
          dmma884(d00, d01, a0[u], bv[u]);
          dmma884(d10, d11, a1[u], bv[u]);
          dmma884(e00, e01, a0[u + 1], bv[u + 1]);
          dmma884(e10, e11, a1[u + 1], bv[u + 1]);
        }
      }
      const int cl = 2 * tq;   // column within the tile
      if (kp == 0) {
        const int cc = nt * 8 + cl;
        wc[cc + gq * WLD] = d00 + e00;
        wc[cc + 1 + gq * WLD] = d01 + e01;
        wc[cc + (8 + gq) * WLD] = d10 + e10;
        wc[cc + 1 + (8 + gq) * WLD] = d11 + e11;
      } else {
        double* wp = wpart + ((kp - 1) * ntn + nt) * NB * 8;
        wp[cl + gq * 8] = d00 + e00;
        wp[cl + 1 + gq * 8] = d01 + e01;
        wp[cl + (8 + gq) * 8] = d10 + e10;
        wp[cl + 1 + (8 + gq) * 8] = d11 + e11;
      }
    }
    __syncthreads();
    HQ_TMARK(0);
    if (kparts > 1) {
      for (int e = t; e < NB * cw; e += NT) {
        const int a = e / cw, cc = e % cw, nt = cc >> 3;
        double v = wc[cc + a * WLD];
        for (int kp = 1; kp < kparts; ++kp) v += wpart[((kp - 1) * ntn + nt) * NB * 8 + (cc & 7) + a * 8];
        wc[cc + a * WLD] = v;
      }
      __syncthreads();
    }
    // W2 = T^op W: thread (a, cc); lanes run along cc (T entries broadcast)
    for (int e = t; e < NB * cw; e += NT) {
      const int a = e / cw, cc = e % cw;
      double v = 0.0;
      if (a < pw) {
        if (trans_t) { for (int b = 0; b <= a; ++b) v = fma(tp[b + a * NB], wc[cc + b * WLD], v); }
        else { for (int b = a; b < pw; ++b) v = fma(tp[a + b * NB], wc[cc + b * WLD], v); }
      }
      wc2[a + cc * W2LD] = v;
    }
    __syncthreads();
    HQ_TMARK(1);
    // ---- X_chunk -= Y W2 : warp w takes row tiles mt = w, w + NW, ...; the
    // W2 fragments of all column tiles stay in registers, the Y fragment of a
    // row tile is loaded once for all its column tiles
    double* Xw = X + (size_t)c0 * ldx;
    const int ntm = (rows + 7) / 8;
    double bw[CW / 8][4];
#pragma unroll
    for (int nt = 0; nt < CW / 8; ++nt)
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int jb = nt * 8 + gq;
        bw[nt][q] = (nt < ntn && jb < cw) ? wc2[4 * q + tq + jb * W2LD] : 0.0;
      }
#pragma unroll 2
    for (int mt = wid; mt < ntm; mt += NW) {
      const int i = mt * 8 + gq;
      double av[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int a = 4 * q + tq;
        av[q] = (i < rows && a < pw) ? -yv(i, a) : 0.0;
      }
#pragma unroll
      for (int nt = 0; nt < CW / 8; ++nt) {
        if (nt >= ntn) break;
        const int j = nt * 8 + 2 * tq;
        const double* x0 = Xr + (size_t)j * ldr;
        double d0, d1;
        if (XSH) {
          const unsigned x0a = hq_smem_addr(x0);
          d0 = (i < rows && j < cw) ? hq_lds(x0a + 8u * i) : 0.0;
          d1 = (i < rows && j + 1 < cw) ? hq_lds(x0a + 8u * (ldr + i)) : 0.0;
        } else {
          d0 = (i < rows && j < cw) ? x0[i] : 0.0;
          d1 = (i < rows && j + 1 < cw) ? x0[ldr + i] : 0.0;
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) dmma884(d0, d1, av[q], bw[nt][q]);
        double* xo = Xw + (size_t)j * ldx;
        if (i < rows && j < cw) xo[i] = d0;
        if (i < rows && j + 1 < cw) xo[ldx + i] = d1;
      }
    }
    __syncthreads();
    HQ_TMARK(2);
  }
}

template <class SM>
__device__ __forceinline__ void apply_panel_cols(const double* Y, int ldy, int rows, int pw, const double* tp,
                                                 double* X, int ldx, int ncols, bool trans_t, SM& S,
                                                 double* xs = nullptr, int xs_cap = 0) {
  if (xs && (min(CW, (xs_cap / pad_ld(rows)) & ~7) < 8)) xs = nullptr;   // the impl's own test
  const bool ysh = __isShared(Y) != 0, xsh = xs != nullptr || __isShared(X) != 0;   // block-uniform
  if (ysh) {
    if (xsh) apply_panel_cols_impl<true, true>(Y, ldy, rows, pw, tp, X, ldx, ncols, trans_t, S, xs, xs_cap);
    else apply_panel_cols_impl<true, false>(Y, ldy, rows, pw, tp, X, ldx, ncols, trans_t, S, xs, xs_cap);
  } else {
    if (xsh) apply_panel_cols_impl<false, true>(Y, ldy, rows, pw, tp, X, ldx, ncols, trans_t, S, xs, xs_cap);
    else apply_panel_cols_impl<false, false>(Y, ldy, rows, pw, tp, X, ldx, ncols, trans_t, S, xs, xs_cap);
  }
}

// Merge panel p0 (reflectors P, ld ldp; T factor tp) into the full
// compact-WY T: T[0:p0, p] = -T[0:p0,0:p0] (Y[:,0:p0]^T Y_p) T_p (wy.py:53).
// Needs the T blocks of all earlier panels.
__device__ __noinline__ void merge_T(const hq_qr_prob& Q, const double* W, int ld, int m, int r, int p0,
                        const double* P, int ldp, const double* tpv, QrSmem& S) {
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  const int pw = min(NB, r - p0), rows = m - p0;
  const double* tp_ = tpv;
  {
    if (Q.tfull) {
      double* TF = Q.tfull;
      const int ldt = Q.ldt;
      const int gq = lane >> 2, tq = lane & 3;
      for (int e = t; e < pw * pw; e += NT) TF[(p0 + e % pw) + (size_t)(p0 + e / pw) * ldt] = tp_[e % pw + (e / pw) * NB];
      if (p0 > 0) {
        // X (p0 x NB) = Y[:,0:p0]^T Y_p over local rows 0..rows-1 (DMMA)
        const int ntm = (p0 + 7) / 8;
        for (int tile = wid; tile < ntm * 2; tile += NW) {
          const int mt = tile >> 1, nt = tile & 1;
          const int b = mt * 8 + gq, a = nt * 8 + gq;
          double d0 = 0.0, d1 = 0.0;
          dmma_kloop(d0, d1, 0, rows, [&](int k0, double (&av)[8], double (&bv)[8]) {
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              const int i = k0 + 4 * u + tq;
              av[u] = (i < rows && b < p0) ? W[(p0 + i) + (size_t)b * ld] : 0.0;
              bv[u] = (i < rows && a < pw) ? yval(P, ldp, i, a) : 0.0;
            }
          });
          const int r = mt * 8 + gq, c = nt * 8 + 2 * tq;
          if (r < p0) { S.ybuf[r + c * XS_LD] = d0; S.ybuf[r + (c + 1) * XS_LD] = d1; }
        }
        __syncthreads();
        // X := X T_p (in place per row)
        for (int b = t; b < p0; b += NT) {
          double xr[NB];
#pragma unroll
          for (int a = 0; a < NB; ++a) xr[a] = a < pw ? S.ybuf[b + a * XS_LD] : 0.0;
#pragma unroll
          for (int a = 0; a < NB; ++a) {
            double v = 0.0;
#pragma unroll
            for (int c = 0; c < NB; ++c)
              if (c <= a) v = fma(xr[c], tp_[c + a * NB], v);
            if (a < pw) S.ybuf[b + a * XS_LD] = v;
          }
        }
        __syncthreads();
        // T[0:p0, p0:p0+pw] = -T11 X   (T11 upper, p0 x p0, read from TF; DMMA)
        for (int tile = wid; tile < ntm * 2; tile += NW) {
          const int mt = tile >> 1, nt = tile & 1;
          const int r = mt * 8 + gq, a = nt * 8 + gq;
          double d0 = 0.0, d1 = 0.0;
          dmma_kloop(d0, d1, mt * 8, p0, [&](int k0, double (&av)[8], double (&bv)[8]) {
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              const int c = k0 + 4 * u + tq;
              av[u] = (r < p0 && c < p0 && c >= r) ? -TF[r + (size_t)c * ldt] : 0.0;
              bv[u] = (c < p0 && a < pw) ? S.ybuf[c + a * XS_LD] : 0.0;
            }
          });
          const int ro = mt * 8 + gq, co = nt * 8 + 2 * tq;
          if (ro < p0 && co < pw) TF[ro + (size_t)(p0 + co) * ldt] = d0;
          if (ro < p0 && co + 1 < pw) TF[ro + (size_t)(p0 + co + 1) * ldt] = d1;
        }
      }
      __syncthreads();
    }
  }
}

// Cluster mode splits the full-T merge of panel p over the CTAs that are not
// factoring, pipelined one phase apart so it never extends a phase:
//   phase p+1: X_p = Y[:,0:p0]^T Y_p (p0 x pw, DMMA tiles split over the
//              parts) into a global scratch (double-buffered by panel parity);
//              part 0 also stores T_p's diagonal block into tfull;
//   phase p+2: T[0:p0, p0:p0+pw] = -T11 (X_p T_p) (tiles split over the
//              parts; T11 complete since panel p-1's merge ran in phase p+1).
// Visibility between phases comes from the cluster barrier ending a phase.
__device__ __noinline__ void merge_X_split(const hq_qr_prob& Q, const double* W, int ld, int m, int r, int p0,
                                           double* X, int part, int nparts, QrSmem& S) {
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  const int pw = min(NB, r - p0), rows = m - p0;
  const int gq = lane >> 2, tq = lane & 3;
  if (part == 0) {
    const double* tp_ = Q.tpanel + (size_t)(p0 / NB) * NB * NB;
    for (int e = t; e < pw * pw; e += NT)
      Q.tfull[(p0 + e % pw) + (size_t)(p0 + e / pw) * Q.ldt] = tp_[e % pw + (e / pw) * NB];
  }
  if (p0 == 0) return;
  const double* P = W + p0 + (size_t)p0 * ld;
  const int ntm = (p0 + 7) / 8;
  for (int tile = part * NW + wid; tile < ntm * 2; tile += nparts * NW) {
    const int mt = tile >> 1, nt = tile & 1;
    const int b = mt * 8 + gq, a = nt * 8 + gq;
    double d0 = 0.0, d1 = 0.0;
    dmma_kloop(d0, d1, 0, rows, [&](int k0, double (&av)[8], double (&bv)[8]) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int i = k0 + 4 * u + tq;
        av[u] = (i < rows && b < p0) ? W[(p0 + i) + (size_t)b * ld] : 0.0;
        bv[u] = (i < rows && a < pw) ? yval(P, ld, i, a) : 0.0;
      }
    });
    const int ro = mt * 8 + gq, c = nt * 8 + 2 * tq;
    if (ro < p0) { X[ro + (size_t)c * r] = d0; X[ro + (size_t)(c + 1) * r] = d1; }
  }
}

__device__ __noinline__ void merge_T12_split(const hq_qr_prob& Q, int r, int p0, const double* X, int part,
                                             int nparts, QrSmem& S) {
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  const int pw = min(NB, r - p0);
  if (p0 == 0) return;
  const int gq = lane >> 2, tq = lane & 3;
  const double* tp_ = Q.tpanel + (size_t)(p0 / NB) * NB * NB;
  double* TF = Q.tfull;
  const int ldt = Q.ldt;
  // X' = X T_p for every row (cheap, redundant per part) into shared memory
  for (int b = t; b < p0; b += NT) {
    double xr[NB];
#pragma unroll
    for (int a = 0; a < NB; ++a) xr[a] = a < pw ? X[b + (size_t)a * r] : 0.0;
#pragma unroll
    for (int a = 0; a < NB; ++a) {
      double v = 0.0;
#pragma unroll
      for (int c = 0; c < NB; ++c)
        if (c <= a) v = fma(xr[c], tp_[c + a * NB], v);
      S.ybuf[b + a * XS_LD] = a < pw ? v : 0.0;
    }
  }
  __syncthreads();
  const int ntm = (p0 + 7) / 8;
  for (int tile = part * NW + wid; tile < ntm * 2; tile += nparts * NW) {
    const int mt = tile >> 1, nt = tile & 1;
    const int rr = mt * 8 + gq, a = nt * 8 + gq;
    double d0 = 0.0, d1 = 0.0;
    dmma_kloop(d0, d1, mt * 8, p0, [&](int k0, double (&av)[8], double (&bv)[8]) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int c = k0 + 4 * u + tq;
        av[u] = (rr < p0 && c < p0 && c >= rr) ? -TF[rr + (size_t)c * ldt] : 0.0;
        bv[u] = (c < p0 && a < pw) ? S.ybuf[c + a * XS_LD] : 0.0;
      }
    });
    const int ro = mt * 8 + gq, co = nt * 8 + 2 * tq;
    if (ro < p0 && co < pw) TF[ro + (size_t)(p0 + co) * ldt] = d0;
    if (ro < p0 && co + 1 < pw) TF[ro + (size_t)(p0 + co + 1) * ldt] = d1;
  }
}

// Reduce panel p0 held at P (rows x pw, ld ldp; shared or global) into R +
// unit lower reflectors; publish gamma (tau) and T_p (S.tp, Q.tpanel).
__device__ void factor_panel_core(const hq_qr_prob& Q, double* P, int ldp, int rows, int pw, int p0,
                                  QrSmem& S) {
  const int t = threadIdx.x;
  if (t < NB * NB) S.tp[t] = 0.0;
  __syncthreads();
  HQ_T0
  // rows per lane E sized to the panel (lanes past the end only cost issue slots)
  if (rows <= 128) panel_factor_reg<4>(P, ldp, rows, pw, Q.tau + p0, S);
  else if (rows <= 192) panel_factor_reg<6>(P, ldp, rows, pw, Q.tau + p0, S);
  else if (rows <= 256) panel_factor_reg<8>(P, ldp, rows, pw, Q.tau + p0, S);
  else if (rows <= 384) panel_factor_reg<12>(P, ldp, rows, pw, Q.tau + p0, S);
  else if (rows <= 512) panel_factor_reg<16>(P, ldp, rows, pw, Q.tau + p0, S);
  else if (rows <= 768) panel_factor_reg<24>(P, ldp, rows, pw, Q.tau + p0, S);
  else if (rows <= 1024) panel_factor_reg<32>(P, ldp, rows, pw, Q.tau + p0, S);
  else panel_factor_block(P, ldp, rows, pw, Q.tau + p0, S);
  HQ_TMARK(5);
  if (Q.tpanel && t < NB * NB) Q.tpanel[(size_t)(p0 / NB) * NB * NB + t] = S.tp[t];
}

// Factor panel p0 of problem Q: stage it (when it fits), reduce it, publish
// gamma / T_p, (single-CTA path: update the trailing columns while the
// panel is staged, staging chunks of them through S.ybuf), merge T_p into the
// full compact-WY T when requested, write the panel back.
__device__ void factor_panel_step(const hq_qr_prob& Q, double* W, int ld, int m, int k, int r, int p0,
                                  bool do_trailing, bool do_merge, QrSmem& S) {
  const int t = threadIdx.x;
  const int pw = min(NB, r - p0), rows = m - p0;
  double* Pg = W + p0 + (size_t)p0 * ld;
  const bool staged = rows <= STAGE_ROWS;
  double* P = Pg;
  int ldp = ld;
  if (staged) {
    ldp = pad_ld(rows);
    stage_cols(S.panel, ldp, Pg, ld, rows, pw);
    P = S.panel;
  }
  factor_panel_core(Q, P, ldp, rows, pw, p0, S);
  // trailing columns: A_trail := Q_p^T A_trail
  // (X chunks are staged in S.ybuf; a staged panel shorter than STAGE_ROWS
  // leaves the tail of S.panel free, which is contiguous with S.ybuf: wider
  // chunks, fewer passes over Y)
  if (do_trailing && p0 + pw < k) {
    double* xs = staged ? S.panel + (size_t)ldp * NB : S.ybuf;
    const int xs_cap = staged ? (STAGE_ROWS + 4) * NB - ldp * NB + YBUF : YBUF;
    apply_panel_cols(P, ldp, rows, pw, S.tp, W + p0 + (size_t)(p0 + pw) * ld, ld, k - p0 - pw, true, S,
                     xs, xs_cap);
  }
  __syncthreads();
  if (do_merge) merge_T(Q, W, ld, m, r, p0, P, ldp, S.tp, S);
  if (staged)
    for (int c = 0; c < pw; ++c)
      for (int i = t; i < rows; i += NT) Pg[i + (size_t)c * ld] = P[i + c * ldp];
  __syncthreads();
}

__global__ void __launch_bounds__(NT) qr_kernel(const hq_qr_prob* __restrict__ probs,
                                                int* __restrict__ rank) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  QrSmem& S = *reinterpret_cast<QrSmem*>(smem_raw);
  const hq_qr_prob Q = probs[blockIdx.x];
  const int m = hq_dim(rank, Q.m, Q.m_ri), k = hq_dim(rank, Q.k, Q.k_ri);
  const int r = m < k ? m : k;
  for (int p0 = 0; p0 < r; p0 += NB) factor_panel_step(Q, Q.w, Q.ldw, m, k, r, p0, true, true, S);
}

// Householder QR of one problem on a G-CTA cluster.  Column blocks of NB are
// owned round-robin (block b by CTA b % G).  Phase ph: every CTA applies
// panel ph-1 to its blocks >= ph -- the owner of block ph first, so that it
// can factor panel ph immediately while the others are still updating -- and
// one cluster barrier (release/acquire at cluster scope, covering the panel
// and T_p written to global memory) separates the phases.
template <int G>
__global__ void __launch_bounds__(NT, 1) qr_cluster_kernel(const hq_qr_prob* __restrict__ probs,
                                                           int* __restrict__ rank) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  QrSmem& S = *reinterpret_cast<QrSmem*>(smem_raw);
  cg::cluster_group cluster = cg::this_cluster();
  const int cr = (int)cluster.block_rank();
  const hq_qr_prob Q = probs[blockIdx.x / G];
  const int m = hq_dim(rank, Q.m, Q.m_ri), k = hq_dim(rank, Q.k, Q.k_ri);
  const int r = m < k ? m : k;
  const int t = threadIdx.x;
  const int np = (r + NB - 1) / NB, nbk = (k + NB - 1) / NB;
  double* W = Q.w;
  const int ld = Q.ldw;
#ifdef HQ_DEBUG_TIMING
  long long tph = clock64();
#endif
  // with a full T, one extra phase finishes the pipelined merge of the last panel
  const int nph = np + (Q.tfull && np > 0 ? 1 : 0);
  double* Xs = Q.tpanel + (size_t)np * NB * NB;   // merge scratch: 2 x (r x NB)
  for (int ph = 0; ph <= nph; ++ph) {
#ifdef HQ_DEBUG_TIMING
    long long tA = clock64(), tB = tA, tC = tA;
#endif
    if (ph >= 1 && ph <= np) {
      const int q0 = (ph - 1) * NB, qw = min(NB, r - q0), rows = m - q0;
      if (t < NB * NB) S.tp[t] = Q.tpanel[(size_t)(ph - 1) * NB * NB + t];
      const double* Yg = W + q0 + (size_t)q0 * ld;
      // block assignment of this phase: CTA ph % G updates and factors block
      // ph alone (its chain bounds the phase); the later blocks go round-robin
      // to the other CTAs (all CTAs once there is nothing left to factor)
      const int fct = ph % G;
      const bool factoring = ph < np;
      int b0, bstep;
      if (!factoring) { b0 = ph + cr; bstep = G; }
      else if (cr == fct) { b0 = ph; bstep = nbk; }
      else { b0 = ph + 1 + (cr - fct - 1 + G) % G; bstep = G - 1; }
      const bool partial = ph == np && qw < NB && k > r && ((ph - 1) % G) == cr;
      const bool busy = b0 < nbk || partial;
      // panel ph-1 is read once per owned block: stage it (asynchronous
      // copies, one L2 round trip) when it fits
      const double* Y = Yg;
      int ldy = ld;
      if (busy && pad_ld(rows) * NB <= YBUF) {
        ldy = pad_ld(rows);
        stage_cols(S.ybuf, ldy, Yg, ld, rows, qw);
        Y = S.ybuf;
      } else {
        __syncthreads();
      }
      // a partial last panel (r not a multiple of NB, k > r): the rest of its
      // own block lies beyond the reflectors and still needs panel ph-1
      if (partial) {
        const int c1 = min(k, q0 + NB);
        apply_panel_cols(Y, ldy, rows, qw, S.tp, W + q0 + (size_t)r * ld, ld, c1 - r, true, S, S.panel,
                         (STAGE_ROWS + 4) * NB);
      }
      for (int b = b0; b < nbk; b += bstep) {
        const int c0 = b * NB, cw = min(NB, k - c0);
        double* Xg = W + q0 + (size_t)c0 * ld;
        if (b == ph && ph < np && rows <= STAGE_ROWS) {
          // block ph becomes panel ph: stage it, apply panel ph-1 in shared
          // memory, factor it in place, write it back once
#ifdef HQ_DEBUG_TIMING
          tB = clock64();
#endif
          const int lds = pad_ld(rows);
          stage_cols(S.panel, lds, Xg, ld, rows, cw);
          apply_panel_cols(Y, ldy, rows, qw, S.tp, S.panel, lds, cw, true, S);
          factor_panel_core(Q, S.panel + NB, lds, rows - NB, min(NB, r - ph * NB), ph * NB, S);
          __syncthreads();
          for (int c = 0; c < cw; ++c)
            for (int i = t; i < rows; i += NT) Xg[i + (size_t)c * ld] = S.panel[i + c * lds];
          // factoring overwrote S.tp with T_ph: restore T_(ph-1)
          if (t < NB * NB) S.tp[t] = Q.tpanel[(size_t)(ph - 1) * NB * NB + t];
          __syncthreads();
#ifdef HQ_DEBUG_TIMING
          tC = clock64();
#endif
        } else {
          apply_panel_cols(Y, ldy, rows, qw, S.tp, Xg, ld, cw, true, S, S.panel, (STAGE_ROWS + 4) * NB);
          if (b == ph && ph < np) {
            factor_panel_step(Q, W, ld, m, k, r, ph * NB, false, false, S);
            if (t < NB * NB) S.tp[t] = Q.tpanel[(size_t)(ph - 1) * NB * NB + t];
            __syncthreads();
          }
        }
      }
    } else if (ph == 0 && np > 0 && cr == 0) {
      factor_panel_step(Q, W, ld, m, k, r, 0, false, false, S);
    }
    // full compact-WY T: the CTAs not factoring this phase form X of panel
    // ph-1 and the T12 block of panel ph-2 (split merge, see merge_X_split)
    if (Q.tfull && ph >= 1) {
      const bool fact_now = ph < np;
      const int fct = ph % G;
      if (!(fact_now && cr == fct)) {
        const int nparts = fact_now ? G - 1 : G;
        const int part = fact_now ? (cr - fct - 1 + G) % G : cr;
        __syncthreads();
        if (ph - 1 < np) merge_X_split(Q, W, ld, m, r, (ph - 1) * NB, Xs + (size_t)((ph - 1) & 1) * r * NB,
                                       part, nparts, S);
        if (ph >= 2) {
          __syncthreads();
          merge_T12_split(Q, r, (ph - 2) * NB, Xs + (size_t)((ph - 2) & 1) * r * NB, part, nparts, S);
        }
      }
    }
    __syncthreads();
#ifdef HQ_DEBUG_TIMING
    long long tD = clock64();
#endif
    cluster.sync();
#ifdef HQ_DEBUG_TIMING
    long long tE = clock64();
    if (threadIdx.x == 0 && blockIdx.x < 8 && ph < 64 && hq_dbg) {
      long long* d = hq_dbg + (blockIdx.x * 64 + ph) * 4;
      d[0] = tB - tA; d[1] = tC - tB; d[2] = tD - tC; d[3] = tE - tD;
    }
#endif
  }
}

// grid (problem, column chunk of cwk): the columns of X are independent, so
// each CTA applies all reflectors to its own chunk.  The launch sizes the
// shared memory for its tallest problem (ldcap = pad_ld(max rows)): the chunk
// of X (cwk = 32, 16 or 8 columns, the widest that fits beside one panel of
// reflectors) stays in shared memory for the whole sweep over the panels, and
// every panel's reflectors and T factor arrive by bulk copies (one
// cp.async.bulk per column, completion on an mbarrier) -- into the other of
// two buffers while the current panel is applied when both fit (nbuf = 2).
// Problems taller than the launch's capacity (ldcap = 0: none staged) run
// from global memory.
struct ApqSmem {
  double tp[2][NB * NB];
  double wsp[WSP];
  unsigned long long bar[4];   // [0], [1]: panel buffers; [2]: the chunk of X
};
static_assert(sizeof(ApqSmem) % 16 == 0, "staging buffers follow ApqSmem 16-byte aligned");
// apply_panel_cols reads S.wsp only
constexpr int APQ_SMEM_MAX = 232448;   // opt-in shared memory per CTA (227 KB)

__global__ void __launch_bounds__(NT) applyq_kernel(const hq_applyq_prob* __restrict__ probs,
                                                    int* __restrict__ rank, int cwk, int ldcap, int nbuf) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  ApqSmem& S = *reinterpret_cast<ApqSmem*>(smem_raw);
  double* const xbuf = reinterpret_cast<double*>(smem_raw + sizeof(ApqSmem));
  double* const ybuf0 = xbuf + (size_t)ldcap * cwk;
  double* const ybuf1 = nbuf == 2 ? ybuf0 + (size_t)ldcap * NB : ybuf0;
  const hq_applyq_prob A = probs[blockIdx.x];
  const int m = hq_dim(rank, A.m, A.m_ri), k = hq_dim(rank, A.k, A.k_ri);
  const int call = hq_dim(rank, A.c, A.c_ri);
  const int r = m < k ? m : k;
  const int t = threadIdx.x;
  const int cbeg = blockIdx.y * cwk;
  if (m <= 0 || cbeg >= call) return;
  const int c = min(cwk, call - cbeg);
  double* Xg = A.x + (size_t)cbeg * A.ldx;
  const bool staged = ldcap > 0 && pad_ld(m) <= ldcap;
  const int np = (r + NB - 1) / NB;
  if (!staged) {
    // ---- global-memory path
    if (A.x0) {
      const int r0 = hq_dim(rank, A.r0, A.r0_ri);
      const double* X0 = A.x0 + (size_t)cbeg * A.ldx0;
      for (int j = 0; j < c; ++j)
        for (int i = t; i < m; i += NT) Xg[i + (size_t)j * A.ldx] = i < r0 ? X0[i + (size_t)j * A.ldx0] : 0.0;
      __syncthreads();
    }
    for (int s = 0; s < np; ++s) {
      const int p = A.trans ? s : np - 1 - s;
      const int p0 = p * NB, pw = min(NB, r - p0), rows = m - p0;
      if (t < NB * NB) S.tp[0][t] = A.tpanel[(size_t)p * NB * NB + t];
      __syncthreads();
      apply_panel_cols(A.w + p0 + (size_t)p0 * A.ldw, A.ldw, rows, pw, S.tp[0], Xg + p0, A.ldx, c, A.trans != 0, S);
    }
    return;
  }
  // ---- staged path
  const int ldx = pad_ld(m);
  const bool ybulk = ((((uintptr_t)A.w | (uintptr_t)A.tpanel) & 15) == 0) && (A.ldw & 1) == 0;
  if (t == 0) { mbar_init(&S.bar[0], 1); mbar_init(&S.bar[1], 1); mbar_init(&S.bar[2], 1); }
  __syncthreads();
  unsigned par[2] = {0u, 0u};
  // start the copy of panel step s (reflectors + T factor) into its buffer
  auto issue = [&](int s) {
    const int b = nbuf == 2 ? (s & 1) : 0;
    const int p = A.trans ? s : np - 1 - s;
    const int p0 = p * NB, pw = min(NB, r - p0), rows = m - p0;
    const double* Y = A.w + p0 + (size_t)p0 * A.ldw;
    const double* tpg = A.tpanel + (size_t)p * NB * NB;
    double* yb = b ? ybuf1 : ybuf0;
    const int ldy = pad_ld(rows);
    if (ybulk) {
      const int re = rows & ~1;
      if (t < 32) {
        if (t == 0) {
          mbar_expect_tx(&S.bar[b], (unsigned)(pw * re + NB * NB) * 8u);
          bulk_g2s(S.tp[b], tpg, NB * NB * 8u, &S.bar[b]);
        }
        __syncwarp();
        if (re > 0 && t < pw) bulk_g2s(yb + (size_t)t * ldy, Y + (size_t)t * A.ldw, (unsigned)re * 8u, &S.bar[b]);
      } else if (rows & 1) {
        for (int j = t - 32; j < pw; j += NT - 32) yb[re + (size_t)j * ldy] = Y[re + (size_t)j * A.ldw];
      }
    } else {
      if (t < NB * NB) S.tp[b][t] = tpg[t];
      for (int j = 0; j < pw; ++j)
        for (int i = t; i < rows; i += NT) cp_async8(yb + i + (size_t)j * ldy, Y + i + (size_t)j * A.ldw);
    }
  };
  auto arrived = [&](int s) {
    const int b = nbuf == 2 ? (s & 1) : 0;
    if (ybulk) { mbar_wait(&S.bar[b], par[b]); par[b] ^= 1u; }
    else cp_async_wait_all();
    __syncthreads();
  };
  if (np > 0) issue(0);
  if (A.x0) {
    const int r0 = hq_dim(rank, A.r0, A.r0_ri);
    const double* X0 = A.x0 + (size_t)cbeg * A.ldx0;
    for (int j = 0; j < c; ++j)
      for (int i = t; i < m; i += NT) xbuf[i + (size_t)j * ldx] = i < r0 ? X0[i + (size_t)j * A.ldx0] : 0.0;
  } else {
    unsigned px = 0;
    stage_cols_bulk(xbuf, ldx, Xg, A.ldx, m, c, &S.bar[2], px);
  }
  for (int s = 0; s < np; ++s) {
    if (nbuf == 2 && s + 1 < np) issue(s + 1);
    arrived(s);   // its barrier also publishes the chunk of X before the first panel
    const int b = nbuf == 2 ? (s & 1) : 0;
    const int p = A.trans ? s : np - 1 - s;
    const int p0 = p * NB, pw = min(NB, r - p0), rows = m - p0;
    apply_panel_cols(b ? ybuf1 : ybuf0, pad_ld(rows), rows, pw, S.tp[b], xbuf + p0, ldx, c, A.trans != 0, S);
    if (nbuf == 1 && s + 1 < np) issue(s + 1);
  }
  if (np == 0) __syncthreads();
  store_cols_bulk(Xg, A.ldx, xbuf, ldx, m, c);
}

// dst (rows x K) = [alpha_1 P_1 | alpha_2 P_2 | ...]; K -> rank[ktot_ri]
__global__ void concat_kernel(const hq_concat_prob* __restrict__ probs,
                              const hq_piece* __restrict__ pieces, int* __restrict__ rank) {
  const hq_concat_prob C = probs[blockIdx.y];
  int col = 0;
  for (int q = 0; q < C.npiece; ++q) {
    const hq_piece Pc = pieces[C.piece0 + q];
    const int nc = hq_dim(rank, Pc.cols, Pc.cols_ri);
    // two rows per thread by 16-byte accesses when every column start is
    // 16-byte aligned on all sides; four columns in flight either way
    const bool vec = (C.rows & 1) == 0 && ((Pc.ld | C.ldd | (C.dst2 ? C.ldd2 : 0)) & 1) == 0 &&
                     ((((uintptr_t)Pc.p | (uintptr_t)C.dst | (uintptr_t)C.dst2) & 15) == 0);
    if (vec) {
      for (int i = 2 * (blockIdx.x * blockDim.x + threadIdx.x); i < C.rows; i += 2 * gridDim.x * blockDim.x) {
#pragma unroll 4
        for (int j = 0; j < nc; ++j) {
          double2 v = __ldg(reinterpret_cast<const double2*>(Pc.p + i + (size_t)j * Pc.ld));
          v.x *= Pc.alpha;
          v.y *= Pc.alpha;
          *reinterpret_cast<double2*>(C.dst + i + (size_t)(col + j) * C.ldd) = v;
          if (C.dst2) *reinterpret_cast<double2*>(C.dst2 + i + (size_t)(col + j) * C.ldd2) = v;
        }
      }
    } else {
      for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < C.rows; i += gridDim.x * blockDim.x) {
#pragma unroll 4
        for (int j = 0; j < nc; ++j) {
          const double v = Pc.alpha * Pc.p[i + (size_t)j * Pc.ld];
          C.dst[i + (size_t)(col + j) * C.ldd] = v;
          if (C.dst2) C.dst2[i + (size_t)(col + j) * C.ldd2] = v;
        }
      }
    }
    col += nc;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0 && C.ktot_ri >= 0) rank[C.ktot_ri] = col;
}

// panel = [leaf; slab_1^T; slab_2^T; ...]  (compressed leaf column)
__global__ void leaf_gather_kernel(const hq_leaf_prob* __restrict__ probs,
                                   const hq_slab* __restrict__ slabs, int* __restrict__ rank) {
  const hq_leaf_prob L = probs[blockIdx.y];
  const int nl = L.nl;
  const int c = blockIdx.x;  // column
  if (c >= nl) return;
  for (int i = threadIdx.x; i < nl; i += blockDim.x)
    L.panel[i + (size_t)c * L.ldp] = L.leaf[i + (size_t)c * nl];
  int row = nl;
  for (int s = 0; s < L.nslab; ++s) {
    const hq_slab B = slabs[L.slab0 + s];
    const int kk = rank[B.k_ri];
    for (int i = threadIdx.x; i < kk; i += blockDim.x)
      L.panel[row + i + (size_t)c * L.ldp] = B.v[c + (size_t)i * B.ld];
    row += kk;
  }
  if (c == 0 && threadIdx.x == 0 && L.m_ri >= 0) rank[L.m_ri] = row;
}

// leaf <- panel[0:nl, :] (R + Y), slab Y rows -> yv
__global__ void leaf_scatter_kernel(const hq_leaf_prob* __restrict__ probs,
                                    const hq_slab* __restrict__ slabs, int* __restrict__ rank) {
  const hq_leaf_prob L = probs[blockIdx.y];
  const int nl = L.nl;
  const int c = blockIdx.x;
  if (c >= nl) return;
  for (int i = threadIdx.x; i < nl; i += blockDim.x)
    L.leaf[i + (size_t)c * nl] = L.panel[i + (size_t)c * L.ldp];
  int row = nl;
  for (int s = 0; s < L.nslab; ++s) {
    const hq_slab B = slabs[L.slab0 + s];
    const int kk = rank[B.k_ri];
    for (int i = threadIdx.x; i < kk; i += blockDim.x)
      B.yv[c + (size_t)i * B.ldy] = L.panel[row + i + (size_t)c * L.ldp];
    row += kk;
  }
}

__global__ void zero_kernel(const int64_t* __restrict__ regions) {
  double* p = reinterpret_cast<double*>(regions[2 * blockIdx.y]);
  const int64_t n = regions[2 * blockIdx.y + 1];
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    p[e] = 0.0;
}

__global__ void copy_kernel(const hq_copy_item* __restrict__ items, const int* __restrict__ rank) {
  const hq_copy_item it = items[blockIdx.x];
  const int cols = hq_dim(rank, it.cols, it.cols_ri);
  const size_t n = (size_t)it.rows * cols;
  for (size_t e = threadIdx.x; e < n; e += blockDim.x) {
    const int i = (int)(e % it.rows), j = (int)(e / it.rows);
    double v = it.src[i + (size_t)j * it.lds];
    if (it.mode == 1 && i > j) v = 0.0;
    if (it.mode == 2) v = i < j ? 0.0 : (i == j ? 1.0 : v);
    it.dst[i + (size_t)j * it.ldd] = v;
  }
}

// single-CTA exclusive scan of rows*cols -> dst = base + offset, ldd = rows
__global__ void pack_offsets_kernel(hq_copy_item* items, int nitem, const int* rank, double* base,
                                    int64_t* total, int which) {
  __shared__ int64_t carry;
  __shared__ int64_t wsum[32];
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int c0 = 0; c0 < nitem; c0 += blockDim.x) {
    const int i = c0 + threadIdx.x;
    int64_t v = 0;
    if (i < nitem) v = (int64_t)items[i].rows * hq_dim(rank, items[i].cols, items[i].cols_ri);
    int64_t x = v;
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[wid] = x;
    __syncthreads();
    if (wid == 0) {
      int64_t w = lane < (int)(blockDim.x >> 5) ? wsum[lane] : 0;
      for (int o = 1; o < 32; o <<= 1) {
        const int64_t y = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += y;
      }
      wsum[lane] = w;
    }
    __syncthreads();
    const int64_t excl = carry + x - v + (wid > 0 ? wsum[wid - 1] : 0);
    if (i < nitem) {
      if (which) { items[i].src = base + excl; items[i].lds = items[i].rows; }
      else { items[i].dst = base + excl; items[i].ldd = items[i].rows; }
    }
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry = excl + v;
    __syncthreads();
  }
  if (threadIdx.x == 0) total[0] = carry;
}

__global__ void rowblk_kernel(const hq_rowblk_prob* __restrict__ probs, int* __restrict__ rank) {
  const hq_rowblk_prob B = probs[blockIdx.y];
  const int c = blockIdx.x;
  const int nch = (B.rows_total + B.ch - 1) / B.ch;
  if (c >= nch) return;
  const int K = hq_dim(rank, B.k, B.k_ri);
  // stacked offset of chunk c: every full chunk contributes min(ch, K) rows
  const int kr_full = min(B.ch, K);
  const int off = c * kr_full;
  const int rows_c = min(B.ch, B.rows_total - c * B.ch);
  const int kr = min(rows_c, K);
  if (B.mode == 0) {
    for (int e = threadIdx.x; e < kr * K; e += blockDim.x) {
      const int a = e % kr, b = e / kr;
      B.s[(off + a) + (size_t)b * B.lds] = a <= b ? B.w[(c * B.ch + a) + (size_t)b * B.ldw] : 0.0;
    }
    if (c == nch - 1 && threadIdx.x == 0) rank[B.ms_ri] = off + kr;
  } else {
    const int nc = hq_dim(rank, B.ncol, B.ncol_ri);
    for (int e = threadIdx.x; e < rows_c * nc; e += blockDim.x) {
      const int i = e % rows_c, j = e / rows_c;
      B.w[(c * B.ch + i) + (size_t)j * B.ldw] = i < kr ? B.s[(off + i) + (size_t)j * B.lds] : 0.0;
    }
  }
}

bool g_attr_done = false;
}  // namespace

static int qr_smem_attr() {
  if (!g_attr_done) {
    cudaError_t e = cudaFuncSetAttribute(qr_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(QrSmem));
    if (e != cudaSuccess) return (int)e;
    g_attr_done = true;
  }
  return 0;
}

template <int G>
static int launch_qr_cluster(cudaStream_t st, const hq_qr_prob* probs, int nprob, int* rank) {
  static bool attr = false;
  auto kern = qr_cluster_kernel<G>;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(QrSmem));
    if (e != cudaSuccess) return (int)e;
    attr = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nprob * G);
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = sizeof(QrSmem);
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = G;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return (int)cudaLaunchKernelEx(&cfg, kern, probs, rank);
}

extern "C" int hq_qr(void* stream, const hq_qr_prob* probs, int nprob, int* rank, int cluster) {
  if (nprob <= 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  if (cluster >= 8) return launch_qr_cluster<8>(st, probs, nprob, rank);
  if (cluster >= 4) return launch_qr_cluster<4>(st, probs, nprob, rank);
  if (cluster >= 2) return launch_qr_cluster<2>(st, probs, nprob, rank);
  int e = qr_smem_attr();
  if (e) return e;
  qr_kernel<<<nprob, NT, sizeof(QrSmem), st>>>(probs, rank);
  return hq_err(cudaGetLastError());
}

extern "C" int hq_applyq(void* stream, const hq_applyq_prob* probs, int nprob, int* rank,
                         int max_cols, int max_rows) {
  if (nprob <= 0) return 0;
  static bool attr = false;
  static int force_cw = 0, force_nbuf = 0;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(applyq_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, APQ_SMEM_MAX);
    if (e != cudaSuccess) return hq_err(e);
    if (const char* v = getenv("HQ_APQ_CW")) force_cw = atoi(v);       // experiments only
    if (const char* v = getenv("HQ_APQ_NBUF")) force_nbuf = atoi(v);
    attr = true;
  }
  // chunk width / buffers from the tallest problem of the launch (unknown: 512 rows)
  const long long avail = (APQ_SMEM_MAX - (long long)sizeof(ApqSmem)) / 8;
  const int ld = pad_ld(max_rows > 0 ? max_rows : 512);
  int cwk = 0;
  for (int cw : {32, 16, 8})
    if ((long long)ld * (cw + NB) <= avail && (force_cw == 0 || cw <= force_cw)) { cwk = cw; break; }
  int ldcap = ld, nbuf = 1;
  if (cwk == 0 || force_cw < 0) { cwk = 32; ldcap = 0; }
  else if ((long long)ld * (cwk + 2 * NB) <= avail && force_nbuf != 1) nbuf = 2;
  const size_t smem = sizeof(ApqSmem) + (size_t)ldcap * (cwk + nbuf * NB) * 8;
  const int nchunk = max_cols > 0 ? (max_cols + cwk - 1) / cwk : 1;
  applyq_kernel<<<dim3(nprob, nchunk), NT, smem, (cudaStream_t)stream>>>(probs, rank, cwk, ldcap, nbuf);
  return hq_err(cudaGetLastError());
}

extern "C" int hq_concat(void* stream, const hq_concat_prob* probs, int nprob,
                         const hq_piece* pieces, int* rank, int max_rows) {
  if (nprob <= 0) return 0;
  dim3 grid((max_rows + 255) / 256, nprob);
  if (grid.x == 0) grid.x = 1;
  concat_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(probs, pieces, rank);
  return hq_err(cudaGetLastError());
}

extern "C" int hq_leaf_gather(void* stream, const hq_leaf_prob* probs, int nprob,
                              const hq_slab* slabs, int* rank, int max_nl) {
  if (nprob <= 0) return 0;
  leaf_gather_kernel<<<dim3(max_nl, nprob), 128, 0, (cudaStream_t)stream>>>(probs, slabs, rank);
  return hq_err(cudaGetLastError());
}

extern "C" int hq_leaf_scatter(void* stream, const hq_leaf_prob* probs, int nprob,
                               const hq_slab* slabs, int* rank, int max_nl) {
  if (nprob <= 0) return 0;
  leaf_scatter_kernel<<<dim3(max_nl, nprob), 128, 0, (cudaStream_t)stream>>>(probs, slabs, rank);
  return hq_err(cudaGetLastError());
}

extern "C" int hq_zero(void* stream, const int64_t* regions, int nregion, int64_t max_count) {
  if (nregion <= 0) return 0;
  int gx = (int)((max_count + 255) / 256);
  if (gx > 1024) gx = 1024;
  if (gx < 1) gx = 1;
  zero_kernel<<<dim3(gx, nregion), 256, 0, (cudaStream_t)stream>>>(regions);
  return hq_err(cudaGetLastError());
}

extern "C" int hq_copy(void* stream, const hq_copy_item* items, int nitem, const int* rank) {
  if (nitem <= 0) return 0;
  copy_kernel<<<nitem, 256, 0, (cudaStream_t)stream>>>(items, rank);
  return hq_err(cudaGetLastError());
}

extern "C" int hq_pack_offsets(void* stream, hq_copy_item* items, int nitem, const int* rank,
                               double* base, int64_t* total, int which) {
  if (nitem <= 0) return 0;
  pack_offsets_kernel<<<1, 1024, 0, (cudaStream_t)stream>>>(items, nitem, rank, base, total, which);
  return hq_err(cudaGetLastError());
}

extern "C" int hq_rowblocks(void* stream, const hq_rowblk_prob* probs, int nprob, int* rank,
                            int max_chunks) {
  if (nprob <= 0 || max_chunks <= 0) return 0;
  rowblk_kernel<<<dim3(max_chunks, nprob), 256, 0, (cudaStream_t)stream>>>(probs, rank);
  return hq_err(cudaGetLastError());
}
