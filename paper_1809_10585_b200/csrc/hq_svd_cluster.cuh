// One-sided block Jacobi on a thread-block cluster (included by hq_svd.cu).
// For truncation cores too large for one SM (m*n > ~24K doubles, or more
// pairs per round than one CTA has lane groups), the n columns of X are split
// into 2G blocks of bs columns; CTA c of a G-CTA cluster holds two blocks in
// its shared memory.  A sweep = intra-block pairs (circle method inside both
// blocks) + the 2G-1 rounds of a block round-robin tournament: each round
// every CTA rotates all pairs between its two blocks (the slot-0 columns stay
// in registers for the whole round, only slot-1 columns stream through
// shared memory), then every CTA pushes its two blocks into the spare buffer
// set of the CTAs that own their next tournament positions (distributed
// shared memory stores) and the cluster meets at ONE barrier; buffer sets
// alternate, so nothing is copied locally.  The convergence flags travel with
// the last push of a sweep.  Columns never leave the cluster's SMs until U_k
// is written.
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

#ifndef HQ_SVD_SINGLE_MAX_PAIRS
#define HQ_SVD_SINGLE_MAX_PAIRS 16
#endif

namespace {
constexpr int CNT = 512, CNW = CNT / 32;
constexpr int C_MAX_BS = 64;          // max columns per block
constexpr int C_SMEM_DOUBLES = 26880; // 210 KB: 2 buffer sets x 2 blocks (the kernel reserves ~224 KB for the single-CTA fallback anyway)

struct CSmem {
  double buf[C_SMEM_DOUBLES];
  double nrm[4][C_MAX_BS];   // squared norms, [set * 2 + slot]
  int col[4][C_MAX_BS];      // global column index per slot (-1: pad)
  double sig_all[1024];
  int flag[2][16];           // rotation flags of every CTA, by sweep parity
  double2 trash[32];         // sink for the stores of rows past the column end
  int rot;
  int cnt;
#ifdef HQ_DEBUG_SWEEPS
  long long dbg[4];
#endif
};

// block owner map of the circle tournament: position -> (cta, slot)
// top row: positions 0..G-1 are slot 0 of CTA c; bottom row: slot 1 of CTA
// c holds position 2G-1-c.  Each round, position 0 stays, the others rotate.
__device__ __forceinline__ int circ_next(int pos, int G) {
  // block at tournament position pos moves to this position next round
  const int P = 2 * G;
  if (pos == 0) return 0;
  return pos == P - 1 ? 1 : pos + 1;
}

template <int G, int LP, int E>
__device__ __noinline__ void svd_cluster_body(const hq_svd_prob& P, int* __restrict__ rank, int m, int n,
                                                 double thr, CSmem& S, cg::cluster_group& cluster) {
  const int cr = (int)cluster.block_rank();
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  constexpr int GPW = 32 / LP;
  const int grp = wid * GPW + lane / LP, gl = lane % LP, ngroups = CNW * GPW;
  const int ld = (m + 1) & ~1;
  const int bs = (n + 2 * G - 1) / (2 * G);
  // buffer set k: blocks Bk(slot) = buf + (2k + slot) bs ld; sets alternate per exchange
  auto blk = [&](int set, int slot) { return S.buf + (size_t)(2 * set + slot) * bs * ld; };
  // ---- initial load into set 0: CTA cr holds positions cr (slot 0) and 2G-1-cr (slot 1)
  for (int slot = 0; slot < 2; ++slot) {
    const int pos = slot == 0 ? cr : 2 * G - 1 - cr;
    for (int jj = 0; jj < bs; ++jj) {
      const int j = pos * bs + jj;
      double* dst = blk(0, slot) + (size_t)jj * ld;
      for (int i = t; i < ld; i += CNT) {
        double v = 0.0;
        if (j < n && i < m) v = P.xform ? ((j <= i || P.xform == 2) ? P.c[j + (size_t)i * P.ldc] : 0.0)
                                        : P.c[i + (size_t)j * P.ldc];
        dst[i] = v;
      }
      if (t == 0) S.col[slot][jj] = j < n ? j : -1;
    }
  }
  // destination (cta, slot) of my two blocks after each tournament round
  int dcta[2], dslot[2];
  for (int slot = 0; slot < 2; ++slot) {
    const int np = circ_next(slot == 0 ? cr : 2 * G - 1 - cr, G);
    dcta[slot] = np < G ? np : 2 * G - 1 - np;
    dslot[slot] = np < G ? 0 : 1;
  }
  cluster.sync();
  const double tol = 4.0 * sqrt((double)m) * 2.220446049250313e-16;
  const double tiny2 = (1e-3 * thr) * (1e-3 * thr), thr2 = thr * thr, tol2 = tol * tol;
  const bool reg_x = bs <= ngroups;   // one pass of groups per round: slot-0 column in registers
  int cur = 0;
#ifdef HQ_DEBUG_SWEEPS
  if (t < 4) S.dbg[t] = 0;
  long long dbg_t[4] = {0, 0, 0, 0};
  long long dbg_c = clock64();
#define HQ_DBG_MARK(k) do { const long long c_ = clock64(); dbg_t[k] += c_ - dbg_c; dbg_c = c_; } while (0)
#else
#define HQ_DBG_MARK(k) do { } while (0)
#endif
  int nsw = 0;
  for (int sweep = 0; sweep < MAX_SWEEPS; ++sweep) {
    nsw = sweep + 1;
    double* B0 = blk(cur, 0);
    double* B1 = blk(cur, 1);
    double* nrm0 = S.nrm[2 * cur];
    double* nrm1 = S.nrm[2 * cur + 1];
    const int* col0 = S.col[2 * cur];
    const int* col1 = S.col[2 * cur + 1];
    // squared norms of the two working blocks
    for (int j = wid; j < 2 * bs; j += CNW) {
      const double* x = (j < bs ? B0 : B1) + (size_t)(j % bs) * ld;
      double v = 0.0;
      for (int i = lane; i < ld; i += 32) v = fma(x[i], x[i], v);
      v = warp_sum(v);
      if (lane == 0) (j < bs ? nrm0 : nrm1)[j % bs] = v;
    }
    if (t == 0) S.rot = 0;
    __syncthreads();
    HQ_DBG_MARK(0);
    // intra-block pairs of both working blocks (round robin inside each block)
    {
      const int npb = bs + (bs & 1), N = npb - 1, hp = npb / 2;
      for (int r = 0; r < N; ++r) {
        for (int g0 = 0; g0 < 2 * hp; g0 += ngroups) {
          if (g0 + wid * GPW >= 2 * hp) break;  // warp-uniform
          const int gi = g0 + grp;
          const int bk = gi >= hp ? 1 : 0, pi = gi - bk * hp;
          const int* colb = bk ? col1 : col0;
          double* nrmb = bk ? nrm1 : nrm0;
          int p = 0, q = 0;
          bool act = gi < 2 * hp;
          if (act) {
            p = r; q = N;
            if (pi != 0) {
              p = r + pi; if (p >= N) p -= N;
              q = r - pi; if (q < 0) q += N;
            }
            if (p > q) { const int x = p; p = q; q = x; }
            act = q < bs && colb[p] >= 0 && colb[q] >= 0;
          }
          if (!act) { p = 0; q = 0; }
          double a = act ? nrmb[p] : 0.0, b = act ? nrmb[q] : 0.0;
          double* Bb = bk ? B1 : B0;
          double xp[E];
          const int rr = jacobi_pair<LP, E, false>(xp, Bb + (size_t)p * ld, Bb + (size_t)q * ld, a, b, ld, tol2,
                                                   tiny2, thr2, gl, act, S.trash);
          if (rr && gl == 0) { nrmb[p] = a; nrmb[q] = b; if (rr > 1) S.rot = 1; }
        }
        __syncthreads();
      }
    }
    HQ_DBG_MARK(1);
    // 2G-1 tournament rounds of inter-block pairs, each followed by a push
    for (int round = 0; round < 2 * G - 1; ++round) {
      if (reg_x) {
        const int i = grp;
        const bool own = i < bs && col0[i] >= 0;
        double xp[E];
        double a = own ? nrm0[i] : 0.0;
#pragma unroll
        for (int e = 0; e < E / 2; ++e) {
          const int ii = 2 * gl + 2 * LP * e;
          double2 v = make_double2(0.0, 0.0);
          if (own && ii < ld) v = *reinterpret_cast<const double2*>(B0 + (size_t)i * ld + ii);
          xp[2 * e] = v.x; xp[2 * e + 1] = v.y;
        }
        bool any = false;
        for (int r = 0; r < bs; ++r) {
#ifdef HQ_DEBUG_SWEEPS
          const long long q0 = clock64();
#endif
          if (wid * GPW < bs) {  // warp-uniform
            int j = i + r; if (j >= bs) j -= bs;
            if (!own) j = 0;
            const bool act = own && col1[j] >= 0;
            double b = act ? nrm1[j] : 0.0;
            const int rr = jacobi_pair<LP, E, true>(xp, B0, B1 + (size_t)j * ld, a, b, ld, tol2, tiny2, thr2, gl,
                                                     act, S.trash);
            if (rr && gl == 0) nrm1[j] = b;
            any |= rr > 1;
          }
#ifdef HQ_DEBUG_SWEEPS
          const long long q1 = clock64();
#endif
          __syncthreads();
#ifdef HQ_DEBUG_SWEEPS
          if (t == 0) { S.dbg[0] += q1 - q0; S.dbg[1] += clock64() - q1; S.dbg[2] += 1; }
#endif
        }
        if (own) {
#pragma unroll
          for (int e = 0; e < E / 2; ++e) {
            const int ii = 2 * gl + 2 * LP * e;
            if (ii < ld)
              *reinterpret_cast<double2*>(B0 + (size_t)i * ld + ii) = make_double2(xp[2 * e], xp[2 * e + 1]);
          }
          if (gl == 0) { nrm0[i] = a; if (any) S.rot = 1; }
        }
      } else {
        for (int r = 0; r < bs; ++r) {
          for (int g0 = 0; g0 < bs; g0 += ngroups) {
            if (g0 + wid * GPW >= bs) break;  // warp-uniform
            const int i = g0 + grp;
            int j = i + r; if (j >= bs) j -= bs;
            bool act = i < bs && col0[i] >= 0 && col1[j] >= 0;
            double a = act ? nrm0[i] : 0.0, b = act ? nrm1[j] : 0.0;
            double xp[E];
            const int rr = jacobi_pair<LP, E, false>(xp, B0 + (size_t)(act ? i : 0) * ld,
                                                      B1 + (size_t)(act ? j : 0) * ld, a, b, ld, tol2, tiny2, thr2,
                                                      gl, act, S.trash);
            if (rr && gl == 0) { nrm0[i] = a; nrm1[j] = b; if (rr > 1) S.rot = 1; }
          }
          __syncthreads();
        }
      }
      __syncthreads();
      HQ_DBG_MARK(2);
      // push both blocks (and their norms / column ids) to the next owners' spare set
      const int nxt = cur ^ 1;
      for (int slot = 0; slot < 2; ++slot) {
        CSmem* R = cluster.map_shared_rank(&S, dcta[slot]);
        const double2* src = reinterpret_cast<const double2*>(blk(cur, slot));
        double2* dst = reinterpret_cast<double2*>(R->buf + (size_t)(2 * nxt + dslot[slot]) * bs * ld);
        for (int e = t; e < bs * ld / 2; e += CNT) dst[e] = src[e];
      }
      for (int slot = 0; slot < 2; ++slot) {
        CSmem* R = cluster.map_shared_rank(&S, dcta[slot]);
        for (int jj = t; jj < bs; jj += CNT) {
          R->nrm[2 * nxt + dslot[slot]][jj] = S.nrm[2 * cur + slot][jj];
          R->col[2 * nxt + dslot[slot]][jj] = S.col[2 * cur + slot][jj];
        }
      }
      if (round == 2 * G - 2 && t < G) cluster.map_shared_rank(&S, t)->flag[sweep & 1][cr] = S.rot;
      cluster.sync();
      HQ_DBG_MARK(3);
      cur = nxt;
      B0 = blk(cur, 0); B1 = blk(cur, 1);
      nrm0 = S.nrm[2 * cur]; nrm1 = S.nrm[2 * cur + 1];
      col0 = S.col[2 * cur]; col1 = S.col[2 * cur + 1];
    }
    int any = 0;
#pragma unroll
    for (int c = 0; c < G; ++c) any |= S.flag[sweep & 1][c];
    if (!any) break;
    // the blocks are now at shifted positions; the next sweep starts from
    // the current placement (any placement is a valid starting position)
  }
#ifdef HQ_DEBUG_SWEEPS
  if (cr == 0 && t == 0 && P.flag_ri >= 0) {
    rank[P.flag_ri + 1] = nsw;
    for (int k = 0; k < 4; ++k) rank[P.flag_ri + 2 + k] = (int)(dbg_t[k] >> 4);
    rank[P.flag_ri + 6] = (int)(S.dbg[0] / max(1LL, S.dbg[2]));
    rank[P.flag_ri + 7] = (int)(S.dbg[1] / max(1LL, S.dbg[2]));
  }
#endif
#undef HQ_DBG_MARK
  (void)nsw;
  double* Bs[2] = {blk(cur, 0), blk(cur, 1)};
  double* nrms[2] = {S.nrm[2 * cur], S.nrm[2 * cur + 1]};
  const int* cols[2] = {S.col[2 * cur], S.col[2 * cur + 1]};
  // ---- singular values, global order, output U_k
  for (int j = wid; j < 2 * bs; j += CNW) {
    const double* x = Bs[j / bs] + (size_t)(j % bs) * ld;
    double v = 0.0;
    for (int i = lane; i < ld; i += 32) v = fma(x[i], x[i], v);
    v = sqrt(warp_sum(v));
    if (lane == 0) nrms[j / bs][j % bs] = cols[j / bs][j % bs] >= 0 ? v : -1.0;
  }
  cluster.sync();
  // gather sigma of every slot of every CTA
  for (int e = t; e < G * 2 * bs; e += CNT) {
    const int c = e / (2 * bs), k = e % (2 * bs);
    CSmem* R = cluster.map_shared_rank(&S, c);
    S.sig_all[e] = R->nrm[2 * cur + k / bs][k % bs];
  }
  if (t == 0) S.cnt = 0;
  cluster.sync();
  const int tot = G * 2 * bs;
  for (int k = wid; k < 2 * bs; k += CNW) {
    const int e = cr * 2 * bs + k;
    const double sj = S.sig_all[e];
    if (!(sj > thr)) continue;
    int pos = 0;
    for (int o = lane; o < tot; o += 32) {
      const double so = S.sig_all[o];
      pos += (so > sj || (so == sj && o < e)) ? 1 : 0;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) pos += __shfl_xor_sync(0xffffffffu, pos, off);
    if (lane == 0) atomicAdd(&S.cnt, 1);
    if (pos < P.cap) {
      const double inv = 1.0 / sj;
      const double* x = Bs[k / bs] + (size_t)(k % bs) * ld;
      for (int i = lane; i < m; i += 32) P.u[i + (size_t)pos * P.ldu] = x[i] * inv;
    }
  }
  cluster.sync();
  if (cr == 0 && t == 0) {
    int kk = 0;
    for (int c = 0; c < G; ++c) kk += cluster.map_shared_rank(&S, c)->cnt;
    if (kk > P.cap) { if (P.flag_ri >= 0) rank[P.flag_ri] = 1; kk = P.cap; }
    rank[P.rank_ri] = kk;
  }
  cluster.sync();
}

template <int G>
__global__ void __launch_bounds__(CNT, 1) svd_cluster_kernel(const hq_svd_prob* __restrict__ probs,
                                                             int* __restrict__ rank,
                                                             const double* __restrict__ scal) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  cg::cluster_group cluster = cg::this_cluster();
  const int cr = (int)cluster.block_rank();
  const hq_svd_prob P = probs[blockIdx.x / G];
  const int t = threadIdx.x;
  const int m = hq_dim(rank, P.m, P.m_ri);
  int n = hq_dim(rank, P.n, P.n_ri);
  if (P.xform) n = min(n, m);
  n = min(n, 1024);
  const double thr = P.eps_scale * (P.eps_slot >= 0 ? scal[P.eps_slot] : 1.0);
  if (m <= 0 || n <= 0) {
    if (cr == 0 && t == 0) rank[P.rank_ri] = 0;
    return;
  }
  // the plan sizes clusters from capacities; the run-time core decides: one
  // SM when it fits with few pairs per round (no exchange rounds), the
  // cluster when its blocks fit the cluster's shared memory, else CTA 0 alone
  // on the global-memory path
  const int ld = (m + 1) & ~1;
  const int bs = (n + 2 * G - 1) / (2 * G);
  const bool fits_single = (size_t)ld * n <= SMEM_DOUBLES;
  const bool fits_cluster = m <= 640 && 4 * bs * ld <= C_SMEM_DOUBLES && bs <= C_MAX_BS;
  if (!fits_cluster || (fits_single && (n + 1) / 2 <= HQ_SVD_SINGLE_MAX_PAIRS)) {
    if (cr == 0) svd_single(P, rank, scal, *reinterpret_cast<SvdSmem*>(smem_raw));
    return;
  }
  CSmem& S = *reinterpret_cast<CSmem*>(smem_raw);
  // lane-group shape from the pairs per CTA (bs) and the rows (m)
  // (rows per lane E sized to m: lanes past the column end only waste issue
  // slots on the latency-bound rounds)
  if constexpr (G == 16) {
    // 16-CTA clusters carry the widest cores only (m > 256): one lane group of 32 per pair
    if (m <= 256) svd_cluster_body<G, 32, 8>(P, rank, m, n, thr, S, cluster);
    else if (m <= 384) svd_cluster_body<G, 32, 12>(P, rank, m, n, thr, S, cluster);
    else if (m <= 512) svd_cluster_body<G, 32, 16>(P, rank, m, n, thr, S, cluster);
    else svd_cluster_body<G, 32, 20>(P, rank, m, n, thr, S, cluster);
    return;
  }
  if (m > 512) {
    svd_cluster_body<G, 32, 20>(P, rank, m, n, thr, S, cluster);
  } else if (bs <= 16 || m > 256) {
    if (m <= 128) svd_cluster_body<G, 32, 4>(P, rank, m, n, thr, S, cluster);
    else if (m <= 192) svd_cluster_body<G, 32, 6>(P, rank, m, n, thr, S, cluster);
    else if (m <= 256) svd_cluster_body<G, 32, 8>(P, rank, m, n, thr, S, cluster);
    else if (m <= 384) svd_cluster_body<G, 32, 12>(P, rank, m, n, thr, S, cluster);
    else svd_cluster_body<G, 32, 16>(P, rank, m, n, thr, S, cluster);
  } else if (bs <= 32 || m > 128) {
    if (m <= 128) svd_cluster_body<G, 16, 8>(P, rank, m, n, thr, S, cluster);
    else if (m <= 160) svd_cluster_body<G, 16, 10>(P, rank, m, n, thr, S, cluster);
    else if (m <= 192) svd_cluster_body<G, 16, 12>(P, rank, m, n, thr, S, cluster);
    else if (m <= 224) svd_cluster_body<G, 16, 14>(P, rank, m, n, thr, S, cluster);
    else svd_cluster_body<G, 16, 16>(P, rank, m, n, thr, S, cluster);
  } else {
    if (m <= 64) svd_cluster_body<G, 8, 8>(P, rank, m, n, thr, S, cluster);
    else if (m <= 128) svd_cluster_body<G, 8, 16>(P, rank, m, n, thr, S, cluster);
    else svd_cluster_body<G, 16, 16>(P, rank, m, n, thr, S, cluster);
  }
}
}  // namespace
