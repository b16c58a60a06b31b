// Block one-sided Jacobi on the FP64 tensor pipe (included by hq_svd.cu).
//
// The n columns of X (m x n, in the global work buffer: L2-resident) are
// grouped into blocks of 8.  A sweep is a round-robin tournament over the
// blocks; in every round each warp takes one pair of blocks (16 columns W):
//   1. G = W^T W (16 x 16) on DMMA, fresh from the columns (so every entry
//      carries a rounding error relative to |x_p| |x_q|, the scaled accuracy
//      one-sided Jacobi relies on);
//   2. if some pair of W is not yet orthogonal (|g_pq| > tol sqrt(g_pp g_qq)),
//      two-sided cyclic Jacobi on G with the rotations accumulated in V
//      (16 x 16) -- the same rotation formula and exclusion rules as the
//      scalar kernel (jacobi_tan / jacobi_cos); on a positive definite G the
//      two-sided iteration keeps that scaled accuracy (Demmel-Veselic);
//   3. W <- W V on DMMA.
// So the O(m n^2) work per sweep runs as 16-wide products on the tensor
// pipe and the CTA synchronizes once per tournament round (n/8 - 1 per
// sweep) instead of once per column pair round (n - 1).  The iteration stops
// after a sweep whose largest fresh off-diagonal |g|/sqrt(ab) was below
// 1e-7 (quadratic convergence, as in the scalar kernel).  Singular values
// are the final column norms; U_k as in svd_single.
// reference: svd + truncation_rank in core.py:250-253, dense.py:82-99
namespace {
constexpr int BJ_NT = 512, BJ_NW = BJ_NT / 32;
#ifndef HQ_BJ_INNER
#define HQ_BJ_INNER 1
#endif
constexpr int BJ_INNER = HQ_BJ_INNER;   // inner sweeps per task (the classic block method: one)

struct BjWarp {
  double G[16][17];
  double V[16][17];
  double c[8], s[8];
  double na[8], nb[8];   // rotated diagonal (a - t g, b + t g) of each pair
};
struct BjSmem {
  BjWarp w[BJ_NW];
  double nrm[MAX_N];
  int rotf[3];   // per-sweep flags, slot sweep % 3 (see svd_block_body)
  int cnt;
};

// positions of pair k in round r of the circle method on P = 2h positions
__device__ __forceinline__ void circle_pair(int r, int k, int P, int& p, int& q) {
  const int N = P - 1;
  if (k == 0) { p = r; q = N; }
  else { p = r + k; if (p >= N) p -= N; q = r - k; if (q < 0) q += N; }
  if (p > q) { const int x = p; p = q; q = x; }
}

// Jacobi task on blocks I, J (columns 8I.., 8J..; columns >= n are zero).
// Returns true when a fresh off-diagonal exceeded the quadratic stop level.
__device__ __noinline__ bool bj_task(double* __restrict__ X, int ld, int m, int n, int I, int J, double tol2,
                                     double tiny2, double thr2, BjWarp& W) {
  const int lane = threadIdx.x & 31;
  const int gq = lane >> 2, tq = lane & 3;
  // ---- 1. Gram on the tensor pipe.  k-steps cover rows 8u + 2tq + {0,1}
  // (the same row permutation for both operands, so the sum is the Gram):
  // one 16-byte load per block and lane per two k-steps.
  const int ca = 8 * I + gq, cb = 8 * J + gq;
  const bool va = ca < n, vb = cb < n;
  const double* xa = X + (size_t)(va ? ca : 0) * ld;
  const double* xb = X + (size_t)(vb ? cb : 0) * ld;
  double aa0 = 0.0, aa1 = 0.0, ab0 = 0.0, ab1 = 0.0, bb0 = 0.0, bb1 = 0.0;
  {
    constexpr int U = 8;   // row groups of 8 in flight (16 x 16-byte loads per lane)
    int r0 = 0;
    for (; r0 + 8 * U <= ld; r0 += 8 * U) {
      double2 fa[U], fb[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int rr = r0 + 8 * u + 2 * tq;
        fa[u] = va ? __ldcg(reinterpret_cast<const double2*>(xa + rr)) : make_double2(0.0, 0.0);
        fb[u] = vb ? __ldcg(reinterpret_cast<const double2*>(xb + rr)) : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        dmma884(aa0, aa1, fa[u].x, fa[u].x);
        dmma884(ab0, ab1, fa[u].x, fb[u].x);
        dmma884(bb0, bb1, fb[u].x, fb[u].x);
        dmma884(aa0, aa1, fa[u].y, fa[u].y);
        dmma884(ab0, ab1, fa[u].y, fb[u].y);
        dmma884(bb0, bb1, fb[u].y, fb[u].y);
      }
    }
    for (; r0 < ld; r0 += 8) {
      const int rr = r0 + 2 * tq;
      const bool in = rr < ld;   // ld even: rr + 1 < ld too
      const double2 fa = (va && in) ? __ldcg(reinterpret_cast<const double2*>(xa + rr)) : make_double2(0.0, 0.0);
      const double2 fb = (vb && in) ? __ldcg(reinterpret_cast<const double2*>(xb + rr)) : make_double2(0.0, 0.0);
      dmma884(aa0, aa1, fa.x, fa.x);
      dmma884(ab0, ab1, fa.x, fb.x);
      dmma884(bb0, bb1, fb.x, fb.x);
      dmma884(aa0, aa1, fa.y, fa.y);
      dmma884(ab0, ab1, fa.y, fb.y);
      dmma884(bb0, bb1, fb.y, fb.y);
    }
  }
  // lane holds D[gq][2tq + h]; G is symmetric: the upper triangle comes from
  // the products as computed, the lower is its mirror (bitwise symmetric)
  {
    const int i = gq, j0 = 2 * tq;
    W.G[i][j0] = aa0; W.G[i][j0 + 1] = aa1;
    W.G[i][8 + j0] = ab0; W.G[i][8 + j0 + 1] = ab1;
    W.G[8 + i][8 + j0] = bb0; W.G[8 + i][8 + j0 + 1] = bb1;
  }
  __syncwarp();
  for (int e = lane; e < 256; e += 32) {
    const int i = e >> 4, j = e & 15;
    if (i > j) W.G[i][j] = W.G[j][i];
  }
  __syncwarp();
  // ---- convergence test on the fresh Gram (same rules as jacobi_pair)
  bool need = false, sig = false;
  for (int e = lane; e < 256; e += 32) {
    const int p = e >> 4, q = e & 15;
    if (p >= q) continue;
    const double a = W.G[p][p], b = W.G[q][q], g = W.G[p][q];
    const bool work = !(a + b < thr2) && !(a < tiny2 && b < tiny2);
    if (work && g != 0.0 && g * g > tol2 * (a * b)) {
      need = true;
      if (g * g > QSTOP2 * (a * b)) sig = true;
    }
  }
  need = __any_sync(0xffffffffu, need);
  sig = __any_sync(0xffffffffu, sig);
  if (!need) return false;
  // ---- 2. two-sided Jacobi on G, V accumulates the rotations
  for (int e = lane; e < 256; e += 32) W.V[e >> 4][e & 15] = (e >> 4) == (e & 15) ? 1.0 : 0.0;
  __syncwarp();
  for (int sw = 0; sw < BJ_INNER; ++sw) {
    bool any_sweep = false;
    for (int r = 0; r < 15; ++r) {
      bool rot = false;
      if (lane < 8) {
        int p, q;
        circle_pair(r, lane, 16, p, q);
        const double a = W.G[p][p], b = W.G[q][q], g = W.G[p][q];
        const bool work = !(a + b < thr2) && !(a < tiny2 && b < tiny2);
        rot = work && g != 0.0 && g * g > tol2 * (a * b);
        double c = 1.0, s = 0.0;
        if (rot) {
          const double tt = jacobi_tan(a, b, g);
          c = jacobi_cos(tt);
          s = c * tt;
          W.na[lane] = fmax(a - tt * g, 0.0);
          W.nb[lane] = b + tt * g;
        }
        W.c[lane] = c; W.s[lane] = s;
      }
      if (!__any_sync(0xffffffffu, rot)) continue;   // warp-uniform
      any_sweep = true;
      __syncwarp();
      // columns p, q of G and V: (x_p, x_q) <- (c x_p - s x_q, s x_p + c x_q)
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int e = lane + 32 * u, i = e & 15, k = e >> 4;
        int p, q;
        circle_pair(r, k, 16, p, q);
        const double c = W.c[k], s = W.s[k];
        if (s != 0.0) {
          const double gp = W.G[i][p], gqv = W.G[i][q];
          W.G[i][p] = c * gp - s * gqv;
          W.G[i][q] = s * gp + c * gqv;
          const double vp = W.V[i][p], vq = W.V[i][q];
          W.V[i][p] = c * vp - s * vq;
          W.V[i][q] = s * vp + c * vq;
        }
      }
      __syncwarp();
      // rows p, q of G
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int e = lane + 32 * u, j = e & 15, k = e >> 4;
        int p, q;
        circle_pair(r, k, 16, p, q);
        const double c = W.c[k], s = W.s[k];
        if (s != 0.0) {
          const double gp = W.G[p][j], gqv = W.G[q][j];
          W.G[p][j] = c * gp - s * gqv;
          W.G[q][j] = s * gp + c * gqv;
        }
      }
      __syncwarp();
      // the rotated 2x2 block exactly: diag(a - t g, b + t g), zero coupling
      // (the cancellation-free update of jacobi_pair)
      if (lane < 8 && W.s[lane] != 0.0) {
        int p, q;
        circle_pair(r, lane, 16, p, q);
        W.G[p][p] = W.na[lane];
        W.G[q][q] = W.nb[lane];
        W.G[p][q] = 0.0;
        W.G[q][p] = 0.0;
      }
      __syncwarp();
    }
    if (!any_sweep) break;
  }
  // ---- 3. W <- W V on the tensor pipe, 8 rows at a time
  // B fragments: V[4s + tq][8h + gq] for k-steps s and output halves h
  double vb_[4][2];
#pragma unroll
  for (int s = 0; s < 4; ++s)
#pragma unroll
    for (int h = 0; h < 2; ++h) vb_[s][h] = W.V[4 * s + tq][8 * h + gq];
  // global column of local column c (-1: padding)
  auto gcol = [&](int c) { const int g = c < 8 ? 8 * I + c : 8 * J + c - 8; return g < n ? g : -1; };
  int ac[4];
#pragma unroll
  for (int s = 0; s < 4; ++s) ac[s] = gcol(4 * s + tq);
  int oc[2][2];
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int e = 0; e < 2; ++e) oc[h][e] = gcol(8 * h + 2 * tq + e);
  // 4 row tiles per step: their 16 loads per lane are in flight together
  // (rows are independent, so a step's loads precede its own stores only)
  constexpr int T4 = 4;
  for (int r0 = 0; r0 < m; r0 += 8 * T4) {
    double av[T4][4];
#pragma unroll
    for (int u = 0; u < T4; ++u) {
      const int i = r0 + 8 * u + gq;
      const bool in = i < m;
#pragma unroll
      for (int s = 0; s < 4; ++s) av[u][s] = (in && ac[s] >= 0) ? __ldcg(X + i + (size_t)ac[s] * ld) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < T4; ++u) {
      const int i = r0 + 8 * u + gq;
      double d[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
      for (int s = 0; s < 4; ++s)
#pragma unroll
        for (int h = 0; h < 2; ++h) dmma884(d[h][0], d[h][1], av[u][s], vb_[s][h]);
      if (i < m) {
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int e = 0; e < 2; ++e)
            if (oc[h][e] >= 0) X[i + (size_t)oc[h][e] * ld] = d[h][e];
      }
    }
  }
  __syncwarp();
  return sig;
}

// One problem on G CTAs (G = 1: plain launch; G > 1: a thread-block cluster).
// X lives in global memory (L2; loads bypass L1, __ldcg), so the CTAs of a
// cluster share it without DSMEM: the tasks of a round are spread over all
// G x 16 warps and the round ends with one cluster barrier (release /
// acquire at cluster scope orders the column updates).  Only the sweep's
// convergence flags travel through distributed shared memory.
template <int G>
__device__ __forceinline__ void bj_sync() {
  if constexpr (G == 1) __syncthreads();
  else cg::this_cluster().sync();
}

template <int G>
__device__ void svd_block_body(const hq_svd_prob& Pin, int* __restrict__ rank, const double* __restrict__ scal,
                               BjSmem& S) {
  const hq_svd_prob P = Pin;
  const int cr = G > 1 ? (int)cg::this_cluster().block_rank() : 0;
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  const int gw = cr * BJ_NW + wid;           // warp index over the cluster
  const int m = hq_dim(rank, P.m, P.m_ri);
  int n = hq_dim(rank, P.n, P.n_ri);
  if (P.xform) n = min(n, m);
  const double thr = P.eps_scale * (P.eps_slot >= 0 ? scal[P.eps_slot] : 1.0);
  if (cr == 0 && t == 0 && P.flag_ri >= 0 && (n > MAX_N || (P.n >= MAX_N && P.n_ri >= 0 && rank[P.n_ri] > P.n)))
    rank[P.flag_ri] = 1;
  n = min(n, MAX_N);
  if (m <= 0 || n <= 0) {
    if (cr == 0 && t == 0) rank[P.rank_ri] = 0;
    return;   // uniform over the cluster: no CTA waits at a barrier
  }
  // X in the work buffer, even leading dimension (16-byte aligned columns),
  // rows m..ld-1 zero
  const int ld = (m + 1) & ~1;
  double* X = P.work;
  for (int e = cr * BJ_NT + t; e < ld * n; e += G * BJ_NT) {
    const int i = e % ld, j = e / ld;
    // xform: X[i][j] = R[j][i] (1: j <= i, 2: all), R stored in c with leading dim ldc
    X[e] = P.xform ? ((i < m && (j <= i || P.xform == 2)) ? P.c[j + (size_t)i * P.ldc] : 0.0)
                   : (i < m ? P.c[i + (size_t)j * P.ldc] : 0.0);
  }
  if (t < 3) S.rotf[t] = 0;
  bj_sync<G>();
  const double tol = 4.0 * sqrt((double)m) * 2.220446049250313e-16;
  const double tol2 = tol * tol, thr2 = thr * thr, tiny2 = (1e-3 * thr) * (1e-3 * thr);
  const int nb = (n + 7) / 8, nbp = nb + (nb & 1), ntask = nbp / 2;
#ifdef HQ_DEBUG_SWEEPS
  int nsw = 0;
#endif
  for (int sweep = 0; sweep < MAX_SWEEPS; ++sweep) {
#ifdef HQ_DEBUG_SWEEPS
    nsw = sweep + 1;
#endif
    // slot sweep % 3 collects this sweep's flag; the next sweep's slot is
    // cleared now.  Three slots: a CTA that enters sweep s + 1 clears the
    // slot of sweep s - 1, which every CTA of the cluster finished reading
    // before the first barrier of sweep s (a CTA may still be reading the
    // flags of sweep s, so two slots would race and let the CTAs disagree
    // about termination)
    const int fs = sweep % 3;
    if (t == 0) S.rotf[(sweep + 1) % 3] = 0;
    for (int r = 0; r < nbp - 1; ++r) {
      for (int k = gw; k < ntask; k += G * BJ_NW) {
        int I, J;
        circle_pair(r, k, nbp, I, J);
        if (I >= nb) continue;   // both blocks are padding
        if (bj_task(X, ld, m, n, I, J, tol2, tiny2, thr2, S.w[wid]) && lane == 0) S.rotf[fs] = 1;
      }
      bj_sync<G>();
    }
    int any = S.rotf[fs];
    if constexpr (G > 1) {
      cg::cluster_group cl = cg::this_cluster();
#pragma unroll
      for (int c = 0; c < G; ++c) any |= *cl.map_shared_rank(&S.rotf[fs], c);
    }
    if (!any) break;
  }
#ifdef HQ_DEBUG_SWEEPS
  if (cr == 0 && t == 0 && P.flag_ri >= 0) rank[P.flag_ri + 1] = nsw;
#endif
  // singular values = exact column norms (every CTA computes all of them);
  // U_k sorted by descending sigma, each kept column written by one warp of
  // the cluster
  for (int j = wid; j < n; j += BJ_NW) {
    const double* xj = X + (size_t)j * ld;
    double v = 0.0;
    for (int i = lane; i < m; i += 32) {
      const double x = __ldcg(xj + i);
      v = fma(x, x, v);
    }
    v = sqrt(warp_sum(v));
    if (lane == 0) S.nrm[j] = v;
  }
  if (t == 0) S.cnt = 0;
  __syncthreads();
  for (int j = wid; j < n; j += BJ_NW) {
    const double sj = S.nrm[j];
    if (!(sj > thr)) continue;
    if (lane == 0) atomicAdd(&S.cnt, 1);
    if (j % G != cr) continue;
    int pos = 0;
    for (int o = lane; o < n; o += 32) {
      const double so = S.nrm[o];
      pos += (so > sj || (so == sj && o < j)) ? 1 : 0;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) pos += __shfl_xor_sync(0xffffffffu, pos, off);
    if (pos < P.cap) {
      const double inv = 1.0 / sj;
      const double* xj = X + (size_t)j * ld;
      for (int i = lane; i < m; i += 32) P.u[i + (size_t)pos * P.ldu] = __ldcg(xj + i) * inv;
    }
  }
  __syncthreads();
  if (cr == 0 && t == 0) {
    int kk = S.cnt;
    if (kk > P.cap) { if (P.flag_ri >= 0) rank[P.flag_ri] = 1; kk = P.cap; }
    rank[P.rank_ri] = kk;
  }
  // no CTA leaves while another may still read its flags
  if constexpr (G > 1) cg::this_cluster().sync();
}

template <int G>
__global__ void __launch_bounds__(BJ_NT, 1) svd_block_kernel(const hq_svd_prob* __restrict__ probs,
                                                            int* __restrict__ rank,
                                                            const double* __restrict__ scal) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  svd_block_body<G>(probs[blockIdx.x / G], rank, scal, *reinterpret_cast<BjSmem*>(smem_raw));
}
}  // namespace
