// One-sided block Jacobi on a thread-block cluster (included by hq_svd.cu).
// For truncation cores too large for one SM's shared memory (m*n > ~24K
// doubles, i.e. n >~ 155), the n columns of X are split into 2G blocks of bs
// columns; CTA c of a G-CTA cluster holds two blocks in its shared memory.
// A sweep = intra-block pairs (round 0) + the 2G-1 rounds of a block
// round-robin tournament (circle method): each round every CTA rotates all
// pairs between its two blocks, then the blocks move between CTAs through
// distributed shared memory (pull into staging buffers, cluster barrier,
// local copy).  Columns never leave the cluster's SMs until U_k is written.
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

namespace {
constexpr int CNT = 512, CNW = CNT / 32;
constexpr int C_MAX_BS = 64;          // max columns per block
constexpr int C_SMEM_DOUBLES = 22528; // 176 KB: 4 block buffers (2 work + 2 staging)

struct CSmem {
  double buf[C_SMEM_DOUBLES];
  double nrm[4][C_MAX_BS];   // carried squared norms of the four block buffers
  int col[4][C_MAX_BS];      // global column index held in each buffer slot (-1: pad)
  double sig_all[1024];
  int rot;
  int done;
  int cnt;
};

// rotate pair (x, y) of columns held in smem (ld even), group of LP lanes
template <int LP>
__device__ __forceinline__ bool rotate_pair(double* cx, double* cy, double& a, double& b, int ld,
                                            double tol, double tiny2, double thr2, int gl, bool act) {
  constexpr int E = 16;
  double xp[E], xq[E];
  const bool work = act && !(a + b < thr2) && !(a < tiny2 && b < tiny2);
  double g0 = 0.0, g1 = 0.0;
#pragma unroll
  for (int e = 0; e < E / 2; ++e) {
    const int i = 2 * gl + 2 * LP * e;
    double2 vp = make_double2(0.0, 0.0), vq = make_double2(0.0, 0.0);
    if (work && i < ld) {
      vp = *reinterpret_cast<const double2*>(cx + i);
      vq = *reinterpret_cast<const double2*>(cy + i);
    }
    xp[2 * e] = vp.x; xp[2 * e + 1] = vp.y;
    xq[2 * e] = vq.x; xq[2 * e + 1] = vq.y;
    g0 = fma(vp.x, vq.x, g0);
    g1 = fma(vp.y, vq.y, g1);
  }
  double g = g0 + g1;
#pragma unroll
  for (int o = LP / 2; o > 0; o >>= 1) g += __shfl_xor_sync(0xffffffffu, g, o);
  const bool rot = work && g != 0.0 && g * g > (tol * tol) * (a * b);
  if (rot) {
    // zeta = (b - a) / 2g in single precision on exponent-normalized operands
    int eg;
    frexp(g, &eg);
    const double num = ldexp(b - a, -eg), den = ldexp(2.0 * g, -eg);   // |den| in [1, 2)
    double tt;
    if (fabs(num) < 1e18) {
      const float zf = __fdividef((float)num, (float)den);
      tt = (double)(copysignf(1.0f, zf) / (fabsf(zf) + sqrtf(fmaf(zf, zf, 1.0f))));
    } else {
      tt = 0.5 * den / num;
    }
    const double c = rsqrt(1.0 + tt * tt), sn = c * tt;
#pragma unroll
    for (int e = 0; e < E / 2; ++e) {
      const int i = 2 * gl + 2 * LP * e;
      if (i < ld) {
        *reinterpret_cast<double2*>(cx + i) =
            make_double2(c * xp[2 * e] - sn * xq[2 * e], c * xp[2 * e + 1] - sn * xq[2 * e + 1]);
        *reinterpret_cast<double2*>(cy + i) =
            make_double2(sn * xp[2 * e] + c * xq[2 * e], sn * xp[2 * e + 1] + c * xq[2 * e + 1]);
      }
    }
    a = fmax(a - tt * g, 0.0);
    b = b + tt * g;
  }
  return rot;
}

// block owner map of the circle tournament: position -> (cta, slot)
// top row: positions 0..G-1 are slot 0 of CTA c; bottom row: slot 1 of CTA
// c holds position 2G-1-c.  Each round, position 0 stays, the others rotate.
__device__ __forceinline__ int circ_next(int pos, int G) {
  // block at tournament position pos moves to this position next round
  const int P = 2 * G;
  if (pos == 0) return 0;
  return pos == P - 1 ? 1 : pos + 1;
}

template <int G, int LP>
__global__ void __launch_bounds__(CNT, 1) svd_cluster_kernel(const hq_svd_prob* __restrict__ probs,
                                                             int* __restrict__ rank,
                                                             const double* __restrict__ scal) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  CSmem& S = *reinterpret_cast<CSmem*>(smem_raw);
  cg::cluster_group cluster = cg::this_cluster();
  const int cr = (int)cluster.block_rank();
  const hq_svd_prob P = probs[blockIdx.x / G];
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  constexpr int GPW = 32 / LP;
  const int grp = wid * GPW + lane / LP, gl = lane % LP, ngroups = CNW * GPW;
  const int m = hq_dim(rank, P.m, P.m_ri);
  int n = hq_dim(rank, P.n, P.n_ri);
  if (P.xform) n = min(n, m);
  n = min(n, 1024);
  const double thr = P.eps_scale * (P.eps_slot >= 0 ? scal[P.eps_slot] : 1.0);
  if (m <= 0 || n <= 0) {
    if (cr == 0 && t == 0) rank[P.rank_ri] = 0;
    return;
  }
  const int ld = (m + 1) & ~1;
  const int bs = (n + 2 * G - 1) / (2 * G);
  if (4 * bs * ld > C_SMEM_DOUBLES || bs > C_MAX_BS || G * 2 * bs > 1024) {
    // the plan picked a cluster too small for this run-time size
    if (cr == 0 && t == 0) {
      if (P.flag_ri >= 0) rank[P.flag_ri] = 1;
      rank[P.rank_ri] = 0;
    }
    return;
  }
  // buffers: 0,1 = working slots; 2,3 = staging
  double* B[4];
  for (int k = 0; k < 4; ++k) B[k] = S.buf + (size_t)k * bs * ld;
  // ---- initial load: CTA cr holds positions cr (slot 0) and 2G-1-cr (slot 1)
  for (int slot = 0; slot < 2; ++slot) {
    const int pos = slot == 0 ? cr : 2 * G - 1 - cr;
    for (int jj = 0; jj < bs; ++jj) {
      const int j = pos * bs + jj;
      double* dst = B[slot] + (size_t)jj * ld;
      for (int i = t; i < ld; i += CNT) {
        double v = 0.0;
        if (j < n && i < m) v = P.xform ? (j <= i ? P.c[j + (size_t)i * P.ldc] : 0.0)
                                        : P.c[i + (size_t)j * P.ldc];
        dst[i] = v;
      }
      if (t == 0) S.col[slot][jj] = j < n ? j : -1;
    }
  }
  __syncthreads();
  const double tol = 4.0 * sqrt((double)m) * 2.220446049250313e-16;
  const double tiny2 = (1e-3 * thr) * (1e-3 * thr), thr2 = thr * thr;
  for (int sweep = 0; sweep < MAX_SWEEPS; ++sweep) {
    // squared norms of the two working blocks
    for (int j = wid; j < 2 * bs; j += CNW) {
      const double* x = B[j / bs] + (size_t)(j % bs) * ld;
      double v = 0.0;
      for (int i = lane; i < ld; i += 32) v = fma(x[i], x[i], v);
      v = warp_sum(v);
      if (lane == 0) S.nrm[j / bs][j % bs] = v;
    }
    if (t == 0) S.rot = 0;
    __syncthreads();
    // intra-block pairs of both working blocks (round robin inside each block)
    {
      const int npb = bs + (bs & 1), N = npb - 1;
      for (int r = 0; r < N; ++r) {
        for (int g0 = 0; g0 < 2 * (npb / 2); g0 += ngroups) {
          const int gi = g0 + grp;
          const int blk = gi / (npb / 2), pi = gi % (npb / 2);
          int p = 0, q = 0;
          bool act = gi < 2 * (npb / 2);
          if (act) {
            pair_of(r, pi, N, p, q);
            act = q < bs && S.col[blk][p] >= 0 && S.col[blk][q] >= 0;
          }
          double a = act ? S.nrm[blk][p] : 0.0, b = act ? S.nrm[blk][q] : 0.0;
          const bool rr = rotate_pair<LP>(B[blk & 1] + (size_t)p * ld, B[blk & 1] + (size_t)q * ld, a, b,
                                          ld, tol, tiny2, thr2, gl, act);
          if (rr && gl == 0) { S.nrm[blk][p] = a; S.nrm[blk][q] = b; S.rot = 1; }
        }
        __syncthreads();
      }
    }
    // 2G-1 tournament rounds of inter-block pairs
    for (int round = 0; round < 2 * G - 1; ++round) {
      for (int r = 0; r < bs; ++r) {
        for (int g0 = 0; g0 < bs; g0 += ngroups) {
          const int i = g0 + grp;
          const int j = (i + r) % bs;
          bool act = i < bs && S.col[0][i] >= 0 && S.col[1][j] >= 0;
          double a = act ? S.nrm[0][i] : 0.0, b = act ? S.nrm[1][j] : 0.0;
          const bool rr = rotate_pair<LP>(B[0] + (size_t)i * ld, B[1] + (size_t)j * ld, a, b, ld, tol, tiny2,
                                          thr2, gl, act);
          if (rr && gl == 0) { S.nrm[0][i] = a; S.nrm[1][j] = b; S.rot = 1; }
        }
        __syncthreads();
      }
      if (round == 2 * G - 2) break;
      // move blocks: the block at position p goes to circ_next(p); pull the
      // blocks that land in my two slots from their current owners
      cluster.sync();
      for (int slot = 0; slot < 2; ++slot) {
        const int mypos = slot == 0 ? cr : 2 * G - 1 - cr;
        // source position: the one whose circ_next == mypos
        int src = mypos;
        for (int p = 0; p < 2 * G; ++p)
          if (circ_next(p, G) == mypos) { src = p; break; }
        const int scta = src < G ? src : 2 * G - 1 - src;
        const int sslot = src < G ? 0 : 1;
        CSmem* R = cluster.map_shared_rank(&S, scta);
        const double* sb = R->buf + (size_t)sslot * bs * ld;
        double* db = B[2 + slot];
        for (int e = t; e < bs * ld; e += CNT) db[e] = sb[e];
        for (int jj = t; jj < bs; jj += CNT) {
          S.nrm[2 + slot][jj] = R->nrm[sslot][jj];
          S.col[2 + slot][jj] = R->col[sslot][jj];
        }
      }
      cluster.sync();
      for (int e = t; e < 2 * bs * ld; e += CNT) B[0][e] = B[2][e];   // buffers 0,1 contiguous
      for (int jj = t; jj < 2 * bs; jj += CNT) {
        S.nrm[jj / bs][jj % bs] = S.nrm[2 + jj / bs][jj % bs];
        S.col[jj / bs][jj % bs] = S.col[2 + jj / bs][jj % bs];
      }
      __syncthreads();
    }
    // cluster-wide convergence test
    cluster.sync();
    if (t == 0) {
      int any = 0;
      for (int c = 0; c < G; ++c) any |= cluster.map_shared_rank(&S, c)->rot;
      S.done = any ? 0 : 1;
    }
    cluster.sync();
    if (S.done) break;
    // the blocks are now at shifted positions; restart the tournament from
    // the current placement (any placement is a valid starting position)
  }
  // ---- singular values, global order, output U_k
  for (int j = wid; j < 2 * bs; j += CNW) {
    const double* x = B[j / bs] + (size_t)(j % bs) * ld;
    double v = 0.0;
    for (int i = lane; i < ld; i += 32) v = fma(x[i], x[i], v);
    v = sqrt(warp_sum(v));
    if (lane == 0) S.nrm[j / bs][j % bs] = S.col[j / bs][j % bs] >= 0 ? v : -1.0;
  }
  cluster.sync();
  // gather (column id, sigma) of every slot of every CTA
  for (int e = t; e < G * 2 * bs; e += CNT) {
    const int c = e / (2 * bs), k = e % (2 * bs);
    CSmem* R = cluster.map_shared_rank(&S, c);
    S.sig_all[e] = R->nrm[k / bs][k % bs];
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
      const double* x = B[k / bs] + (size_t)(k % bs) * ld;
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
}  // namespace
