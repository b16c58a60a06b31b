// Hestenes one-sided Jacobi (included by hq_svd.cu).
// Per round of the round-robin schedule: (A) one warp per pair computes the
// column dot product g, (B) one thread per pair turns (a, b, g) into the
// rotation (scalar work done once per pair, not 32x), (C) one warp per pair
// rotates the two columns and updates the carried squared norms.
namespace {
constexpr int NT = 512, NW = NT / 32;
constexpr int SMEM_DOUBLES = 24576;  // 192 KB: X staged in smem when m*n fits
constexpr int MAX_N = 1024;
constexpr int MAX_SWEEPS = 40;
// Sweep stop: a sweep whose largest rotated pair had |g| / sqrt(a b) below
// QSTOP ends the iteration -- by the quadratic convergence of cyclic Jacobi
// the next sweep's pairs would be O(QSTOP^2) ~ 1e-14, the rotation tolerance
// itself, so that sweep only verifies (measured on the truncation cores: 9 %
// fewer rounds, orthogonality of U unchanged).
constexpr double QSTOP2 = 1e-14;

// cs is last: the small-core kernel allocates only a prefix of it
struct SvdSmem {
  double nrm[MAX_N];
  short act[MAX_N];   // active columns (compaction of negligible ones)
  int nact;
  double g[MAX_N / 2];
  double rc[MAX_N / 2];
  double rs[MAX_N / 2];
  double rt[MAX_N / 2];
  double2 trash[32];  // sink for the stores of rows past the column end
  int rot;
  int cnt;
  alignas(16) double cs[SMEM_DOUBLES];   // staged X, 16-byte aligned columns
};

__device__ __forceinline__ void pair_of(int r, int pi, int N, int& p, int& q) {
  if (pi == 0) { p = r; q = N; }
  else { p = (r + pi) % N; q = (r - pi + N) % N; }
  if (p > q) { const int x = p; p = q; q = x; }
}

__device__ __forceinline__ double rcp_approx(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  return r;
}
__device__ __forceinline__ double rsqrt_approx(double x) {
  double r;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  return r;
}

// Tangent t of the Jacobi rotation for the pair with squared norms a, b and
// inner product g (g != 0): t = sign(z) / (|z| + sqrt(1 + z^2)), z = (b-a)/2g.
// Any t gives an exactly orthogonal rotation once c = (1+t^2)^(-1/2) is
// accurate, so t is formed from the hardware reciprocal / reciprocal-sqrt
// approximations (~2^-22 relative: at most one extra sweep); only c is
// computed to full FP64 accuracy by the caller.
// c = (1 + t^2)^(-1/2) to full FP64 accuracy: hardware reciprocal square
// root (~2^-22) refined by two Newton steps (quadratic: ~2^-44, ~2^-88),
// shorter than the library rsqrt's generic path
__device__ __forceinline__ double jacobi_cos(double tt) {
  const double w = fma(tt, tt, 1.0);
  double y = rsqrt_approx(w);
  const double hw = 0.5 * w;
  y = y * fma(-hw * y, y, 1.5);
  y = y * fma(-hw * y, y, 1.5);
  return y;
}

__device__ __forceinline__ double jacobi_tan(double a, double b, double g) {
  const double d = b - a;
  const double h = fabs(d) * (0.5 * rcp_approx(fabs(g)));
  const double w = fma(h, h, 1.0);
  const double t = h < 1e150 ? rcp_approx(fma(w, rsqrt_approx(w), h)) : 0.5 * rcp_approx(h);
  return ((d >= 0.0) == (g > 0.0)) ? t : -t;
}

// One pair update by a group of LP lanes; lane gl owns rows 2gl + 2LP e + {0,1}
// (e < E/2) of both columns, so a group moves 16 B x LP contiguous bytes per
// access (conflict-free 128-bit shared memory traffic).  XREG: column x lives
// in the registers xp across calls (only y streams through shared memory).
// Rows past the column end read row 0 (masked) and store into a sink, so the
// body is branch-free apart from the rotation itself.
template <int LP, int E, bool XREG>
__device__ __forceinline__ int jacobi_pair(double (&xp)[E], double* cx, double* cy, double& a, double& b,
                                            int ld, double tol2, double tiny2, double thr2, int gl, bool act,
                                            double2* trash) {
  const bool work = act && !(a + b < thr2) && !(a < tiny2 && b < tiny2);
  double xq[E];
  double g0 = 0.0, g1 = 0.0, g2 = 0.0, g3 = 0.0;
#pragma unroll
  for (int e = 0; e < E / 2; ++e) {
    const int i = 2 * gl + 2 * LP * e;
    const bool in = work && i < ld;
    const int ii = in ? i : 0;
    const double2 vq = *reinterpret_cast<const double2*>(cy + ii);
    if (!XREG) {
      const double2 vp = *reinterpret_cast<const double2*>(cx + ii);
      xp[2 * e] = in ? vp.x : 0.0;
      xp[2 * e + 1] = in ? vp.y : 0.0;
    }
    xq[2 * e] = in ? vq.x : 0.0;
    xq[2 * e + 1] = in ? vq.y : 0.0;
    if (e & 1) {
      g2 = fma(xp[2 * e], xq[2 * e], g2);
      g3 = fma(xp[2 * e + 1], xq[2 * e + 1], g3);
    } else {
      g0 = fma(xp[2 * e], xq[2 * e], g0);
      g1 = fma(xp[2 * e + 1], xq[2 * e + 1], g1);
    }
  }
  double g = (g0 + g1) + (g2 + g3);
#pragma unroll
  for (int o = LP / 2; o > 0; o >>= 1) g += __shfl_xor_sync(0xffffffffu, g, o);
  const bool rot = work && g != 0.0 && g * g > tol2 * (a * b);
  const int code = rot ? (g * g > QSTOP2 * (a * b) ? 2 : 1) : 0;
  if (rot) {
    const double tt = jacobi_tan(a, b, g);
    const double c = jacobi_cos(tt), sn = c * tt;
    double2* sink = trash + (threadIdx.x & 31);
#pragma unroll
    for (int e = 0; e < E / 2; ++e) {
      const int i = 2 * gl + 2 * LP * e;
      const double x0 = xp[2 * e], x1 = xp[2 * e + 1], y0 = xq[2 * e], y1 = xq[2 * e + 1];
      const double2 nx = make_double2(c * x0 - sn * y0, c * x1 - sn * y1);
      const double2 ny = make_double2(sn * x0 + c * y0, sn * x1 + c * y1);
      if (XREG) {
        xp[2 * e] = nx.x;
        xp[2 * e + 1] = nx.y;
      } else {
        *(i < ld ? reinterpret_cast<double2*>(cx + i) : sink) = nx;
      }
      *(i < ld ? reinterpret_cast<double2*>(cy + i) : sink) = ny;
    }
    a = fmax(a - tt * g, 0.0);
    b = b + tt * g;
  }
  return code;
}

// Stable compaction of the active column list (warp 0): columns whose squared
// norm fell below tiny2 leave the rotation set.
__device__ __forceinline__ void compact_active(short* act, int& nact_out, const double* nrm, int nact,
                                               double tiny2) {
  const int lane = threadIdx.x & 31;
  int k = 0;
  for (int j0 = 0; j0 < nact; j0 += 32) {
    const int jj = j0 + lane;
    const int j = jj < nact ? act[jj] : 0;
    const bool keep = jj < nact && !(nrm[j] < tiny2);
    const unsigned bal = __ballot_sync(0xffffffffu, keep);
    __syncwarp();
    if (keep) act[k + __popc(bal & ((1u << lane) - 1u))] = (short)j;
    k += __popc(bal);
    __syncwarp();
  }
  if (lane == 0) nact_out = k;
}

// One-sided Jacobi with each pair owned by a group of LP lanes holding both
// columns in registers (E = rows per lane per column): one smem read and one
// smem write of each column per round, dot product reduced with log2(LP)
// shuffles, the rotation parameters computed by the group.  Warps without a
// pair in a round skip straight to the barrier (they would otherwise steal
// issue slots from the latency-bound active warps).
template <int LP, bool SMEM, int E, int NTH = 512>
__device__ int jacobi_groups(double* Xg, int ld, int m, int n, double tol, double tiny2, double thr,
                             SvdSmem& S) {
  // SMEM: index the staged copy through S.cs so the compiler emits LDS/STS
  double* X = SMEM ? S.cs : Xg;
  constexpr int GPW = 32 / LP, NT = NTH, NW = NTH / 32;   // shadow the 512-thread defaults
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  const int grp = wid * GPW + lane / LP, gl = lane % LP;
  const int ngroups = NW * GPW;
  const double tol2 = tol * tol, thr2 = thr * thr;
  for (int j = t; j < n; j += NT) S.act[j] = (short)j;
  if (t == 0) S.nact = n;
  __syncthreads();
  int sweep = 0;
  for (; sweep < MAX_SWEEPS; ++sweep) {
    const int nact0 = S.nact;
    for (int jj = wid; jj < nact0; jj += NW) {
      const int j = S.act[jj];
      const double* xj = X + (size_t)j * ld;
      double v = 0.0;
      for (int i = lane; i < m; i += 32) v = fma(xj[i], xj[i], v);
      v = warp_sum(v);
      if (lane == 0) S.nrm[j] = v;
    }
    __syncthreads();
    // after the first sweep, columns far below the threshold (norm < 1e-3 thr)
    // leave the rotation set: they are dropped by the truncation and moving
    // them changes the kept columns by less than that
    if (sweep >= 1 && wid == 0) compact_active(S.act, S.nact, S.nrm, nact0, tiny2);
    if (t == 0) S.rot = 0;
    __syncthreads();
    const int nact = S.nact;
    const int npair = (nact + 1) / 2, N = 2 * npair - 1;
    if (N <= 0) { ++sweep; break; }
    for (int r = 0; r < N; ++r) {
      for (int pi0 = 0; pi0 < npair; pi0 += ngroups) {
        if (pi0 + wid * GPW >= npair) break;  // warp-uniform
        const int pi = pi0 + grp;
        int p = 0, q = n;
        if (pi < npair) {
          // round-robin (circle) pair pi of round r
          int pp = r, qq = N;
          if (pi != 0) {
            pp = r + pi; if (pp >= N) pp -= N;
            qq = r - pi; if (qq < 0) qq += N;
          }
          if (pp < nact && qq < nact) {
            p = S.act[pp]; q = S.act[qq];
            if (p > q) { const int x = p; p = q; q = x; }
          }
        }
        const bool act = q < n;
        double a = 0.0, b = 0.0;
        if (act) { a = S.nrm[p]; b = S.nrm[q]; }
        if (SMEM) {
          double xp[E];
          double* cp = X + (size_t)p * ld;
          const int rr = jacobi_pair<LP, E, false>(xp, cp, act ? X + (size_t)q * ld : cp, a, b, ld, tol2, tiny2,
                                                   thr2, gl, act, S.trash);
          if (rr && gl == 0) {
            S.nrm[p] = a;
            S.nrm[q] = b;
            if (rr > 1) S.rot = 1;
          }
        } else {
          const bool work = act && !(a + b < thr2) && !(a < tiny2 && b < tiny2);
          double xp[E], xq[E];
          double g0 = 0.0, g1 = 0.0, g2 = 0.0, g3 = 0.0;
          double* cp = X + (size_t)p * ld;
          double* cq = X + (size_t)(work ? q : p) * ld;
#pragma unroll
          for (int e = 0; e < E; ++e) {
            const int i = gl + e * LP;
            xp[e] = (work && i < m) ? cp[i] : 0.0;
            xq[e] = (work && i < m) ? cq[i] : 0.0;
          }
#pragma unroll
          for (int e = 0; e < E; e += 4) {
            g0 = fma(xp[e], xq[e], g0);
            g1 = fma(xp[e + 1], xq[e + 1], g1);
            g2 = fma(xp[e + 2], xq[e + 2], g2);
            g3 = fma(xp[e + 3], xq[e + 3], g3);
          }
          double g = (g0 + g1) + (g2 + g3);
#pragma unroll
          for (int o = LP / 2; o > 0; o >>= 1) g += __shfl_xor_sync(0xffffffffu, g, o);
          const bool rot = work && g != 0.0 && g * g > tol2 * (a * b);
          if (rot) {
            const double tt = jacobi_tan(a, b, g);
            const double c = jacobi_cos(tt), sn = c * tt;
#pragma unroll
            for (int e = 0; e < E; ++e) {
              const int i = gl + e * LP;
              if (i < m) {
                const double x = xp[e], y = xq[e];
                cp[i] = c * x - sn * y;
                cq[i] = sn * x + c * y;
              }
            }
            if (gl == 0) {
              S.nrm[p] = fmax(a - tt * g, 0.0);
              S.nrm[q] = b + tt * g;
              if (g * g > QSTOP2 * (a * b)) S.rot = 1;
            }
          }
        }
      }
      __syncthreads();
    }
    if (S.rot == 0) { ++sweep; break; }
    __syncthreads();
  }
  return sweep;
}


// NTH threads; cap: doubles of S.cs the launch allocated
template <int NTH = 512>
__device__ __noinline__ void svd_single(const hq_svd_prob& Pin, int* __restrict__ rank,
                                        const double* __restrict__ scal, SvdSmem& S, int cap = SMEM_DOUBLES) {
  constexpr int NT = NTH, NW = NTH / 32;   // shadow the 512-thread defaults
  const hq_svd_prob P = Pin;
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  const int m = hq_dim(rank, P.m, P.m_ri);
  int n = hq_dim(rank, P.n, P.n_ri);
  if (P.xform) n = min(n, m);
  const double thr = P.eps_scale * (P.eps_slot >= 0 ? scal[P.eps_slot] : 1.0);
  if (t == 0 && P.flag_ri >= 0 && (n > MAX_N || (P.n >= MAX_N && P.n_ri >= 0 && rank[P.n_ri] > P.n)))
    rank[P.flag_ri] = 1;
  n = min(n, MAX_N);
  if (m <= 0 || n <= 0) {
    if (t == 0) rank[P.rank_ri] = 0;
    return;
  }
  const int lds = (m + 1) & ~1;  // even leading dim: 16 B aligned columns for double2
  const bool staged = (size_t)lds * n <= (size_t)cap;
  double* X;
  int ld;
  if (staged) { X = S.cs; ld = lds; }
  else if (P.xform) { X = P.work; ld = m; }
  else { X = P.c; ld = P.ldc; }
  if (P.xform) {
    // X[i][j] = R[j][i] (xform 1: j <= i, 2: all), R stored in c with leading dim ldc
    for (int e = t; e < m * n; e += NT) {
      const int i = e % m, j = e / m;
      X[i + (size_t)j * ld] = (j <= i || P.xform == 2) ? P.c[j + (size_t)i * P.ldc] : 0.0;
    }
  } else if (staged) {
    for (int e = t; e < m * n; e += NT) X[e % m + (size_t)(e / m) * ld] = P.c[e % m + (size_t)(e / m) * P.ldc];
  }
  if (staged && lds != m)
    for (int j = t; j < n; j += NT) X[m + (size_t)j * ld] = 0.0;
  __syncthreads();
  const double tol = 4.0 * sqrt((double)m) * 2.220446049250313e-16;
  const double tiny2 = (1e-3 * thr) * (1e-3 * thr);
  const int np = n + (n & 1), N = np - 1, npair = np / 2;
#pragma nv_diag_suppress 550
  int nsweeps = 0;
#pragma nv_diag_default 550
  if (m <= 512) {
    // register-cached path: a group of LP lanes owns a pair (E <= 16 rows per lane)
    if (staged) {
      // lane-group shape: as many lanes per pair as one pass of groups allows
      // (shorter per-pair dependency chains), enough rows per lane for m
      const int np0 = (n + 1) / 2;
      if (np0 <= NW || m > 256) {
        if (m <= 128) nsweeps = jacobi_groups<32, true, 4, NTH>(X, ld, m, n, tol, tiny2, thr, S);
        else if (m <= 256) nsweeps = jacobi_groups<32, true, 8, NTH>(X, ld, m, n, tol, tiny2, thr, S);
        else nsweeps = jacobi_groups<32, true, 16, NTH>(X, ld, m, n, tol, tiny2, thr, S);
      } else if (np0 <= 2 * NW || m > 128) {
        if (m <= 128) nsweeps = jacobi_groups<16, true, 8, NTH>(X, ld, m, n, tol, tiny2, thr, S);
        else nsweeps = jacobi_groups<16, true, 16, NTH>(X, ld, m, n, tol, tiny2, thr, S);
      } else {
        if (m <= 64) nsweeps = jacobi_groups<8, true, 8, NTH>(X, ld, m, n, tol, tiny2, thr, S);
        else if (m <= 128) nsweeps = jacobi_groups<8, true, 16, NTH>(X, ld, m, n, tol, tiny2, thr, S);
        else nsweeps = jacobi_groups<16, true, 16, NTH>(X, ld, m, n, tol, tiny2, thr, S);
      }
    } else {
      if (m <= 128) nsweeps = jacobi_groups<8, false, 16, NTH>(X, ld, m, n, tol, tiny2, thr, S);
      else if (m <= 256) nsweeps = jacobi_groups<16, false, 16, NTH>(X, ld, m, n, tol, tiny2, thr, S);
      else nsweeps = jacobi_groups<32, false, 16, NTH>(X, ld, m, n, tol, tiny2, thr, S);
    }
  }
  for (int sweep = 0; sweep < MAX_SWEEPS && N > 0 && !(m <= 512); ++sweep) {
    nsweeps = sweep + 1;
    for (int j = wid; j < n; j += NW) {
      const double* xj = X + (size_t)j * ld;
      double v = 0.0;
      for (int i = lane; i < m; i += 32) v = fma(xj[i], xj[i], v);
      v = warp_sum(v);
      if (lane == 0) S.nrm[j] = v;
    }
    if (t == 0) S.rot = 0;
    __syncthreads();
    for (int r = 0; r < N; ++r) {
      // (A) dot products
      for (int pi = wid; pi < npair; pi += NW) {
        int p, q;
        pair_of(r, pi, N, p, q);
        double g = 0.0;
        if (q < n && !(S.nrm[p] < tiny2 && S.nrm[q] < tiny2)) {
          const double* xp = X + (size_t)p * ld;
          const double* xq = X + (size_t)q * ld;
          for (int i = lane; i < m; i += 32) g = fma(xp[i], xq[i], g);
          g = warp_sum(g);
        }
        if (lane == 0) S.g[pi] = g;
      }
      __syncthreads();
      // (B) rotation parameters, one thread per pair
      for (int pi = t; pi < npair; pi += NT) {
        int p, q;
        pair_of(r, pi, N, p, q);
        double c = 1.0, sn = 0.0, tt = 0.0;
        const double g = S.g[pi];
        if (q < n && g != 0.0) {
          const double a = S.nrm[p], b = S.nrm[q];
          if (fabs(g) > tol * sqrt(a * b)) {
            const double zeta = (b - a) / (2.0 * g);
            tt = fabs(zeta) > 1e150 ? 0.5 / zeta
                                    : (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
            c = rsqrt(1.0 + tt * tt);
            sn = c * tt;
            S.nrm[p] = fmax(a - tt * g, 0.0);
            S.nrm[q] = b + tt * g;
            if (g * g > QSTOP2 * (a * b)) S.rot = 1;
          }
        }
        S.rc[pi] = c; S.rs[pi] = sn; S.rt[pi] = tt;
      }
      __syncthreads();
      // (C) rotations
      for (int pi = wid; pi < npair; pi += NW) {
        if (S.rt[pi] == 0.0) continue;
        int p, q;
        pair_of(r, pi, N, p, q);
        const double c = S.rc[pi], sn = S.rs[pi];
        double* xp = X + (size_t)p * ld;
        double* xq = X + (size_t)q * ld;
        for (int i = lane; i < m; i += 32) {
          const double x = xp[i], y = xq[i];
          xp[i] = c * x - sn * y;
          xq[i] = sn * x + c * y;
        }
      }
      __syncthreads();
    }
    if (S.rot == 0) break;
    __syncthreads();
  }
  // singular values = exact column norms
  for (int j = wid; j < n; j += NW) {
    const double* xj = X + (size_t)j * ld;
    double v = 0.0;
    for (int i = lane; i < m; i += 32) v = fma(xj[i], xj[i], v);
    v = sqrt(warp_sum(v));
    if (lane == 0) S.nrm[j] = v;
  }
  if (t == 0) S.cnt = 0;
  __syncthreads();
  for (int j = wid; j < n; j += NW) {
    const double sj = S.nrm[j];
    if (!(sj > thr)) continue;
    int pos = 0;
    for (int o = lane; o < n; o += 32) {
      const double so = S.nrm[o];
      pos += (so > sj || (so == sj && o < j)) ? 1 : 0;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) pos += __shfl_xor_sync(0xffffffffu, pos, off);
    if (lane == 0) atomicAdd(&S.cnt, 1);
    if (pos < P.cap) {
      const double inv = 1.0 / sj;
      const double* xj = X + (size_t)j * ld;
      for (int i = lane; i < m; i += 32) P.u[i + (size_t)pos * P.ldu] = xj[i] * inv;
    }
  }
  __syncthreads();
  if (t == 0) {
    int kk = S.cnt;
    if (kk > P.cap) { if (P.flag_ri >= 0) rank[P.flag_ri] = 1; kk = P.cap; }
    rank[P.rank_ri] = kk;
#ifdef HQ_DEBUG_SWEEPS
    if (P.flag_ri >= 0) rank[P.flag_ri + 1] = nsweeps;
#endif
  }
  (void)nsweeps;   // read by the HQ_DEBUG_SWEEPS build only
}

// Small cores, many per launch: 128-thread CTAs with only as much staging
// memory as the launch's largest core needs, so several problems share an SM
// (the round-robin rounds are latency chains; co-resident problems fill them).
constexpr int SMALL_NT = 128;
__global__ void __launch_bounds__(SMALL_NT) svd_small_kernel(const hq_svd_prob* __restrict__ probs,
                                                             int* __restrict__ rank,
                                                             const double* __restrict__ scal, int cap) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  svd_single<SMALL_NT>(probs[blockIdx.x], rank, scal, *reinterpret_cast<SvdSmem*>(smem_raw), cap);
}

__global__ void __launch_bounds__(NT, 1) svd_kernel(const hq_svd_prob* __restrict__ probs,
                                                    int* __restrict__ rank,
                                                    const double* __restrict__ scal) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  svd_single(probs[blockIdx.x], rank, scal, *reinterpret_cast<SvdSmem*>(smem_raw));
}
}  // namespace
