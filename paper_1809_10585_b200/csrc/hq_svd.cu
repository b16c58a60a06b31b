// One-sided (Hestenes) Jacobi SVD for the truncation cores, and the power
// iteration step for ||A||_2.
//   svd + truncation_rank : reference core.py:250-253, dense.py:82-99
//   power step            : reference dense.py:102-141, arith.py:293-298
// Jacobi orthogonalizes the columns of C (m x n) with a round-robin pair
// schedule (n'/2 independent rotations per round, one warp per pair); the
// converged column norms are the singular values and the normalized columns
// the left singular vectors.  Only U_k is produced: the caller forms the
// right factor as U_k^T-projections (no division by sigma), see plan.py.
#include "hq_common.cuh"

namespace {
constexpr int NT = 256, NW = NT / 32;
constexpr int SMEM_DOUBLES = 23552;  // 184 KB: C staged in smem when m*n fits
constexpr int MAX_N = 4096;          // max columns (sigma table)
constexpr int MAX_SWEEPS = 40;

struct SvdSmem {
  double cs[SMEM_DOUBLES];
  double sig[MAX_N];
  int rot;
  int cnt;
};

__global__ void __launch_bounds__(NT) svd_kernel(const hq_svd_prob* __restrict__ probs,
                                                 int* __restrict__ rank,
                                                 const double* __restrict__ scal) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SvdSmem& S = *reinterpret_cast<SvdSmem*>(smem_raw);
  const hq_svd_prob P = probs[blockIdx.x];
  const int m = hq_dim(rank, P.m, P.m_ri);
  const int n = min(hq_dim(rank, P.n, P.n_ri), MAX_N);
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  const double thr = P.eps_scale * (P.eps_slot >= 0 ? scal[P.eps_slot] : 1.0);
  if (m <= 0 || n <= 0) {
    if (t == 0) rank[P.rank_ri] = 0;
    return;
  }
  double* C = P.c;
  int ld = P.ldc;
  const bool staged = (size_t)m * n <= SMEM_DOUBLES;
  if (staged) {
    for (int e = t; e < m * n; e += NT) S.cs[e] = C[e % m + (size_t)(e / m) * ld];
    C = S.cs; ld = m;
  }
  __syncthreads();
  const double tol = sqrt((double)m) * 2.220446049250313e-16;
  const double tiny = 1e-2 * thr;
  const int np = n + (n & 1), N = np - 1;  // circle method: N odd, index N fixed
  for (int sweep = 0; sweep < MAX_SWEEPS && N > 0; ++sweep) {
    if (t == 0) S.rot = 0;
    __syncthreads();
    for (int r = 0; r < N; ++r) {
      for (int pi = wid; pi < np / 2; pi += NW) {
        int p, q;
        if (pi == 0) { p = r; q = N; }
        else { p = (r + pi) % N; q = (r - pi + N) % N; }
        if (p >= n || q >= n) continue;
        if (p > q) { const int tmp = p; p = q; q = tmp; }
        double* cp = C + (size_t)p * ld;
        double* cq = C + (size_t)q * ld;
        double a = 0.0, b = 0.0, g = 0.0;
        for (int i = lane; i < m; i += 32) {
          const double x = cp[i], y = cq[i];
          a = fma(x, x, a); b = fma(y, y, b); g = fma(x, y, g);
        }
        a = warp_sum(a); b = warp_sum(b); g = warp_sum(g);
        const double sa = sqrt(a), sb = sqrt(b);
        if (g == 0.0 || fabs(g) <= tol * sa * sb) continue;
        if (sa < tiny && sb < tiny) continue;  // both far below threshold: dropped anyway
        const double zeta = (b - a) / (2.0 * g);
        double tt;
        if (fabs(zeta) > 1e150) tt = 0.5 / zeta;
        else tt = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / sqrt(1.0 + tt * tt), s = c * tt;
        for (int i = lane; i < m; i += 32) {
          const double x = cp[i], y = cq[i];
          cp[i] = c * x - s * y;
          cq[i] = s * x + c * y;
        }
        if (lane == 0) S.rot = 1;
      }
      __syncthreads();
    }
    if (S.rot == 0) break;
    __syncthreads();
  }
  // singular values = column norms
  for (int j = wid; j < n; j += NW) {
    const double* cj = C + (size_t)j * ld;
    double s = 0.0;
    for (int i = lane; i < m; i += 32) s = fma(cj[i], cj[i], s);
    s = sqrt(warp_sum(s));
    if (lane == 0) S.sig[j] = s;
  }
  if (t == 0) S.cnt = 0;
  __syncthreads();
  // keep sigma > thr (ties truncate), ordered by descending sigma (ties by index)
  for (int j = wid; j < n; j += NW) {
    const double s = S.sig[j];
    if (!(s > thr)) continue;
    int pos = 0;
    for (int o = lane; o < n; o += 32) {
      const double so = S.sig[o];
      pos += (so > s || (so == s && o < j)) ? 1 : 0;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) pos += __shfl_xor_sync(0xffffffffu, pos, off);
    if (lane == 0) atomicAdd(&S.cnt, 1);
    if (pos < P.cap) {
      const double inv = 1.0 / s;
      const double* cj = C + (size_t)j * ld;
      for (int i = lane; i < m; i += 32) P.u[i + (size_t)pos * P.ldu] = cj[i] * inv;
    }
  }
  __syncthreads();
  if (t == 0) {
    int kk = S.cnt;
    if (kk > P.cap) { if (P.flag_ri >= 0) rank[P.flag_ri] = 1; kk = P.cap; }
    rank[P.rank_ri] = kk;
  }
}

// One iteration tail of the two-vector power method (dense.py:121-141) for a
// batch of matrices (block b <-> matrix b): g = Y^T Y (ncol x ncol), x and
// w = A^T A x are n x ncol (ld = n), strided by 2n per matrix.
__global__ void __launch_bounds__(1024) power_kernel(double* x0, const double* w0, const double* g0,
                                                     int n, int ncol, double* scal, double eps,
                                                     double tol, int* done0, int* all_done,
                                                     int nmat, int final_step) {
  __shared__ double red[32];
  const int b = blockIdx.x;
  int* done = done0 + b;
  if (*done) return;
  double* x = x0 + (size_t)b * 2 * n;
  const double* w = w0 + (size_t)b * 2 * n;
  const double* g = g0 + 4 * b;
  const int t = threadIdx.x;
  double theta, v0 = 1.0, v1 = 0.0;
  if (ncol == 1) theta = g[0];
  else {
    const double a = g[0], bb = g[3], c = 0.5 * (g[1] + g[2]);
    const double mid = 0.5 * (a + bb), rad = sqrt(0.25 * (a - bb) * (a - bb) + c * c);
    theta = mid + rad;
    if (c == 0.0) { v0 = a >= bb ? 1.0 : 0.0; v1 = a >= bb ? 0.0 : 1.0; }
    else if (a >= bb) { v0 = theta - bb; v1 = c; }
    else { v0 = c; v1 = theta - a; }
    const double nv = sqrt(v0 * v0 + v1 * v1);
    v0 /= nv; v1 /= nv;
  }
  const double est = sqrt(theta > 0.0 ? theta : 0.0);
  bool fin = false;
  if (est == 0.0) fin = true;
  double rs = 0.0;
  if (!fin) {
    for (int i = t; i < n; i += blockDim.x) {
      double wg = w[i] * v0, xg = x[i] * v0;
      if (ncol == 2) { wg += w[i + n] * v1; xg += x[i + n] * v1; }
      const double d = wg - theta * xg;
      rs += d * d;
    }
  }
  rs = block_sum(rs, red);
  if (fin || sqrt(rs) <= 2.0 * tol * theta || ncol == 1 || final_step) {
    if (t == 0) {
      scal[2 * b] = est; scal[2 * b + 1] = eps * est; *done = 1;
      __threadfence();
      if (atomicAdd(all_done + 1, 1) == nmat - 1) all_done[0] = 1;
    }
    return;
  }
  // x = qr(w): Gram-Schmidt with one reorthogonalization
  double s0 = 0.0;
  for (int i = t; i < n; i += blockDim.x) s0 += w[i] * w[i];
  s0 = block_sum(s0, red);
  const double i0 = s0 > 0.0 ? 1.0 / sqrt(s0) : 0.0;
  for (int i = t; i < n; i += blockDim.x) { x[i] = w[i] * i0; x[i + n] = w[i + n]; }
  __syncthreads();
  for (int pass = 0; pass < 2; ++pass) {
    double d = 0.0;
    for (int i = t; i < n; i += blockDim.x) d += x[i] * x[i + n];
    d = block_sum(d, red);
    for (int i = t; i < n; i += blockDim.x) x[i + n] -= d * x[i];
    __syncthreads();
  }
  double s1 = 0.0;
  for (int i = t; i < n; i += blockDim.x) s1 += x[i + n] * x[i + n];
  s1 = block_sum(s1, red);
  const double i1 = s1 > 0.0 ? 1.0 / sqrt(s1) : 0.0;
  for (int i = t; i < n; i += blockDim.x) x[i + n] *= i1;
  if (t == 0) scal[2 * b] = est;
}

bool g_svd_attr = false;
}  // namespace

extern "C" int hq_svd(void* stream, const hq_svd_prob* probs, int nprob, int* rank,
                      const double* scal) {
  if (nprob <= 0) return 0;
  if (!g_svd_attr) {
    cudaError_t e = cudaFuncSetAttribute(svd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)sizeof(SvdSmem));
    if (e != cudaSuccess) return (int)e;
    g_svd_attr = true;
  }
  svd_kernel<<<nprob, NT, sizeof(SvdSmem), (cudaStream_t)stream>>>(probs, rank, scal);
  return hq_err(cudaGetLastError());
}

extern "C" int hq_power_step(void* stream, double* x, double* w, const double* g, int n,
                             int ncol, double* scal, double eps, double tol, int* done,
                             int* all_done, int nmat, int final_step) {
  if (nmat <= 0) return 0;
  power_kernel<<<nmat, 1024, 0, (cudaStream_t)stream>>>(x, w, g, n, ncol, scal, eps, tol, done,
                                                       all_done, nmat, final_step);
  return hq_err(cudaGetLastError());
}

extern "C" int hq_abi_version(void) { return 1; }

extern "C" int hq_device_check(void) {
  int dev = 0, major = 0, minor = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return -(int)e;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
  return major * 10 + minor;
}
