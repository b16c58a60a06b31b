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

#include "hq_svd_kernel.cuh"
#include "hq_svd_cluster.cuh"
#include "hq_svd_block.cuh"

namespace {
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

template <int G>
static cudaLaunchConfig_t cluster_config(cudaStream_t st, int nprob, int smem, cudaLaunchAttribute* at) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nprob * G);
  cfg.blockDim = dim3(CNT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = G;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cfg;
}

// 0: not yet checked, 1: the device can co-schedule a cluster of G CTAs at
// this shared-memory size, -1: it cannot (e.g. a MIG slice or a GPC with
// fewer free SMs): such launches run as 8-CTA clusters instead
template <int G>
static int& cluster_ok() {
  static int ok = 0;
  return ok;
}

template <int G>
static int launch_cluster(cudaStream_t st, const hq_svd_prob* probs, int nprob, int* rank,
                          const double* scal) {
  static bool attr = false;
  auto kern = svd_cluster_kernel<G>;
  const int smem = (int)(sizeof(CSmem) > sizeof(SvdSmem) ? sizeof(CSmem) : sizeof(SvdSmem));
  cudaLaunchAttribute at[1];
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return (int)e;
    if (G > 8) {   // 16-CTA clusters are non-portable (opt-in)
      e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      if (e != cudaSuccess) return (int)e;
    }
    attr = true;
  }
  if (G > 8) {
    int& ok = cluster_ok<G>();
    if (ok == 0) {
      cudaLaunchConfig_t probe = cluster_config<G>(st, 1, smem, at);
      int nclusters = 0;
      const cudaError_t e = cudaOccupancyMaxActiveClusters(&nclusters, kern, &probe);
      ok = (e == cudaSuccess && nclusters > 0) ? 1 : -1;
      if (e != cudaSuccess) (void)cudaGetLastError();
    }
    if (ok < 0) return -1;   // caller falls back to a portable cluster size
  }
  cudaLaunchConfig_t cfg = cluster_config<G>(st, nprob, smem, at);
  return (int)cudaLaunchKernelEx(&cfg, kern, probs, rank, scal);
}

extern "C" int hq_svd(void* stream, const hq_svd_prob* probs, int nprob, int* rank,
                      const double* scal, int cluster, int max_m, int small_doubles) {
  if (nprob <= 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  if (cluster == 0) {
    // small cores: 128-thread CTAs, small_doubles of staging each
    static int attr_bytes = 0;
    if (small_doubles < 64) small_doubles = 64;
    if (small_doubles > SMEM_DOUBLES) small_doubles = SMEM_DOUBLES;
    const int bytes = (int)offsetof(SvdSmem, cs) + 8 * small_doubles;
    if (bytes > attr_bytes) {
      cudaError_t e = cudaFuncSetAttribute(svd_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
      if (e != cudaSuccess) return (int)e;
      attr_bytes = bytes;
    }
    svd_small_kernel<<<nprob, SMALL_NT, bytes, st>>>(probs, rank, scal, small_doubles);
    return hq_err(cudaGetLastError());
  }
  if (cluster >= 2) {
    (void)max_m;  // cores past the cluster's limits run on CTA 0 (kernel-side test)
    if (cluster == 2) return launch_cluster<2>(st, probs, nprob, rank, scal);
    if (cluster <= 4) return launch_cluster<4>(st, probs, nprob, rank, scal);
    if (cluster <= 8) return launch_cluster<8>(st, probs, nprob, rank, scal);
    // 16-CTA clusters only where the device can place them (checked once);
    // otherwise 8 (a core that outgrows the 8-CTA cluster runs on CTA 0)
    const int rc = launch_cluster<16>(st, probs, nprob, rank, scal);
    return rc == -1 ? launch_cluster<8>(st, probs, nprob, rank, scal) : rc;
  }
  if (!g_svd_attr) {
    cudaError_t e = cudaFuncSetAttribute(svd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)sizeof(SvdSmem));
    if (e != cudaSuccess) return (int)e;
    g_svd_attr = true;
  }
  svd_kernel<<<nprob, NT, sizeof(SvdSmem), st>>>(probs, rank, scal);
  return hq_err(cudaGetLastError());
}

template <int G>
static int launch_block(cudaStream_t st, const hq_svd_prob* probs, int nprob, int* rank, const double* scal) {
  static bool attr = false;
  auto kern = svd_block_kernel<G>;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(BjSmem));
    if (e != cudaSuccess) return (int)e;
    attr = true;
  }
  if (G == 1) {
    kern<<<nprob, BJ_NT, sizeof(BjSmem), st>>>(probs, rank, scal);
    return hq_err(cudaGetLastError());
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nprob * G);
  cfg.blockDim = dim3(BJ_NT);
  cfg.dynamicSmemBytes = sizeof(BjSmem);
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = G;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return (int)cudaLaunchKernelEx(&cfg, kern, probs, rank, scal);
}

extern "C" int hq_svd_block(void* stream, const hq_svd_prob* probs, int nprob, int* rank,
                            const double* scal, int cluster) {
  if (nprob <= 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  if (cluster >= 8) return launch_block<8>(st, probs, nprob, rank, scal);
  if (cluster >= 4) return launch_block<4>(st, probs, nprob, rank, scal);
  if (cluster >= 2) return launch_block<2>(st, probs, nprob, rank, scal);
  return launch_block<1>(st, probs, nprob, rank, scal);
}

extern "C" int hq_power_step(void* stream, double* x, double* w, const double* g, int n,
                             int ncol, double* scal, double eps, double tol, int* done,
                             int* all_done, int nmat, int final_step) {
  if (nmat <= 0) return 0;
  power_kernel<<<nmat, 1024, 0, (cudaStream_t)stream>>>(x, w, g, n, ncol, scal, eps, tol, done,
                                                       all_done, nmat, final_step);
  return hq_err(cudaGetLastError());
}

extern "C" int hq_abi_version(void) { return HQ_ABI_VERSION; }

extern "C" int hq_device_check(void) {
  int dev = 0, major = 0, minor = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return -(int)e;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
  return major * 10 + minor;
}
