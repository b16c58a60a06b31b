// Column-pivoted Householder QR of the truncation core, R factor only
// (hq_qrcp): the rank-revealing preconditioner of the truncation Jacobi.
//   truncate_lowrank: reference core.py:239-258 (svd of the core + rank rule
//   core.py:250-253, dense.py:93-99); the pivoted QR itself has no reference
//   counterpart -- it changes how the core's SVD is computed, not its result.
// The core C (m x n, from hq_gemm) is reduced to C P = Q [R11 R12; 0 R22] by
// Householder reflectors with Businger-Golub pivoting, stopping at the first
// step r where the remaining columns are negligible against the truncation
// threshold ((n - r) max_c ||R22[:, c]||^2 <= (stop_scale * scal)^2, i.e.
// ||R22||_F <= 1e-3 thr with the plan's stop_scale).  Columns are never
// swapped: on exit rows 0..r-1 of C hold [R11 R12] P^T (original column
// order), so X = (those rows)^T (n x r) has the left singular vectors of C^T
// up to the dropped R22, and the Jacobi runs on r <= rank + few graded
// columns instead of min(m, n) (measured on the
// bench workload's cores: 2.8x less Jacobi time, identical ranks).
// Q is never formed or applied.
//
// One cluster of G CTAs per problem (G = 1: one CTA).  CTA c owns a slice of
// columns in shared memory, element (i, col) at As[i * lds + col], so the
// reflector application is thread-per-column: TPC threads share a column
// (rows i = h mod TPC), no reduction tree beyond log2(TPC) shuffles, column
// norms downdated by the owning threads (LAPACK dgeqp3's safeguard: recompute
// when cancellation is severe).  Per step every CTA proposes its best column
// WITH its finished reflector to all CTAs through distributed shared memory;
// after ONE cluster barrier every CTA picks the same winner and applies it.
// Slices too large for shared memory are processed in place in global memory
// (warp per column).
#include "hq_common.cuh"
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

namespace {
constexpr int CP_HDR = 4;   // candidate header: tracked norm, gamma, rho, global column

template <int G>
__device__ __forceinline__ void cp_sync() {
  if constexpr (G > 1) cg::this_cluster().sync();
  else __syncthreads();
}

template <int G>
__device__ __forceinline__ double* cp_remote(double* p, int r) {
  if constexpr (G > 1) return cg::this_cluster().map_shared_rank(p, r);
  else return p;
}

// pivot key of a column: its squared norm's bit pattern (monotonic for
// non-negative doubles) with the low 11 bits replaced by 2047 - local column
// (a CTA owns at most 2047 columns): one 64-bit maximum picks the largest norm
// (to 2^-41 relative) and, among equals, the lowest column.  0 = no column.
HQ_DEV unsigned long long cp_key(double vn2, int col) {
  return ((unsigned long long)__double_as_longlong(vn2) & ~0x7FFull) | (unsigned long long)(2047 - col);
}

template <int G>
__global__ void qrcp_kernel(const hq_qrcp_prob* __restrict__ probs, int* __restrict__ rank,
                            const double* __restrict__ scal, int smem_doubles) {
  extern __shared__ __align__(16) double sm[];
  int cr = 0;
  if constexpr (G > 1) cr = (int)cg::this_cluster().block_rank();
  const hq_qrcp_prob P = probs[blockIdx.x / G];
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5, nt = blockDim.x, nw = nt >> 5;
  const int m = hq_dim(rank, P.m, P.m_ri), n = hq_dim(rank, P.n, P.n_ri);
  if (m <= 0 || n <= 0) {   // uniform over the cluster
    if (cr == 0 && t == 0) rank[P.r_ri] = 0;
    return;
  }
  const int kmax = min(m, n);
  const double stop = P.stop_scale * (P.eps_slot >= 0 ? scal[P.eps_slot] : 1.0);
  const double stop2 = stop * stop;
  const int ncl_max = (n + G - 1) / G, c0 = cr * ncl_max;
  const int ncl = max(0, min(ncl_max, n - c0));
  // threads per column (power of two) and the row stride that keeps the
  // half-warps' accesses (a few rows x 32/TPC columns) on distinct banks
  int tpc = 1;
  while (tpc < 32 && ncl_max * tpc * 2 <= nt) tpc *= 2;
  const int cpw = 32 / tpc;                       // columns per warp
  const int q = tpc >= 4 ? 32 / tpc : 0;          // lds mod 16
  const int lds = ncl_max + ((q - ncl_max) % 16 + 16) % 16;
  const int mp = ((m + 1) & ~1) + CP_HDR;
  unsigned long long* keymax = reinterpret_cast<unsigned long long*>(sm);   // [2] by step parity
  double* bc = sm + 2;              // my candidate's header + 1 / u1, warp 0 -> all threads
  double* vn = sm + 8;              // squared column norms, tracked (< 0: column already a pivot)
  double* vref = vn + ncl_max;      // squared norm at the last exact computation
  double* cand = vref + ncl_max;    // [2][G][mp]: candidates by step parity and proposing CTA
  double* As = cand + 2 * G * mp;
  const bool in_smem = ncl_max * tpc <= nt &&
                       (size_t)(As - sm) + (size_t)m * lds <= (size_t)smem_doubles;
  double* Cg = P.c + (size_t)c0 * P.ldc;   // my slice in global memory
  const int ldc = P.ldc;
  // thread -> (column, row phase) of the shared-memory mode
  const int h = lane / cpw, cc = lane % cpw, col = wid * cpw + cc;
  const bool mine = col < ncl;
  if (t < 2) keymax[t] = 0ull;
  __syncthreads();

  // ---- load the slice, exact squared column norms, first pivot keys
  if (in_smem) {
    double ss = 0.0;
    if (mine) {
      const double* src = Cg + (size_t)col * ldc;
      for (int i = h; i < m; i += tpc) {
        const double v = src[i];
        As[i * lds + col] = v;
        ss = fma(v, v, ss);
      }
    }
    for (int o = cpw; o < 32; o <<= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    if (mine && h == 0) { vn[col] = ss; vref[col] = ss; atomicMax(&keymax[0], cp_key(ss, col)); }
  } else {
    for (int c = wid; c < ncl; c += nw) {
      const double* src = Cg + (size_t)c * ldc;
      double ss = 0.0;
      for (int i = lane; i < m; i += 32) ss = fma(src[i], src[i], ss);
      ss = warp_sum(ss);
      if (lane == 0) { vn[c] = ss; vref[c] = ss; atomicMax(&keymax[0], cp_key(ss, c)); }
    }
  }
  __syncthreads();

  int r = kmax;
  for (int j = 0; j < kmax; ++j) {
    double* mycand = cand + (size_t)((j & 1) * G + cr) * mp;
    // ---- phase A (warp 0): best local column and its reflector, to all CTAs
    if (wid == 0) {
      const unsigned long long key = keymax[j & 1];
      const int bi = key ? 2047 - (int)(key & 0x7FFull) : -1;
      const double best = bi >= 0 ? __longlong_as_double((long long)(key & ~0x7FFull)) : -1.0;
      if (lane == 0) keymax[(j + 1) & 1] = 0ull;
      double gamma = 0.0, rho = 0.0, inv = 0.0;
      if (bi >= 0) {
        // raw column into my own candidate slot, sum of squares below the diagonal
        double ss = 0.0, x0 = 0.0;
        for (int i = j + lane; i < m; i += 32) {
          const double v = in_smem ? As[i * lds + bi] : Cg[(size_t)bi * ldc + i];
          mycand[CP_HDR + i] = v;
          if (i > j) ss = fma(v, v, ss); else x0 = v;
        }
        ss = warp_sum(ss);
        x0 = __shfl_sync(0xffffffffu, x0, 0);
        Refl R;
        if (refl_safe(x0, ss)) {
          R = make_refl_fast(x0, ss);
        } else {   // warp-uniform, rare: rescale by max|x| (zero, tiny or huge columns)
          double amax = 0.0;
          __syncwarp();
          for (int i = j + lane; i < m; i += 32) amax = fmax(amax, fabs(mycand[CP_HDR + i]));
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
          const double sc = refl_scale(amax);
          const double isc = sc == 1.0 ? 1.0 : (sc > 1.0 ? 0x1p-600 : 0x1p600);
          ss = 0.0;
          for (int i = j + 1 + lane; i < m; i += 32) { const double v = mycand[CP_HDR + i] * sc; ss = fma(v, v, ss); }
          ss = warp_sum(ss);
          R = make_refl(x0, ss, sc, isc);
        }
        gamma = R.gamma; rho = R.rho; inv = R.inv;
      }
      if constexpr (G == 1) {
        __syncwarp();
        if (bi >= 0)
          for (int i = j + lane; i < m; i += 32) mycand[CP_HDR + i] = i > j ? mycand[CP_HDR + i] * inv : 1.0;
        if (lane == 0) { mycand[0] = best; mycand[1] = gamma; mycand[2] = rho; mycand[3] = bi >= 0 ? (double)(c0 + bi) : -1.0; }
      } else if (lane == 0) {
        bc[0] = best; bc[1] = gamma; bc[2] = rho; bc[3] = bi >= 0 ? (double)(c0 + bi) : -1.0; bc[4] = inv;
      }
    }
    if constexpr (G > 1) {
      // every thread takes part in the broadcast of the scaled reflector:
      // one thread per row writes its value to all G copies (its own last)
      __syncthreads();
      const double inv = bc[4];
      if (bc[3] >= 0.0) {
        for (int i = j + t; i < m; i += nt) {
          const double sv = i > j ? mycand[CP_HDR + i] * inv : 1.0;
#pragma unroll
          for (int rr = 1; rr < G; ++rr) cp_remote<G>(mycand, (cr + rr) % G)[CP_HDR + i] = sv;
          mycand[CP_HDR + i] = sv;
        }
      }
      if (t < G) {
        double* rc = cp_remote<G>(mycand, (cr + t) % G);
        rc[0] = bc[0]; rc[1] = bc[1]; rc[2] = bc[2]; rc[3] = bc[3];
      }
    }
    cp_sync<G>();
    // ---- phase B: the same winner in every CTA
    int wc = 0;
    double wbest = -1.0, wcol = -1.0;
#pragma unroll
    for (int c = 0; c < G; ++c) {
      const double* hd = cand + (size_t)((j & 1) * G + c) * mp;
      const double b = hd[0], gc = hd[3];
      if (gc >= 0.0 && (b > wbest || (b == wbest && gc < wcol))) { wbest = b; wcol = gc; wc = c; }
    }
    if (wcol < 0.0 || wbest <= 0.0 || (double)(n - j) * wbest <= stop2) { r = j; break; }
    const double* wh = cand + (size_t)((j & 1) * G + wc) * mp;
    const double gamma = wh[1], rho = wh[2];
    const double* v = wh + CP_HDR;
    const int pc = wc == cr ? (int)wcol - c0 : -1;   // the pivot, if it is mine
    unsigned long long* knext = &keymax[(j + 1) & 1];
    if (in_smem) {
      const double vold = mine ? vn[col] : -1.0;
      const bool act = mine && col != pc && vold >= 0.0;
      const int i0 = j + ((h - j) % tpc + tpc) % tpc;   // first row >= j with row = h (mod tpc)
      double* a = As + col;
      const int st = tpc * lds;
      double d0 = 0.0, d1 = 0.0, d2 = 0.0, d3 = 0.0;
      if (act) {
        int i = i0;
        const double* ap = a + (size_t)i * lds;
        for (; i + 3 * tpc < m; i += 4 * tpc, ap += 4 * st) {
          d0 = fma(v[i], ap[0], d0);
          d1 = fma(v[i + tpc], ap[st], d1);
          d2 = fma(v[i + 2 * tpc], ap[2 * st], d2);
          d3 = fma(v[i + 3 * tpc], ap[3 * st], d3);
        }
        for (; i < m; i += tpc, ap += st) d0 = fma(v[i], ap[0], d0);
      }
      double dot = (d0 + d1) + (d2 + d3);
      for (int o = cpw; o < 32; o <<= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
      const double tau = gamma * dot;
      double rj = 0.0;
      if (act) {
        int i = i0;
        double* ap = a + (size_t)i * lds;
        if (i == j) { rj = fma(-tau, v[i], ap[0]); ap[0] = rj; i += tpc; ap += st; }
        for (; i + tpc < m; i += 2 * tpc, ap += 2 * st) {
          const double n0 = fma(-tau, v[i], ap[0]), n1 = fma(-tau, v[i + tpc], ap[st]);
          ap[0] = n0; ap[st] = n1;
        }
        if (i < m) ap[0] = fma(-tau, v[i], ap[0]);
      }
      rj = __shfl_sync(0xffffffffu, rj, (j % tpc) * cpw + cc);
      // squared-norm downdate with dgeqp3's safeguard: exact recomputation
      // when the tracked value has cancelled to sqrt(eps) of the last exact one
      double vnew = fmax(fma(-rj, rj, vold), 0.0);
      const bool redo = act && vnew <= 1.4901161193847656e-08 * vref[col];
      if (__any_sync(0xffffffffu, redo)) {
        double ss = 0.0;
        if (redo)
          for (int i = i0 + (i0 == j ? tpc : 0); i < m; i += tpc) ss = fma(a[(size_t)i * lds], a[(size_t)i * lds], ss);
        for (int o = cpw; o < 32; o <<= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
        if (redo) { vnew = ss; if (h == 0) vref[col] = ss; }
      }
      if (act && h == 0) { vn[col] = vnew; atomicMax(knext, cp_key(vnew, col)); }
      if (mine && col == pc) {
        for (int i = i0; i < m; i += tpc) a[(size_t)i * lds] = i == j ? rho : 0.0;
        if (h == 0) vn[col] = -1.0;
      }
    } else {
      for (int c = wid; c < ncl; c += nw) {
        double* a = Cg + (size_t)c * ldc;
        if (c == pc) {
          for (int i = j + lane; i < m; i += 32) a[i] = i == j ? rho : 0.0;
          if (lane == 0) vn[c] = -1.0;
          continue;
        }
        if (vn[c] < 0.0) continue;
        double dot = 0.0;
        for (int i = j + lane; i < m; i += 32) dot = fma(v[i], a[i], dot);
        dot = warp_sum(dot);
        const double tau = gamma * dot;
        double ss = 0.0;   // the exact squared norm comes for free with the update pass
        for (int i = j + lane; i < m; i += 32) {
          const double nv = fma(-tau, v[i], a[i]);
          a[i] = nv;
          if (i > j) ss = fma(nv, nv, ss);
        }
        ss = warp_sum(ss);
        if (lane == 0) { vn[c] = ss; atomicMax(knext, cp_key(ss, c)); }
      }
    }
    __syncthreads();
  }
  // ---- rows 0..r-1 back to C (shared-memory mode), r to the rank table
  if (in_smem) {
    __syncthreads();
    for (int e = t; e < r * ncl; e += nt) {
      const int i = e / ncl, c = e % ncl;
      Cg[(size_t)c * ldc + i] = As[i * lds + c];
    }
  }
  if (cr == 0 && t == 0) rank[P.r_ri] = r;
  cp_sync<G>();   // nobody leaves while a peer may still read or write its shared memory
}

template <int G>
int launch_qrcp(cudaStream_t st, const hq_qrcp_prob* probs, int nprob, int* rank, const double* scal,
                int smem_doubles, int threads) {
  static int attr_bytes = 0;
  auto kern = qrcp_kernel<G>;
  const int bytes = smem_doubles * 8;
  if (bytes > attr_bytes) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e != cudaSuccess) return (int)e;
    attr_bytes = bytes;
  }
  if (G == 1) {
    kern<<<nprob, threads, bytes, st>>>(probs, rank, scal, smem_doubles);
    return hq_err(cudaGetLastError());
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nprob * G);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = bytes;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = G;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return (int)cudaLaunchKernelEx(&cfg, kern, probs, rank, scal, smem_doubles);
}
}  // namespace

extern "C" int hq_qrcp(void* stream, const hq_qrcp_prob* probs, int nprob, int* rank,
                       const double* scal, int cluster, int smem_doubles, int threads) {
  if (nprob <= 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  if (smem_doubles < 64) smem_doubles = 64;
  if (smem_doubles > 28928) smem_doubles = 28928;   // 226 KB
  if (threads != 256 && threads != 512) threads = 512;
  if (cluster >= 8) return launch_qrcp<8>(st, probs, nprob, rank, scal, smem_doubles, threads);
  if (cluster >= 4) return launch_qrcp<4>(st, probs, nprob, rank, scal, smem_doubles, threads);
  if (cluster >= 2) return launch_qrcp<2>(st, probs, nprob, rank, scal, smem_doubles, threads);
  return launch_qrcp<1>(st, probs, nprob, rank, scal, smem_doubles, threads);
}
