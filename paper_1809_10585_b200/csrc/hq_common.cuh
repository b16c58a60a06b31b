// Shared device helpers for the B200 HODLR-QR kernels (FP64, column-major).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include "../../include/hodlrqr_b200.h"

#define HQ_DEV __device__ __forceinline__

// dimension (d, d_ri): rank[d_ri] clamped to [0, d] when d_ri >= 0, else d
HQ_DEV int hq_dim(const int* rank, int d, int ri) {
  if (ri < 0) return d;
  int v = rank[ri];
  return v < 0 ? 0 : (v > d ? d : v);
}

HQ_DEV double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// block-wide sum; `red` must hold >= 32 doubles; result broadcast to all threads
HQ_DEV double block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  double s = 0.0;
  if (wid == 0) {
    s = lane < nw ? red[lane] : 0.0;
    s = warp_sum(s);
    if (lane == 0) red[0] = s;
  }
  __syncthreads();
  s = red[0];
  return s;
}

// block-wide maximum of non-negative values (same contract as block_sum)
HQ_DEV double block_max_nonneg(double v, double* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  double s = 0.0;
  if (wid == 0) {
    s = lane < nw ? red[lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s = fmax(s, __shfl_xor_sync(0xffffffffu, s, o));
    if (lane == 0) red[0] = s;
  }
  __syncthreads();
  s = red[0];
  return s;
}

// value of a stored matrix element under a triangular mask
HQ_DEV double hq_mask(double v, int r, int c, int mask) {
  if (mask == 1) return r <= c ? v : 0.0;              // upper incl. diagonal
  if (mask == 2) return r > c ? v : (r == c ? 1.0 : 0.0);  // unit lower
  return v;
}

static inline int hq_err(cudaError_t e) { return (int)e; }

// Explicit shared-memory accesses for pointers the compiler only knows as
// generic (struct references passed into non-inlined functions): a generic
// LD/ST to shared memory resolves the address space at run time and waits on
// the long scoreboard; LDS/STS do not.
HQ_DEV unsigned hq_smem_addr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
HQ_DEV double hq_lds(unsigned a) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];\n" : "=d"(v) : "r"(a) : "memory");
  return v;
}
HQ_DEV void hq_sts(unsigned a, double v) { asm volatile("st.shared.f64 [%0], %1;\n" ::"r"(a), "d"(v) : "memory"); }

// Deterministic K-split: every slice of an output block has stored its
// partial sum into its own workspace slot; the CTA whose arrival completes
// the block's counter (a device int, zero between uses) returns true, resets
// the counter, and then sums the slots in slice order 0..ks-1 -- the result
// is independent of which slice finished last.  Called by every thread.
HQ_DEV bool hq_split_last(int* counter, int ks) {
  __shared__ int s_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const int old = atomicAdd(counter, 1);
    s_last = old == ks - 1;
    if (s_last) atomicExch(counter, 0);
  }
  __syncthreads();
  const bool last = s_last != 0;
  if (last) __threadfence();
  return last;
}

// D (8x8, 2 per lane) += A (8x4, 1 per lane) * B (4x8, 1 per lane): FP64 DMMA.
// Lane l holds A[l>>2][l&3], B[l&3][l>>2], D[l>>2][2(l&3) + {0,1}].
HQ_DEV void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// 8-byte asynchronous global -> shared copy (all in flight; completed by
// cp_async_wait_all + a barrier)
HQ_DEV void cp_async8(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem) : "memory");
}
// 16-byte variant (both addresses 16-byte aligned); .cg: the data is used
// from shared memory only, no L1 allocation
HQ_DEV void cp_async16(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem) : "memory");
}
HQ_DEV void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// ---- 1-D bulk copies on the TMA engine (cp.async.bulk: no tensor map, the
// source is any 16-byte aligned run of a multiple of 16 bytes -- a column of
// a column-major operand).  Loads complete on an mbarrier (transaction
// bytes), stores in a bulk group.
HQ_DEV void mbar_init(unsigned long long* bar, int count) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(a), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
HQ_DEV void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(a), "r"(bytes) : "memory");
}
HQ_DEV void mbar_wait(unsigned long long* bar, unsigned parity) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "HQ_MBAR_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@p bra HQ_MBAR_DONE;\n"
      "bra HQ_MBAR_WAIT;\n"
      "HQ_MBAR_DONE:\n"
      "}\n" ::"r"(a), "r"(parity) : "memory");
}
HQ_DEV void bulk_g2s(void* smem, const void* gmem, unsigned bytes, unsigned long long* bar) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  const unsigned ba = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(sa),
               "l"(gmem), "r"(bytes), "r"(ba)
               : "memory");
}
HQ_DEV void bulk_s2g(void* gmem, const void* smem, unsigned bytes) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(gmem), "r"(sa), "r"(bytes)
               : "memory");
}
HQ_DEV void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
HQ_DEV void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory"); }
// generic-proxy writes to shared memory -> visible to the bulk-copy engine
HQ_DEV void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

// d += A(8 x K) B(K x 8) over k in [kb, ke) on the FP64 tensor pipe with a
// two-stage register pipeline: the operands of the next 32 k-steps are in
// flight while the current 8 mma.sync run.  fetch(k0, av, bv) fills the
// operands of k-steps k0 .. k0+31 (lane's k = k0 + 4u + (lane & 3)).
template <class F>
HQ_DEV void dmma_kloop(double& d0, double& d1, int kb, int ke, F fetch) {
  if (kb >= ke) return;
  double av[8], bv[8];
  fetch(kb, av, bv);
  for (int k0 = kb; k0 < ke; k0 += 32) {
    double an[8], bn[8];
    const bool more = k0 + 32 < ke;
    if (more) fetch(k0 + 32, an, bn);
#pragma unroll
    for (int u = 0; u < 8; ++u) dmma884(d0, d1, av[u], bv[u]);
    if (more) {
#pragma unroll
      for (int u = 0; u < 8; ++u) { av[u] = an[u]; bv[u] = bn[u]; }
    }
  }
}

// Reflector of the column x = [x0; v] (dense.py:45-68) from the sum of
// squares ss of v (scaled by sc, see below), with the reference's sign
// convention rho = -sign(x0) ||x||, sign(0) = +1, and gamma = 0 for x = 0.
// The reference divides by max|x| before the norm.  Here the unscaled sum is
// used whenever x0^2 + ss lies in [2^-900, 2^900]: then no square overflowed
// and every square that underflowed is below 2^-112 of the total, so the
// result equals the scaled one to rounding.  Otherwise (rare: zero or tiny
// columns, overflow, inf/NaN) the column is rescaled by an exact power of two
// sc chosen from max|x| and the sum recomputed.
struct Refl { double gamma, rho, inv; };
HQ_DEV bool refl_safe(double x0, double ss) {
  const double tot = fma(x0, x0, ss);
  return tot >= 0x1p-900 && tot <= 0x1p900;   // false for 0, inf and NaN
}
HQ_DEV double refl_scale(double amax) {
  return amax < 0x1p-480 ? 0x1p600 : (amax > 0x1p480 ? 0x1p-600 : 1.0);
}
// isc = 1 / sc (exact: sc is a power of two)
HQ_DEV Refl make_refl(double x0, double ss, double sc, double isc) {
  Refl r{0.0, 0.0, 0.0};
  const double xs = x0 * sc;
  const double nrm = sqrt(fma(xs, xs, ss));
  if (nrm != 0.0) {
    const double sg = x0 < 0.0 ? -1.0 : 1.0;   // sign(0) := +1
    const double u1 = xs + sg * nrm;           // no cancellation
    r.rho = -sg * nrm * isc;
    const double iu = 1.0 / u1;
    r.inv = sc * iu;                           // y = v * inv
    r.gamma = 2.0 / (1.0 + ss * iu * iu);
  }
  return r;
}

// Reflector of x = [x0; v] from ss = sum v^2 (both in the safe range, see
// refl_safe) with the hardware reciprocal / reciprocal square root refined
// by Newton steps to full FP64 accuracy: ||x||, 1 / u1 and gamma = |u1| /
// ||x|| (= 2 / (1 + ss / u1^2)) cost two short dependent chains instead of a
// software sqrt and two divisions on the per-step critical path.
HQ_DEV Refl make_refl_fast(double x0, double ss) {
  const double tot = fma(x0, x0, ss);
  double rn;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(rn) : "d"(tot));
  const double ht = 0.5 * tot;
  rn = rn * fma(-ht * rn, rn, 1.5);
  rn = rn * fma(-ht * rn, rn, 1.5);
  double nrm = tot * rn;
  nrm = fma(0.5 * rn, fma(-nrm, nrm, tot), nrm);
  const double sg = x0 < 0.0 ? -1.0 : 1.0;
  const double u1 = fma(sg, nrm, x0);
  double iu;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(iu) : "d"(u1));
  iu = iu * fma(-u1, iu, 2.0);
  iu = iu * fma(-u1, iu, 2.0);
  Refl r;
  r.rho = -sg * nrm;
  r.inv = iu;
  r.gamma = fabs(u1) * rn;
  return r;
}
