/*
 * hodlrqr_b200.h -- C ABI of the B200 HODLR-QR kernel library (libhqb200.so).
 *
 * The reference (hodlrqr, pure Python/numpy) has no native FFI; its hot path
 * is the Python call chain
 *     hqr()                 pkg/src/hodlrqr/hqr.py:80-92
 *       hqr_rec()           pkg/src/hodlrqr/hqr.py:95-194
 *         block_qr()        pkg/src/hodlrqr/wy.py:75-88      (leaf compressed column)
 *         truncate_lowrank  pkg/src/hodlrqr/core.py:239-258  (T_eps recompression)
 *         apply_dense /     pkg/src/hodlrqr/arith.py:35-64   (HODLR x dense)
 *         apply_transpose_dense
 *         low_rank_update   pkg/src/hodlrqr/arith.py:126-145
 *       hodlr_spectral_norm pkg/src/hodlrqr/arith.py:293-298 (power iteration)
 * The Python package paper_1809_10585_b200 keeps that API and drives this
 * library through ctypes.  Every entry point launches ONE batched kernel over
 * an array of problem descriptors that lives in device memory; dimensions
 * marked *_ri are read at run time from the device rank table (int32), so a
 * whole factorization is a fixed launch sequence that can be captured into a
 * CUDA graph once per tree shape and replayed.
 *
 * All matrices are FP64, column-major.  A dimension pair (d, d_ri) means: the
 * value is rank[d_ri] clamped to d when d_ri >= 0, otherwise d.
 * Every launcher returns 0 on success or a cudaError_t code.
 */
#ifndef HODLRQR_B200_H
#define HODLRQR_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- descriptors (layouts mirrored by numpy dtypes in _abi.py) ---------- */

/* one term alpha * op(A) * op(B); mask: 0 full, 1 upper incl. diagonal,
   2 unit lower (strict lower + ones); masks act on the STORED matrix */
typedef struct hq_gemm_term {
  const double* a;
  const double* b;
  int32_t lda, ldb;
  int32_t ta, tb;
  int32_t k, k_ri;
  int32_t mask_a, mask_b;
  double alpha;
} hq_gemm_term;

/* C (m x n) = beta*C + sum_t term_t   (reference: every @ in arith.py/hqr.py).
   K-split launches are deterministic: each K slice of an output block writes
   its partial sum into its own slot of ws, the last slice to arrive (counter
   cnt[block]) adds the slots in slice order 0..ks-1 and writes C; the result
   is bit-identical run to run and independent of the arrival order.  ws and
   cnt are per problem; the slot layout is given per launcher below. */
typedef struct hq_gemm_prob {
  double* c;
  int32_t ldc;
  int32_t m, m_ri, n, n_ri;
  int32_t term0, nterm;
  int32_t item0;   /* hq_gemm_skinny mode 5: first work item of this problem */
  double beta;
  double* ws;      /* K-split partial sums (unused when the problem is not split) */
  int32_t* cnt;    /* arrival counters, one per output block: zero on entry, left zero */
} hq_gemm_prob;

/* a column block of a concatenation [alpha_1 P_1, alpha_2 P_2, ...] */
typedef struct hq_piece {
  const double* p;
  int32_t ld;
  int32_t cols, cols_ri;
  int32_t pad_;
  double alpha;
} hq_piece;

/* dst (rows x sum cols) = concat(pieces); optional copy into dst2;
   the total column count is written to rank[ktot_ri]
   (reference: np.hstack of factors before truncate_lowrank, hqr.py:145,154) */
typedef struct hq_concat_prob {
  double* dst;
  double* dst2;
  int32_t ldd, ldd2;
  int32_t rows;
  int32_t piece0, npiece;
  int32_t ktot_ri;
} hq_concat_prob;

/* in-place Householder QR of W (m x k): R on/above the diagonal, unit-lower
   reflectors below, gamma in tau, per-panel T in tpanel (ceil(r/16) blocks of
   16 x 16, r = min(m, k)); optional full compact-WY T (r x r) into tfull
   (reference: wy.py:17-72, dense.py:45-68).  With tfull and cluster >= 2,
   tpanel must have room for 2 * r * 16 more doubles (merge scratch). */
typedef struct hq_qr_prob {
  double* w;
  double* tau;
  double* tpanel;
  double* tfull;
  int32_t ldw, ldt;
  int32_t m, m_ri, k, k_ri;
} hq_qr_prob;

/* X (m x c) := Q X (trans=0) or Q^T X (trans=1) with Q from an hq_qr_prob;
   when x0 != NULL, X is first set to [x0 (r0 x c); 0] */
typedef struct hq_applyq_prob {
  const double* w;
  const double* tau;
  const double* tpanel;
  double* x;
  const double* x0;
  int32_t ldw, ldx, ldx0;
  int32_t m, m_ri, k, k_ri;
  int32_t c, c_ri;
  int32_t r0, r0_ri;
  int32_t trans;
} hq_applyq_prob;

/* one-sided Jacobi SVD of X (m x n).  xform = 0: X = C as stored (destroyed).
   xform = 1: c holds R (from hq_qr of C^T, R upper, min(n,m) x m) and
   X = R^T (m x min(m,n)): the LQ-preconditioned matrix whose left singular
   vectors are those of C and on which Jacobi converges in a few sweeps.
   Keeps the k' columns with sigma > thr, thr = eps_scale * scal[eps_slot]
   (eps_slot < 0: eps_scale), writes the left singular vectors U_k (m x k',
   sigma descending) and k' into rank[rank_ri]; k' > cap sets rank[flag_ri]
   and clamps.  work: ((m + 1) & ~1) * n doubles (X when it does not fit
   shared memory; always with hq_svd_block).
   (reference: svd + truncation_rank in core.py:250-253, dense.py:93-99) */
typedef struct hq_svd_prob {
  double* c;
  double* u;
  double* work;
  int32_t ldc, ldu;
  int32_t m, m_ri, n, n_ri;
  int32_t cap, rank_ri, flag_ri, eps_slot;
  double eps_scale;
  int32_t xform, pad_;
} hq_svd_prob;

/* column-pivoted Householder QR of a truncation core C (m x n, destroyed), R
   only, stopped at the first step r where the remaining columns are
   negligible: (n - r) max ||R22[:, c]||^2 <= (stop_scale * scal[eps_slot])^2
   (eps_slot < 0: stop_scale^2; stop_scale = 0: only exactly zero columns
   stop it).  Columns are not swapped: on exit rows 0..r-1 of c hold
   [R11 R12] P^T in the original column order and r is in rank[r_ri]; with
   hq_svd_prob.xform = 2 the Jacobi runs on X = (those rows)^T (n x r), whose
   left singular vectors are those of C^T up to the dropped block.
   (reference: the svd inside truncate_lowrank, core.py:250-253) */
typedef struct hq_qrcp_prob {
  double* c;
  int32_t ldc;
  int32_t m, m_ri, n, n_ri;
  int32_t r_ri, eps_slot, pad_;
  double stop_scale;
} hq_qrcp_prob;

/* a slab of reduced-away rows B_R of an ancestor (hqr.py:112,127) */
typedef struct hq_slab {
  const double* v;   /* V factor rows for this leaf: element (i,c) = v[c + i*ld] */
  double* yv;        /* destination of the matching rows of Y (same layout) */
  int32_t ld, ldy;
  int32_t k_ri;
  int32_t pad_;
} hq_slab;

/* compressed leaf column [A_leaf; B_R; C] (hqr.py:110-119) */
typedef struct hq_leaf_prob {
  double* leaf;
  double* panel;
  int32_t nl, ldp;
  int32_t slab0, nslab;
  int32_t m_ri;
  int32_t pad_;
} hq_leaf_prob;

/* one column-major 2D copy dst(rows x cols) = src; cols from the rank table
   when cols_ri >= 0 (used to restore inputs and to compact the factors for
   the single device->host copy).  mode 0 copies; mode 1 writes the upper
   triangle (zeros below the diagonal: R and T leaves); mode 2 the unit lower
   triangle (ones on the diagonal, zeros above: Y leaves) */
typedef struct hq_copy_item {
  const double* src;
  double* dst;
  int32_t rows, cols, cols_ri, lds, ldd;
  int32_t mode;
} hq_copy_item;

/* TSQR row blocks of a tall factor stack W (rows_total x K, chunks of ch rows
   QR'd in place): mode 0 stacks each chunk's R (its top min(rows_c, K) rows,
   upper part) densely into S (rank[ms_ri] = stacked row count); mode 1
   scatters the matching row blocks of S back to the chunk tops of X (= W
   argument, ncol columns) and zero-fills the rest of every chunk */
typedef struct hq_rowblk_prob {
  double* s;
  double* w;
  int32_t lds, ldw;
  int32_t ch, rows_total;
  int32_t k, k_ri;
  int32_t ncol, ncol_ri;
  int32_t ms_ri, mode;
} hq_rowblk_prob;

/* ---- launchers ---------------------------------------------------------- */
/* bumped whenever a descriptor layout or a launcher signature changes;
   the Python binding refuses a library with another version */
#define HQ_ABI_VERSION 6
int hq_abi_version(void);
int hq_device_check(void);

/* grid = tiles x nprob x ksplit; a problem with nkt k-tiles of 16 (summed
   over its terms) is split into ks = min(ksplit, max(1, nkt / 8)) slices;
   with ks > 1 its ws holds tiles_cap x ks_cap slots of BM x BN doubles
   (slot (tile, z) at (tile * ks_cap + z) * BM * BN, element (i, j) at i + j * BM;
   ks_cap = the same formula on the capacity k's, tiles_cap from the capacity
   m, n) and cnt one counter per output tile.  skip != NULL && *skip != 0
   makes it a no-op */
int hq_gemm(void* stream, const hq_gemm_prob* probs, int nprob, const hq_gemm_term* terms,
            int* rank, int tiles, int ksplit, const int* skip);
/* hq_gemm with the output tile size chosen (tile = 32 or 64; tiles counts
   tile x tile blocks): small products use 32 x 32 tiles to occupy more SMs */
int hq_gemm_tiled(void* stream, const hq_gemm_prob* probs, int nprob, const hq_gemm_term* terms,
                  int* rank, int tiles, int ksplit, int tile, const int* skip);
/* the same product for outputs of at most 4 columns (power-iteration
   blocks^T X, Gram and leaf products).  mode 0: grid (ksplit, nprob), K split
   evenly over CTAs; with ksplit > 1, ws holds ksplit slots of m_cap x n_cap
   (ld m_cap) and cnt one counter; mode 1: one thread per output row
   (max_rows bounds m), ksplit ignored; mode 2: 64 output rows per CTA
   (max_rows bounds m), each term read coalesced in its own layout (rows
   across lanes for op(A) = A, k across lanes for op(A) = A^T), K split into
   ks = min(ksplit, max(1, K / 512)) slices (K summed over the terms): with
   ks > 1, ws holds ceil(m_cap / 64) x ks_cap slots of 64 x NC doubles (slot
   (row block, z) at (rb * ks_cap + z) * 64 * NC, NC = 2 for ncmax <= 2 else 4)
   and cnt one counter per row block; modes 3 / 4: mode 2 specialised to
   launches whose terms are all op(A) = A / all op(A) = A^T; mode 5: one
   launch over problems of different K (all op(A) = A^T, one term each):
   problem i owns work items [item0_i, item0_{i+1}) -- its K slices -- and
   the grid is ksplit = the total item count; every CTA covers all output
   rows of its problem: with more than one item, ws holds one slot of
   m_cap x NC (row-major NC) per item and cnt one counter */
int hq_gemm_skinny(void* stream, const hq_gemm_prob* probs, int nprob, const hq_gemm_term* terms,
                   int* rank, int ksplit, int ncmax, int mode, int max_rows, const int* skip);
int hq_concat(void* stream, const hq_concat_prob* probs, int nprob, const hq_piece* pieces,
              int* rank, int max_rows);
/* cluster >= 2: each problem is factored by a cluster of 2/4/8 CTAs (column
   blocks round-robin, panel factorization overlapped with the trailing
   updates of the previous panel); requires tpanel != NULL */
int hq_qr(void* stream, const hq_qr_prob* probs, int nprob, int* rank, int cluster);
/* grid = nprob x ceil(max_cols / cw): column chunks of X run on separate
   CTAs.  max_rows bounds m over the launch (0: unknown) and sizes the shared
   memory: the chunk (cw = 32, 16 or 8 columns, the widest that fits beside a
   16-reflector panel of max_rows rows) stays in shared memory while the
   panels stream through it by bulk copies; problems taller than what fits
   with cw = 8 (about 1090 rows) run from global memory */
int hq_applyq(void* stream, const hq_applyq_prob* probs, int nprob, int* rank, int max_cols,
              int max_rows);
/* cluster >= 2: one-sided block Jacobi on a cluster of `cluster` CTAs (2, 4
   or 8) per problem, X distributed over their shared memories (DSMEM);
   max_m bounds the row count (<= 512) and selects the lane-group width.
   cluster = 1: one 512-thread CTA per problem.  cluster = 0: small cores,
   one 128-thread CTA per problem with small_doubles doubles of staging
   (>= ((m + 1) & ~1) * n of the largest core, else that core runs from
   global memory), several CTAs per SM */
int hq_svd(void* stream, const hq_svd_prob* probs, int nprob, int* rank, const double* scal,
           int cluster, int max_m, int small_doubles);
/* the same contract as hq_svd (one CTA per problem) by block one-sided
   Jacobi: blocks of 8 columns, per tournament round one warp per block pair
   forms the 16 x 16 Gram on the FP64 tensor pipe, diagonalizes it by
   two-sided Jacobi and applies the accumulated rotation to the 16 columns on
   the tensor pipe.  work must hold ((m + 1) & ~1) * min(m, n) doubles
   (16-byte aligned).  cluster = 2, 4 or 8: each problem on a cluster of that
   many CTAs (the tasks of a round spread over all its warps, one cluster
   barrier per round); 1: one CTA per problem. */
int hq_svd_block(void* stream, const hq_svd_prob* probs, int nprob, int* rank, const double* scal,
                 int cluster);
/* cluster = 1, 2, 4 or 8 CTAs per problem (each holds a column slice in
   shared memory); smem_doubles: dynamic shared memory per CTA in doubles
   (8 + 2 ceil(n/G) + 2 G (m + 5) for the norms and candidate buffers -- always
   required -- plus m (ceil(n/G) + 15) for the slice of an m x n core; slices
   that do not fit are reduced in place in global memory); threads: 256 or 512 */
int hq_qrcp(void* stream, const hq_qrcp_prob* probs, int nprob, int* rank, const double* scal,
            int cluster, int smem_doubles, int threads);
int hq_leaf_gather(void* stream, const hq_leaf_prob* probs, int nprob, const hq_slab* slabs,
                   int* rank, int max_nl);
int hq_leaf_scatter(void* stream, const hq_leaf_prob* probs, int nprob, const hq_slab* slabs,
                    int* rank, int max_nl);
/* copy items (one CTA per item); hq_pack_offsets first rewrites each dst
   (which = 0) or src (which = 1) as base + exclusive prefix sum of rows*cols
   (dense packing with run-time ranks) and stores the total (doubles) in
   total[0] */
int hq_copy(void* stream, const hq_copy_item* items, int nitem, const int* rank);
int hq_pack_offsets(void* stream, hq_copy_item* items, int nitem, const int* rank, double* base,
                    int64_t* total, int which);
int hq_rowblocks(void* stream, const hq_rowblk_prob* probs, int nprob, int* rank, int max_chunks);
/* zero a list of (ptr, count) regions: regions[2i] = ptr, regions[2i+1] = count */
int hq_zero(void* stream, const int64_t* regions, int nregion, int64_t max_count);
/* one step of the two-vector power iteration for ||A||_2 (dense.py:102-141),
   batched: matrix b uses x + 2nb, w + 2nb, g + 4b, scal[2b] (estimate),
   scal[2b+1] (eps * estimate), done[b]; all_done[0] is set once every matrix
   has converged (all_done[1] counts) and gates the batched hq_gemm calls */
int hq_power_step(void* stream, double* x, double* w, const double* g, int n, int ncol,
                  double* scal, double eps, double tol, int* done, int* all_done, int nmat,
                  int final_step);

#ifdef __cplusplus
}
#endif
#endif /* HODLRQR_B200_H */
