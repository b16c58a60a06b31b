"""Launch plan for the batched, device-resident hQR (Algorithm 2).

The recursion of the reference (hqr.py:95-194) is unrolled ONCE per tree
shape into a fixed sequence of batched kernel launches.  Every dimension that
depends on a truncation rank lives in a device int table ("rank slots") and is
read by the kernels at run time, so the sequence never synchronizes with the
host and is captured into a CUDA graph that is replayed for every matrix of
the same shape.  A launch covers all B matrices of a batch and, where the
algorithm has independent blocks (HODLR x dense products, the low-rank update
of a whole subtree), all blocks of a tree level at once.

HBM layout (one persistent region, per matrix b, column-major FP64):
  leafA[j]  n_j x n_j   input leaf -> R (upper) + Y (strict lower)
  leafT[j]  n_j x n_j   T leaf
  per internal node u (children c1, c2; m1 = |c1|, m2 = |c2|, kc = min(m1, m2, kcap)):
  A12U m1 x kc, A12V m2 x kc   a12 = U V^T; after the node's step it holds R's a12
  A21U m2 x kc, A21V m1 x kc   a21; after left-orthogonalization U = Y's a21 L-factor
                               and V = the B_R rows ("slab") fed to the leaves below
  YV21 m1 x kc                 Y's a21 R-factor (transposed): the Y rows of the slab
  T12U m1 x kc, T12V m2 x kc   T's coupling block
  rank slots rA12, rA21, rT12
The compressed column of a leaf (hqr.py:112) is [A_leaf; slabs of every
first-child ancestor-or-self, restricted to the leaf's columns]; the slab
updates of hqr.py:158-159 are applied in place to those V factors.
"""

from __future__ import annotations

import math
import os
from dataclasses import dataclass

import numpy as np

from . import _abi
from .hodlr import PartitionTree

NB = 16          # QR panel width (hq_qr.cu)
TALL_ROWS = 1024  # factor stacks taller than this are QR'd by one-level TSQR
TSQR_CH = 512     # TSQR chunk rows (register-cached panels)
GEMM_TILE = 64   # GEMM output tile (hq_gemm.cu)
FLAT_ITEM_K = int(os.environ.get("HQ_FLAT_ITEM_K", "2048"))   # K rows per work item of the one-launch V^T X kernel
SKINNY_MAX_COLS = 4  # hq_gemm_skinny: outputs with at most this many columns
SVD_MAX_N = 1024

R_PERSIST, R_PHASE, R_APPLY, R_TRUNC, R_SMALL, R_IN, R_OUT, R_SHARED, R_WS = range(9)
LANE_STRIDE = 10   # scratch region of lane l: base + LANE_STRIDE * l (l = 0 main chain)
GEMM_BK = 16       # k-tile of gemm_kernel (hq_gemm.cu BK)
def gv_rows(max_rows):
    """Output rows per CTA of gemv_kernel for a launch whose tallest problem
    has max_rows rows (hq_gemm.cu gv_rows: the same rule)."""
    return 256 if max_rows >= 256 else (128 if max_rows >= 128 else 64)
SPLIT_TARGET = 2 * 2 * 148   # CTAs a K-split launch aims for (148 SMs)


class Buf:
    """Symbolic device address: region + offset in doubles."""
    __slots__ = ("reg", "off")

    def __init__(self, reg, off):
        self.reg, self.off = reg, int(off)

    def __add__(self, k):
        return Buf(self.reg, self.off + int(k))


NULL = None


@dataclass
class Dim:
    cap: int
    ri: int = -1


class Bump:
    """Bump allocator of one region; remembers allocation starts so that any
    address can be mapped back to the allocation that owns it."""

    def __init__(self, reg):
        self.reg, self.top, self.peak = reg, 0, 0
        self.starts = set()
        self.live = []     # (start, size) of the allocations since the last reset
        self.gen = 0       # reset count: instances of different phases differ

    def alloc(self, n):
        n = int(max(n, 1))
        b = Buf(self.reg, self.top)
        self.starts.add(self.top)
        size = (n + 7) // 8 * 8
        self.live.append((self.top, size))
        self.top += size
        self.peak = max(self.peak, self.top)
        return b

    def reset(self):
        self.top = 0
        self.live = []
        self.gen += 1

    def instance(self, off):
        """(start, size, generation) of the live allocation holding off."""
        import bisect
        i = bisect.bisect_right(self.live, (off, float("inf"))) - 1
        s, n = self.live[max(i, 0)]
        return s, n, self.gen

    def finalize(self):
        self.sorted = sorted(self.starts)

    def owner(self, off):
        import bisect
        i = bisect.bisect_right(self.sorted, off) - 1
        return self.sorted[max(i, 0)]


class Tree:
    """Node geometry of a PartitionTree: level l, index j."""

    def __init__(self, tree: PartitionTree):
        self.L = tree.level
        self.leaf_sizes = [int(s) for s in tree.leaf_sizes]
        self.size, self.off = {}, {}
        offs = np.concatenate([[0], np.cumsum(self.leaf_sizes)])
        for l in range(self.L + 1):
            span = 1 << (self.L - l)
            for j in range(1 << l):
                a, b = j * span, (j + 1) * span
                self.off[(l, j)] = int(offs[a])
                self.size[(l, j)] = int(offs[b] - offs[a])
        self.n = int(offs[-1])

    def is_leaf(self, v):
        return v[0] == self.L

    @staticmethod
    def children(v):
        return (v[0] + 1, 2 * v[1]), (v[0] + 1, 2 * v[1] + 1)

    @staticmethod
    def parent(v):
        return (v[0] - 1, v[1] // 2)

    def internal_nodes(self, v):
        """Internal nodes of the subtree rooted at v (level order)."""
        out = []
        for l in range(v[0], self.L):
            span = 1 << (l - v[0])
            out += [(l, j) for j in range(v[1] * span, (v[1] + 1) * span)]
        return out

    def leaves(self, v):
        span = 1 << (self.L - v[0])
        return [(self.L, j) for j in range(v[1] * span, (v[1] + 1) * span)]

    def ancestors(self, v, stop):
        """Proper ancestors of v up to and including stop (nearest first)."""
        out, u = [], v
        while u != stop:
            u = self.parent(u)
            out.append(u)
        return out

    def slab_owners(self, v):
        """First-child ancestors-or-self w of v (nearest first): their parent's
        a21 block was the B of w's structured column (hqr.py:127)."""
        out, w = [], v
        while w[0] > 0:
            if w[1] % 2 == 0:
                out.append(w)
            w = self.parent(w)
        return out


def level_cap(kcap, level):
    """Rank capacity of the blocks at a tree level (root = 0): kcap itself, or
    entry `level` of a per-level profile (the last entry for deeper levels).
    The factors' ranks grow with the depth (roughly input rank x level), so a
    profile stores the large top-level blocks at their small ranks."""
    if isinstance(kcap, (int, np.integer)):
        return int(kcap)
    return int(kcap[min(level, len(kcap) - 1)])


class Layout:
    """Persistent per-matrix storage (see module docstring)."""

    def __init__(self, tree: Tree, batch: int, kcap: int, bump: Bump, slots):
        self.t, self.B, self.kcap = tree, batch, kcap
        self.kc = {}
        for u in self._all_internal():
            c1, c2 = tree.children(u)
            self.kc[u] = max(1, min(tree.size[c1], tree.size[c2], level_cap(kcap, u[0])))
        self.m = []
        for b in range(batch):
            d = {"leafA": {}, "leafT": {}, "A12U": {}, "A12V": {}, "A21U": {}, "A21V": {},
                 "YV21": {}, "T12U": {}, "T12V": {}, "rA12": {}, "rA21": {}, "rT12": {}}
            for j, nl in enumerate(tree.leaf_sizes):
                d["leafA"][(tree.L, j)] = bump.alloc(nl * nl)
                d["leafT"][(tree.L, j)] = bump.alloc(nl * nl)
            for u in self._all_internal():
                c1, c2 = tree.children(u)
                m1, m2, kc = tree.size[c1], tree.size[c2], self.kc[u]
                for name, rows in (("A12U", m1), ("A12V", m2), ("A21U", m2), ("A21V", m1),
                                   ("YV21", m1), ("T12U", m1), ("T12V", m2)):
                    d[name][u] = bump.alloc(rows * kc)
                for name in ("rA12", "rA21", "rT12"):
                    d[name][u] = slots.take()
            n = tree.n
            d["X"], d["Y"], d["W"] = bump.alloc(2 * n), bump.alloc(2 * n), bump.alloc(2 * n)
            self.m.append(d)
        # power-iteration buffers must be contiguous with stride 2n for the batched kernel
        self.power_stride = None

    def _all_internal(self):
        return self.t.internal_nodes((0, 0)) if self.t.L > 0 else []


class Slots:
    def __init__(self):
        self.n = 0

    def take(self, k=1):
        s = self.n
        self.n += k
        return s


class Builder:
    """Unrolls hqr_rec into batched ops with symbolic addresses."""

    def __init__(self, tree: PartitionTree, batch: int, eps: float, absolute: bool,
                 kcap: int = 512, max_iter: int = 50, tol: float = 1e-3, n_side: int = 3,
                 io: bool = True, track: bool = False, root_b=None, root_c: int = 0):
        """io=False: no factorization I/O streams (operator plans build
        their own, operators.py).  track: record per op the allocation
        instances it reads / writes (multi-GPU partitioning, distributed.py).
        root_b = (p, k), root_c = r2: the general structured column
        [A; B; C] of hqr_rec (hqr.py:38-56, 95-194) -- B = L R (p x n, rank
        <= k) and r2 dense coupling rows C below the HODLR block; they enter
        as two more slabs of every compressed column, outermost."""
        self.track = bool(track)
        self.cur_level = -1
        self.root_b = (int(root_b[0]), int(root_b[1])) if root_b is not None and root_b[0] > 0 else None
        self.root_c = int(root_c)
        self.tree = Tree(tree)
        self.B = batch
        self.eps, self.absolute = float(eps), bool(absolute)
        self.max_iter, self.tol = max_iter, tol
        self.bumps = {}
        for r in range(9):
            self.bump(r)
        self.n_cnt = 0     # split-K arrival counters (device ints, self-resetting)
        self.lane = 0
        self.n_side = n_side
        self._rr = 0
        self.slots = Slots()
        self.flag_slot = self.slots.take()
        self.power_done = self.slots.take(batch)
        self.all_done = self.slots.take(2)
        self.lay = Layout(self.tree, batch, kcap, self.bumps[R_PERSIST], self.slots)
        if self.root_b is not None or self.root_c:
            n = self.tree.n
            P = self.bumps[R_PERSIST]
            for d in self.lay.m:
                if self.root_b is not None:
                    p_, k_ = self.root_b
                    kb = max(1, min(p_, k_, n))
                    d["kB"], d["kBin"] = kb, max(1, k_)
                    d["RB_Lin"], d["RB_Rin"] = P.alloc(p_ * d["kBin"]), P.alloc(n * d["kBin"])
                    d["RB_L"], d["RB_V"], d["RB_Y"] = P.alloc(p_ * kb), P.alloc(n * kb), P.alloc(n * kb)
                    d["rBin"], d["rB"] = self.slots.take(), self.slots.take()
                if self.root_c:
                    d["RC_V"], d["RC_Y"] = P.alloc(n * self.root_c), P.alloc(n * self.root_c)
                    d["rC"] = self.slots.take()
        # power buffers: contiguous [X_b], [W_b] with stride 2n, G with stride 4
        n = self.tree.n
        self.PX = self.bumps[R_PERSIST].alloc(2 * n * batch)
        self.PY = self.bumps[R_PERSIST].alloc(2 * n * batch)
        self.PW = self.bumps[R_PERSIST].alloc(2 * n * batch)
        self.PG = self.bumps[R_PERSIST].alloc(4 * batch)
        self.ops = []
        self.in_items, self.out_items = self._io_items() if io else ([], [])

    def _io_items(self):
        """Compact input/output streams: (arena Buf, rows, Dim cols) in a fixed
        order; offsets are prefix sums of rows*cols with run-time ranks."""
        t, lay = self.tree, self.lay
        ins, outs = [], []
        nin = nout = 0
        for b in range(self.B):
            d = lay.m[b]
            for lf in t.leaves((0, 0)):
                nl = t.size[lf]
                ins.append((d["leafA"][lf], nl, Dim(nl)))
                # R (upper), Y (unit lower) and T (upper) leaves, masked on the device
                outs.append((d["leafA"][lf], nl, Dim(nl), 1))
                outs.append((d["leafA"][lf], nl, Dim(nl), 2))
                outs.append((d["leafT"][lf], nl, Dim(nl), 1))
            for u in (t.internal_nodes((0, 0)) if t.L > 0 else []):
                c1, c2 = t.children(u)
                m1, m2, kc = t.size[c1], t.size[c2], lay.kc[u]
                ins += [(d["A12U"][u], m1, Dim(kc, d["rA12"][u])), (d["A12V"][u], m2, Dim(kc, d["rA12"][u])),
                        (d["A21U"][u], m2, Dim(kc, d["rA21"][u])), (d["A21V"][u], m1, Dim(kc, d["rA21"][u]))]
                outs += [(d["A12U"][u], m1, Dim(kc, d["rA12"][u]), 0), (d["A12V"][u], m2, Dim(kc, d["rA12"][u]), 0),
                         (d["A21U"][u], m2, Dim(kc, d["rA21"][u]), 0), (d["YV21"][u], m1, Dim(kc, d["rA21"][u]), 0),
                         (d["T12U"][u], m1, Dim(kc, d["rT12"][u]), 0), (d["T12V"][u], m2, Dim(kc, d["rT12"][u]), 0)]
            n = t.n
            if self.root_b is not None:
                p_ = self.root_b[0]
                ins += [(d["RB_Lin"], p_, Dim(d["kBin"], d["rBin"])), (d["RB_Rin"], n, Dim(d["kBin"], d["rBin"]))]
                outs += [(d["RB_L"], p_, Dim(d["kB"], d["rB"]), 0), (d["RB_Y"], n, Dim(d["kB"], d["rB"]), 0)]
            if self.root_c:
                ins += [(d["RC_V"], n, Dim(self.root_c))]
                outs += [(d["RC_Y"], n, Dim(self.root_c), 0)]
        self.bumps[R_IN].alloc(sum(r * c.cap for _, r, c in ins))
        self.bumps[R_OUT].alloc(sum(r * c.cap for _, r, c, _ in outs))
        return ins, outs

    # ------------------------------------------------------------ primitives
    def bump(self, reg):
        b = self.bumps.get(reg)
        if b is None:
            b = self.bumps[reg] = Bump(reg)
        return b

    def lane_bump(self, base):
        return self.bump(base + LANE_STRIDE * self.lane)

    def _ph(self, n):
        return self.lane_bump(R_PHASE).alloc(n)

    def _sh(self, n):
        """Values read by several lanes: never reused (R_SHARED)."""
        return self.bumps[R_SHARED].alloc(n)

    def side_lane(self):
        """Round-robin side lane for work off the critical chain; its scratch
        regions are reset (the previous job of the lane precedes it in stream
        order)."""
        if self.n_side <= 0:
            return 0
        self._rr = self._rr % self.n_side + 1
        return self._rr

    def op(self, kind, probs, extra=None):
        extra = dict(extra or {})
        extra["lane"] = self.lane
        extra["level"] = self.cur_level
        if kind == "qr" and "cluster" not in extra:
            force = os.environ.get("HQ_QR_CLUSTER_" + str(extra.get("role", "")).upper())
            extra["cluster"] = int(force) if force else qr_cluster(probs)
        if self.track:
            # the live allocation instances this op touches, resolved now
            # (scratch regions are reused later): the units distributed.py
            # moves between GPUs
            extra["_inst"] = op_resources(self, kind, probs, extra, mem=self._inst_key)
        self.ops.append((kind, probs, extra))

    def _inst_key(self, buf):
        if buf is None:
            return None
        s, n, g = self.bumps[buf.reg].instance(buf.off)
        return ("i", buf.reg, s, n, g)

    def gemm(self, probs, skip=None, ksplit=1):
        """probs: list of (c, ldc, Dim m, Dim n, beta, [terms]); term =
        (a, lda, ta, mask_a, b, ldb, tb, mask_b, Dim k, alpha)."""
        if not probs:
            return
        tiles = max(math.ceil(p[2].cap / GEMM_TILE) * math.ceil(p[3].cap / GEMM_TILE) for p in probs)
        if tiles <= 0:
            return
        # few output tiles: 32 x 32 tiles put 4x the CTAs (SMs) on the product
        tile = GEMM_TILE
        if tiles * len(probs) * ksplit < 96:
            tile = 32
            tiles = max(math.ceil(p[2].cap / 32) * math.ceil(p[3].cap / 32) for p in probs)
        ncmax = max(p[3].cap for p in probs)
        mmax = max(p[2].cap for p in probs)
        kmax = max(max(t[8].cap for t in p[5]) for p in probs)
        # outputs of <= 4 columns (power iteration): the skinny kernels --
        # threads along K for long K, one thread per output row otherwise
        skinny = ncmax <= SKINNY_MAX_COLS
        # skinny products stream their operands (mode 2: coalesced per term
        # layout, per-problem K slices; 3 / 4 when every term is A / A^T);
        # modes 0/1 remain in the ABI
        tas = {t[2] for p in probs for t in p[5]}
        mode = 3 if tas == {0} else (4 if tas == {1} else 2)
        if ksplit > 1:
            # split K only as far as the launch needs CTAs: about SPLIT_TARGET
            # of them (two waves of two per SM); a batch that already fills
            # the GPU keeps whole K (no partial-sum traffic or workspace)
            blocks = math.ceil(mmax / gv_rows(mmax)) if skinny else tiles
            ksplit = max(1, min(ksplit, math.ceil(SPLIT_TARGET / (len(probs) * blocks))))
        ex = dict(tiles=tiles, ksplit=ksplit, skip=skip, skinny=skinny, ncmax=ncmax,
                  mode=mode, max_rows=mmax, tile=tile)
        if ksplit > 1:
            # deterministic K split: per problem, slots for the partial sums of
            # every (output block, slice) and one arrival counter per block,
            # sized from the capacities exactly as the kernels size them
            slots = []
            for p in probs:
                if skinny:
                    ktot = sum(t[8].cap for t in p[5])
                    ks = min(ksplit, max(1, ktot // 512))
                    blocks, per = math.ceil(p[2].cap / gv_rows(mmax)), gv_rows(mmax) * (2 if ncmax <= 2 else 4)
                else:
                    nkt = sum(math.ceil(t[8].cap / GEMM_BK) for t in p[5])
                    ks = min(ksplit, max(1, nkt // 8))
                    blocks = math.ceil(p[2].cap / tile) * math.ceil(p[3].cap / tile)
                    per = tile * tile
                slots.append((blocks, ks, per))
            self._split_ws(ex, slots)
        self.op("gemm", probs, ex)

    def take_cnt(self, k):
        c = self.n_cnt
        self.n_cnt += int(k)
        return c

    def _split_ws(self, ex, slots):
        """slots[i] = (output blocks, slices, doubles per slot) of problem i:
        workspace in the lane's R_WS region (private to this op; the lane's
        next op reuses it) and arrival counters, recorded in the op's extra."""
        wsb = self.lane_bump(R_WS)
        wsb.reset()
        ws, cnt = [], []
        for blocks, ks, per in slots:
            if ks <= 1:
                ws.append(None)
                cnt.append(-1)
                continue
            ws.append(wsb.alloc(blocks * ks * per))
            cnt.append(self.take_cnt(blocks))
        ex["ws"], ex["cnt"] = ws, cnt

    def zero(self, regions):
        if regions:
            self.op("zero", regions)

    # ------------------------------------------------------------ HODLR x dense
    def _fset(self, fs, b):
        d = self.lay.m[b]
        if fs == "A":
            return (("a12", d["A12U"], d["A12V"], d["rA12"]), ("a21", d["A21U"], d["A21V"], d["rA21"])), d["leafA"], 0
        if fs == "Y":
            return (("a21", d["A21U"], d["YV21"], d["rA21"]),), d["leafA"], 2
        if fs == "T":
            return (("a12", d["T12U"], d["T12V"], d["rT12"]),), d["leafT"], 1
        if fs == "R":
            return (("a12", d["A12U"], d["A12V"], d["rA12"]),), d["leafA"], 1
        raise ValueError(fs)

    def happly(self, v, fs, trans, xs, outs, nc, alpha=1.0, beta=0.0, skip=None):
        """out_b = alpha * op(F_b|subtree v) X_b + beta * out_b for every matrix b.
        xs/outs: lists of (Buf, ld); nc: (cap, [ri_b]).  Two launches:
        phase 1 tmp_blk = V^T X (U^T X), phase 2 per leaf: leaf term + sum of
        U tmp (V tmp) over the blocks covering the leaf (arith.py:35-64)."""
        t = self.tree
        v0 = t.off[v]
        ncap, nris = nc
        ab = self.lane_bump(R_APPLY)
        ab.reset()
        p1, p2, kmax = [], [], 0
        tmp = {}
        for b in range(self.B):
            blocks, leafbuf, mask = self._fset(fs, b)
            X, ldx = xs[b]
            for u in t.internal_nodes(v) if not t.is_leaf(v) else []:
                c1, c2 = t.children(u)
                r1, r2 = t.off[c1] - v0, t.off[c2] - v0
                m1, m2 = t.size[c1], t.size[c2]
                kc = self.lay.kc[u]
                for kind, U, V, R in blocks:
                    rows0, nrows, cols0, ncols = (r1, m1, r2, m2) if kind == "a12" else (r2, m2, r1, m1)
                    buf = ab.alloc(kc * ncap)
                    tmp[(b, u, kind)] = buf
                    if trans:   # tmp = U^T X[rows]
                        term = (U[u], nrows, 1, 0, X + rows0, ldx, 0, 0, Dim(nrows), 1.0)
                        kmax = max(kmax, nrows)
                    else:       # tmp = V^T X[cols]
                        term = (V[u], ncols, 1, 0, X + cols0, ldx, 0, 0, Dim(ncols), 1.0)
                        kmax = max(kmax, ncols)
                    p1.append((buf, kc, Dim(kc, R[u]), Dim(ncap, nris[b]), 0.0, [term]))
        if p1 and ncap <= SKINNY_MAX_COLS:
            # streaming V^T X products of every level in one launch (mode 5):
            # each problem gets ceil-ish K/512 work items (<= 32), listed by
            # prefix sums; split problems sum their slices deterministically
            items, tot, slots = [], 0, []
            nc = 2 if ncap <= 2 else 4
            for prob in p1:
                items.append(tot)
                it = max(1, min(32, sum(t[8].cap for t in prob[5]) // FLAT_ITEM_K))
                tot += it
                slots.append((1, it, prob[2].cap * nc))
            ex = dict(tiles=1, ksplit=tot, skip=skip, skinny=True, ncmax=ncap, mode=5,
                      max_rows=max(pr[2].cap for pr in p1), tile=64, items=items)
            self._split_ws(ex, slots)
            self.op("gemm", p1, ex)
        elif p1:
            ksplit = 1
            if kmax >= 1024:
                ksplit = min(32, kmax // 256)   # per problem the kernel uses <= nktiles/8 slices
            self.gemm(p1, skip=skip, ksplit=ksplit)
        for b in range(self.B):
            blocks, leafbuf, mask = self._fset(fs, b)
            X, ldx = xs[b]
            O, ldo = outs[b]
            bd = {kind: (U, V, R) for kind, U, V, R in blocks}
            for lf in t.leaves(v):
                o, nl = t.off[lf] - v0, t.size[lf]
                terms = [(leafbuf[lf], nl, 1 if trans else 0, mask, X + o, ldx, 0, 0, Dim(nl), alpha)]
                for u in t.ancestors(lf, v) if lf != v else []:
                    c1, c2 = t.children(u)
                    in_c1 = t.off[lf] < t.off[c2]
                    if trans:
                        kind = "a21" if in_c1 else "a12"
                        base = t.off[c1] if in_c1 else t.off[c2]
                    else:
                        kind = "a12" if in_c1 else "a21"
                        base = t.off[c1] if in_c1 else t.off[c2]
                    if kind not in bd:
                        continue
                    U, V, R = bd[kind]
                    F = V if trans else U
                    ldf = t.size[c1] if in_c1 else t.size[c2]
                    terms.append((F[u] + (t.off[lf] - base), ldf, 0, 0, tmp[(b, u, kind)],
                                  self.lay.kc[u], 0, 0, Dim(self.lay.kc[u], R[u]), alpha))
                p2.append((O + o, ldo, Dim(nl), Dim(ncap, nris[b]), beta, terms))
        self.gemm(p2, skip=skip)

    # ------------------------------------------------------------ T_eps
    def trunc(self, probs):
        """Batched recompression (core.py:239-258) of stacked low-rank sums.
        prob = dict(m, n, L=[(Buf, ld, Dim, alpha)], R=[...V-form...],
        eps_slot, eps_scale, U=(Buf, ld), V=(Buf, ld), cap, rank_ri)."""
        if not probs:
            return
        z = self.lane_bump(R_TRUNC)
        z.reset()
        cat, qr, stack, qrs, gm_c, qrc, svd, apq, unstack, apq2, gm_m, gm_v = ([] for _ in range(12))
        pivot = PIVOT_CORE
        maxrows, maxch = 0, 0

        def factor_side(W, rows, kcap, kri, tau, tp):
            """QR of a factor stack; tall stacks (rows > TALL_ROWS) go through a
            one-level TSQR: chunk QRs in parallel, their R's stacked densely
            (hq_rowblocks), QR of the stack.  Returns the R source (buf, ld)
            and the chunk description for the Q application."""
            nonlocal maxch
            if rows <= TALL_ROWS:
                qr.append((W, tau, tp, None, rows, 0, Dim(rows), Dim(kcap, kri)))
                return (W, rows), None
            nch = math.ceil(rows / TSQR_CH)
            maxch = max(maxch, nch)
            npan = max(1, math.ceil(kcap / NB))
            chunks = []
            for c in range(nch):
                rc = min(TSQR_CH, rows - c * TSQR_CH)
                tc, pc = z.alloc(kcap), z.alloc(npan * NB * NB)
                qr.append((W + c * TSQR_CH, tc, pc, None, rows, 0, Dim(rc), Dim(kcap, kri)))
                chunks.append((c * TSQR_CH, rc, tc, pc))
            srows = nch * min(TSQR_CH, kcap)
            S, tS, pS = z.alloc(srows * kcap), z.alloc(kcap), z.alloc(npan * NB * NB)
            ms = self.slots.take()
            stack.append((S, W, srows, rows, TSQR_CH, rows, Dim(kcap, kri), Dim(0), ms, 0))
            qrs.append((S, tS, pS, None, srows, 0, Dim(srows, ms), Dim(kcap, kri)))
            return (S, srows), dict(S=S, srows=srows, tS=tS, pS=pS, ms=ms, chunks=chunks, W=W, rows=rows)

        for p in probs:
            m, n, cap = p["m"], p["n"], p["cap"]
            kcap = sum(d.cap for _, _, d, _ in p["L"])
            assert kcap == sum(d.cap for _, _, d, _ in p["R"]), "L/R piece capacities differ"
            k1, k2 = min(m, kcap), min(n, kcap, SVD_MAX_N)
            WL, WR, WRc = z.alloc(m * kcap), z.alloc(n * kcap), z.alloc(n * kcap)
            tauL, tauR = z.alloc(kcap), z.alloc(kcap)
            npan = max(1, math.ceil(kcap / NB))
            tpL, tpR = z.alloc(npan * NB * NB), z.alloc(npan * NB * NB)
            C, Uk, Mm = z.alloc(k1 * k2), z.alloc(k1 * cap), z.alloc(kcap * cap)
            Xw = z.alloc((k1 + 1) // 2 * 2 * min(k1, k2))
            tauC = z.alloc(min(k1, k2))
            tpC = z.alloc(max(1, math.ceil(min(k1, k2) / NB)) * NB * NB)
            kL, kR = self.slots.take(), self.slots.take()
            cat.append((WL, None, m, kL, p["L"]))
            cat.append((WR, WRc, n, kR, p["R"]))
            maxrows = max(maxrows, m, n)
            (R1, ld1), tsL = factor_side(WL, m, kcap, kL, tauL, tpL)
            (R2, ld2), _ = factor_side(WR, n, kcap, kR, tauR, tpR)
            # C^T = R2 R1^T (masks: upper on the stored R factors).  Its
            # column-pivoted QR, stopped where the remaining columns are below
            # 1e-3 of the threshold (Frobenius norm), leaves r rows of R; the
            # Jacobi runs on X = (those rows)^T (k1 x r): graded, r close to
            # the rank instead of min(k1, k2) columns, few sweeps.  Without
            # pivoting (HQ_PIVOT_CORE=0): X = R_c^T of the plain QR.
            gm_c.append((C, k2, Dim(k2, kR), Dim(k1, kL), 0.0,
                         [(R2, ld2, 0, 1, R1, ld1, 1, 1, Dim(kcap, kL), 1.0)]))
            if pivot:
                rC = self.slots.take()
                qrc.append((C, k2, Dim(k2, kR), Dim(k1, kL), rC, p["eps_slot"], CORE_STOP * p["eps_scale"]))
                svd.append((C, Uk, Xw, k2, k1, Dim(k1, kL), Dim(min(k1, k2), rC), cap, p["rank_ri"],
                            p.get("flag", self.flag_slot), p["eps_slot"], p["eps_scale"], 2))
            else:
                qrc.append((C, tauC, tpC, None, k2, 0, Dim(k2, kR), Dim(k1, kL)))
                svd.append((C, Uk, Xw, k2, k1, Dim(k1, kL), Dim(k2, kR), cap, p["rank_ri"],
                            p.get("flag", self.flag_slot), p["eps_slot"], p["eps_scale"], 1))
            U, ldu = p["U"]
            V, ldv = p["V"]
            if tsL is None:
                apq.append((WL, tauL, tpL, U, Uk, m, ldu, k1, Dim(m), Dim(kcap, kL),
                            Dim(cap, p["rank_ri"]), Dim(k1, kL), 0))
            else:
                # L_out = blockdiag(Q_c) Q_S [U_k; 0]
                srows = tsL["srows"]
                Z = z.alloc(srows * cap)
                apq.append((tsL["S"], tsL["tS"], tsL["pS"], Z, Uk, srows, srows, k1,
                            Dim(srows, tsL["ms"]), Dim(kcap, kL), Dim(cap, p["rank_ri"]),
                            Dim(k1, kL), 0))
                unstack.append((Z, U, srows, ldu, TSQR_CH, m, Dim(kcap, kL), Dim(cap, p["rank_ri"]), -1, 1))
                for (r0, rc, tc, pc) in tsL["chunks"]:
                    apq2.append((WL + r0, tc, pc, U + r0, None, m, ldu, 0, Dim(rc), Dim(kcap, kL),
                                 Dim(cap, p["rank_ri"]), Dim(0), 0))
            # Mm = R1^T U_k ; V = WRc Mm  (right factor = P^T L_out, no 1/sigma)
            gm_m.append((Mm, kcap, Dim(kcap, kL), Dim(cap, p["rank_ri"]), 0.0,
                         [(R1, ld1, 1, 1, Uk, k1, 0, 0, Dim(k1, kL), 1.0)]))
            gm_v.append((V, ldv, Dim(n), Dim(cap, p["rank_ri"]), 0.0,
                         [(WRc, n, 0, 0, Mm, kcap, 0, 0, Dim(kcap, kL), 1.0)]))
        self.op("concat", cat, dict(max_rows=maxrows))
        self.op("qr", qr, dict(role="stack"))
        if stack:
            self.op("rowblk", stack, dict(max_chunks=maxch))
            self.op("qr", qrs, dict(role="tsqr"))
        self.gemm(gm_c)
        if pivot:
            G, smem, threads = qrcp_launch(len(qrc), max(p[2].cap for p in qrc), max(p[3].cap for p in qrc))
            self.op("qrcp", qrc, dict(cluster=G, smem=smem, threads=threads))
        else:
            self.op("qr", qrc, dict(role="core"))
        self.op("svd", svd, svd_cluster(svd))
        self.op("applyq", apq, dict(max_cols=max(p[10].cap for p in apq), max_rows=max(p[8].cap for p in apq)))
        if unstack:
            self.op("rowblk", unstack, dict(max_chunks=maxch))
            self.op("applyq", apq2, dict(max_cols=max(p[10].cap for p in apq2), max_rows=max(p[8].cap for p in apq2)))
        self.gemm(gm_m)
        self.gemm(gm_v)

    # ------------------------------------------------------------ algorithm
    def slabs(self, b, v, sub):
        """(V-rows, Y-rows, ld, rank slot, kc) of every slab owner of v,
        restricted to the rows of node `sub` (nearest first)."""
        d, t = self.lay.m[b], self.tree
        out = []
        for w in t.slab_owners(v):
            pw = t.parent(w)
            o = t.off[sub] - t.off[w]
            out.append((d["A21V"][pw] + o, d["YV21"][pw] + o, t.size[w], d["rA21"][pw],
                        self.lay.kc[pw]))
        # the structured column's own B and C rows (hqr_rec on [A; B; C]):
        # outermost, B before C (hqr.py:112, 127)
        o = t.off[sub]
        if self.root_b is not None:
            out.append((d["RB_V"] + o, d["RB_Y"] + o, t.n, d["rB"], d["kB"]))
        if self.root_c:
            out.append((d["RC_V"] + o, d["RC_Y"] + o, t.n, d["rC"], self.root_c))
        return out

    def first_col(self, v):
        """Does v's structured column have its own B block (the slab nearest
        first in slabs())?  First children: their parent's a21 (hqr.py:127);
        the root: the column's B (hqr_rec); second children: none (hqr.py:163)."""
        return (v[0] > 0 and v[1] % 2 == 0) or (v == (0, 0) and self.root_b is not None)

    def power_iteration(self, n):
        """||A||_2 by the two-vector power method (dense.py:102-141); start
        vectors are uploaded by the host (input independent)."""
        skip = self.all_done
        for it in range(self.max_iter):
            xs = [(self.PX + 2 * n * b, n) for b in range(self.B)]
            ys = [(self.PY + 2 * n * b, n) for b in range(self.B)]
            ws = [(self.PW + 2 * n * b, n) for b in range(self.B)]
            self.happly((0, 0), "A", False, xs, ys, (2, [-1] * self.B), skip=skip)
            g = [(self.PG + 4 * b, 2, Dim(2), Dim(2), 0.0,
                  [(self.PY + 2 * n * b, n, 1, 0, self.PY + 2 * n * b, n, 0, 0, Dim(n), 1.0)])
                 for b in range(self.B)]
            gs = min(64, max(1, n // 256))
            self.gemm(g, skip=skip, ksplit=gs)
            self.happly((0, 0), "A", True, ys, ws, (2, [-1] * self.B), skip=skip)
            self.op("power", None, dict(n=n, final=int(it == self.max_iter - 1)))

    def build(self):
        t = self.tree
        # restore the input from the compact staging buffer (first op)
        self.op("pack_copy", self.in_items, dict(which=1, base=Buf(R_IN, 0), total=0))
        if not self.absolute:
            self.power_iteration(t.n)
        # the structured column's B: left-orthogonalized (hqr.py:101; core.py:
        # 229-236) by a truncation at threshold 0 (SVD basis, same product)
        if self.root_b is not None:
            probs = []
            for b in range(self.B):
                d = self.lay.m[b]
                p_ = self.root_b[0]
                probs.append(dict(m=p_, n=t.n, L=[(d["RB_Lin"], p_, Dim(d["kBin"], d["rBin"]), 1.0)],
                                  R=[(d["RB_Rin"], t.n, Dim(d["kBin"], d["rBin"]), 1.0)],
                                  eps_slot=-1, eps_scale=0.0, U=(d["RB_L"], p_), V=(d["RB_V"], t.n),
                                  cap=d["kB"], rank_ri=d["rB"]))
            self.trunc(probs)
        # left-orthogonalize the a21 blocks of the leftmost spine: the only B
        # blocks never recompressed by an earlier update (core.py:229-236)
        if t.L > 0:
            spine = [(l, 0) for l in range(t.L)]
            probs = []
            for b in range(self.B):
                d = self.lay.m[b]
                for u in spine:
                    c1, c2 = t.children(u)
                    kc = self.lay.kc[u]
                    probs.append(dict(m=t.size[c2], n=t.size[c1],
                                      L=[(d["A21U"][u], t.size[c2], Dim(kc, d["rA21"][u]), 1.0)],
                                      R=[(d["A21V"][u], t.size[c1], Dim(kc, d["rA21"][u]), 1.0)],
                                      eps_slot=-1, eps_scale=0.0, U=(d["A21U"][u], t.size[c2]),
                                      V=(d["A21V"][u], t.size[c1]), cap=kc, rank_ri=d["rA21"][u]))
            self.trunc(probs)
        self.rec((0, 0))
        # compact the factors for one device->host copy (last op)
        self.op("pack_copy", self.out_items, dict(which=0, base=Buf(R_OUT, 0), total=1))
        for b in self.bumps.values():
            b.finalize()
        return self

    def eps_slot(self, b):
        return 2 * b + 1

    def rec(self, v):
        t = self.tree
        if t.is_leaf(v):
            self.leaf_qr(v)
            return
        c1, c2 = t.children(v)
        self.rec(c1)
        self.s_phase(v)
        self.rec(c2)
        self.t_phase(v)

    def leaf_qr(self, v):
        """Compressed leaf column -> block_qr (hqr.py:110-119)."""
        t = self.tree
        self.cur_level = v[0]
        self.lane = 0
        self.lane_bump(R_PHASE).reset()
        nl = t.size[v]
        if nl > 384:
            raise ValueError("leaf blocks larger than 384 are not supported by the leaf QR kernel")
        gat, qr = [], []
        for b in range(self.B):
            d = self.lay.m[b]
            sl = self.slabs(b, v, v)
            mcap = nl + sum(s[4] for s in sl)
            panel = self._ph(mcap * nl)
            tau = self._ph(nl)
            # panel T's + the cluster kernel's full-T merge scratch (2 x nl x NB)
            tp = self._ph(math.ceil(nl / NB) * NB * NB + 2 * nl * NB)
            m_ri = self.slots.take()
            gat.append((d["leafA"][v], panel, nl, mcap, [(s[0], s[1], s[2], s[2], s[3]) for s in sl],
                        m_ri))
            qr.append((panel, tau, tp, d["leafT"][v], mcap, nl, Dim(mcap, m_ri), Dim(nl)))
        self.op("leaf_gather", gat, dict(max_nl=nl))
        self.op("qr", qr, dict(role="leaf"))
        self.op("leaf_scatter", gat, dict(max_nl=nl))

    def s_phase(self, v):
        """hqr.py:134-159: S~ (one recompression of the four-term sum), S, the
        R coupling block, and the update of the second block column."""
        t = self.tree
        self.cur_level = v[0]
        self.lane = 0
        self.lane_bump(R_PHASE).reset()
        c1, c2 = t.children(v)
        m1, m2 = t.size[c1], t.size[c2]
        kc = self.lay.kc[v]
        B = range(self.B)
        D = [self.lay.m[b] for b in B]
        cap_s = kc
        tmp1 = [self._ph(m1 * kc) for _ in B]
        tmp2 = [self._ph(m2 * kc) for _ in B]
        # t1 = Y(c1)^T A12.L ; t2 = A(c2)^T QB
        self.happly(c1, "Y", True, [(D[b]["A12U"][v], m1) for b in B], [(tmp1[b], m1) for b in B],
                    (kc, [D[b]["rA12"][v] for b in B]))
        self.happly(c2, "A", True, [(D[b]["A21U"][v], m2) for b in B], [(tmp2[b], m2) for b in B],
                    (kc, [D[b]["rA21"][v] for b in B]))
        # S~ = T(T(T(t1 + t2) + t3) + t4): the left-to-right sum of hqr.py:143-147,
        # truncating after every addition exactly like the reference (for
        # ill-conditioned A the computed R is sensitive to this sequence)
        own = [[], []]
        rest = [[], []]
        for b in B:
            sl1, sl2 = self.slabs(b, v, c1), self.slabs(b, v, c2)
            first = self.first_col(v)
            own[0].append(sl1[:1] if first else [])
            own[1].append(sl2[:1] if first else [])
            rest[0].append(sl1[1:] if first else sl1)
            rest[1].append(sl2[1:] if first else sl2)
        cur_L = [[(tmp1[b], m1, Dim(kc, D[b]["rA12"][v]), 1.0)] for b in B]
        cur_R = [[(D[b]["A12V"][v], m2, Dim(kc, D[b]["rA12"][v]), 1.0)] for b in B]
        adds = [
            ([[(D[b]["YV21"][v], m1, Dim(kc, D[b]["rA21"][v]), 1.0)] for b in B],
             [[(tmp2[b], m2, Dim(kc, D[b]["rA21"][v]), 1.0)] for b in B]),
            ([[(yc1, ld, Dim(kw, ri), 1.0) for (vc1, yc1, ld, ri, kw) in own[0][b]] for b in B],
             [[(vc2, ld, Dim(kw, ri), 1.0) for (vc2, yc2, ld, ri, kw) in own[1][b]] for b in B]),
            ([[(yc1, ld, Dim(kw, ri), 1.0) for (vc1, yc1, ld, ri, kw) in rest[0][b]] for b in B],
             [[(vc2, ld, Dim(kw, ri), 1.0) for (vc2, yc2, ld, ri, kw) in rest[1][b]] for b in B]),
        ]
        # a statically empty term (no B block, no ancestor slabs) makes the
        # reference re-truncate an already truncated sum: T(T(x)) = T(x), skip
        adds = [ad for i, ad in enumerate(adds) if i == 0 or any(ad[0][b] for b in B)]
        for step, (addL, addR) in enumerate(adds):
            last = step == len(adds) - 1
            outL = [self._ph(m1 * cap_s) for _ in B]
            outR = [(self._sh if last else self._ph)(m2 * cap_s) for _ in B]
            kk = [self.slots.take() for _ in B]
            probs = []
            for b in B:
                probs.append(dict(m=m1, n=m2, L=cur_L[b] + addL[b], R=cur_R[b] + addR[b],
                                  eps_slot=self.eps_slot(b), eps_scale=1.0,
                                  U=(outL[b], m1), V=(outR[b], m2), cap=cap_s, rank_ri=kk[b]))
            self.trunc(probs)
            cur_L = [[(outL[b], m1, Dim(cap_s, kk[b]), 1.0)] for b in B]
            cur_R = [[(outR[b], m2, Dim(cap_s, kk[b]), 1.0)] for b in B]
        sL = [cur_L[b][0][0] for b in B]
        sR = [cur_R[b][0][0] for b in B]
        ks = kk
        # S = T1^T S~ (hqr.py:150)
        sL2 = [self._sh(m1 * cap_s) for _ in B]
        self.happly(c1, "T", True, [(sL[b], m1) for b in B], [(sL2[b], m1) for b in B], (cap_s, ks))
        # R's a12 = T([A12.L, -Y11 S.L], [A12.R; S.R]) (hqr.py:153-155): off the
        # critical chain (only the output R reads it) -> side lane
        self.lane = self.side_lane()
        self.lane_bump(R_PHASE).reset()
        ys = [self._ph(m1 * cap_s) for _ in B]
        self.happly(c1, "Y", False, [(sL2[b], m1) for b in B], [(ys[b], m1) for b in B], (cap_s, ks))
        probs = []
        for b in B:
            d = D[b]
            probs.append(dict(m=m1, n=m2,
                              L=[(d["A12U"][v], m1, Dim(kc, d["rA12"][v]), 1.0), (ys[b], m1, Dim(cap_s, ks[b]), -1.0)],
                              R=[(d["A12V"][v], m2, Dim(kc, d["rA12"][v]), 1.0), (sR[b], m2, Dim(cap_s, ks[b]), 1.0)],
                              eps_slot=self.eps_slot(b), eps_scale=1.0, U=(d["A12U"][v], m1),
                              V=(d["A12V"][v], m2), cap=kc, rank_ri=d["rA12"][v]))
        self.trunc(probs)
        self.lane = 0
        # cross = QB (Y_B S.L) (hqr.py:156)
        w1 = [self._ph(kc * cap_s) for _ in B]
        cross = [self._sh(m2 * cap_s) for _ in B]
        ks1 = min(32, m1 // 256) if m1 >= 1024 else 1
        self.gemm([(w1[b], kc, Dim(kc, D[b]["rA21"][v]), Dim(cap_s, ks[b]), 0.0,
                    [(D[b]["YV21"][v], m1, 1, 0, sL2[b], m1, 0, 0, Dim(m1), 1.0)]) for b in B],
                  ksplit=ks1)
        self.gemm([(cross[b], m2, Dim(m2), Dim(cap_s, ks[b]), 0.0,
                    [(D[b]["A21U"][v], m2, 0, 0, w1[b], kc, 0, 0, Dim(kc, D[b]["rA21"][v]), 1.0)]) for b in B])
        # A22 <- A22 - cross S.R: leaves densely, blocks recompressed (arith.py:126-145)
        leafp = []
        for b in B:
            for lf in t.leaves(c2):
                o, nl = t.off[lf] - t.off[c2], t.size[lf]
                leafp.append((D[b]["leafA"][lf], nl, Dim(nl), Dim(nl), 1.0,
                              [(cross[b] + o, m2, 0, 0, sR[b] + o, m2, 1, 0, Dim(cap_s, ks[b]), -1.0)]))
        self.gemm(leafp)
        # the a21 blocks of c2's leftmost spine are the next B blocks of the
        # chain: recompress them on the main lane, every other block of the
        # subtree on a side lane (dependencies are tracked per buffer)
        spine = set()
        u = c2
        while not t.is_leaf(u):
            spine.add(u)
            u = t.children(u)[0]
        probs, side = [], []
        for b in B:
            d = D[b]
            for u in t.internal_nodes(c2) if not t.is_leaf(c2) else []:
                u1, u2 = t.children(u)
                k_u = self.lay.kc[u]
                for kind in ("a12", "a21"):
                    if kind == "a12":
                        rs, rn, cs, cn, U, V, R = u1, t.size[u1], u2, t.size[u2], d["A12U"], d["A12V"], d["rA12"]
                    else:
                        rs, rn, cs, cn, U, V, R = u2, t.size[u2], u1, t.size[u1], d["A21U"], d["A21V"], d["rA21"]
                    ro, co = t.off[rs] - t.off[c2], t.off[cs] - t.off[c2]
                    (probs if (kind == "a21" and u in spine) else side).append(dict(m=rn, n=cn,
                                      L=[(U[u], rn, Dim(k_u, R[u]), 1.0), (cross[b] + ro, m2, Dim(cap_s, ks[b]), -1.0)],
                                      R=[(V[u], cn, Dim(k_u, R[u]), 1.0), (sR[b] + co, m2, Dim(cap_s, ks[b]), 1.0)],
                                      eps_slot=self.eps_slot(b), eps_scale=1.0, U=(U[u], rn), V=(V[u], cn),
                                      cap=k_u, rank_ri=R[u]))
        self.trunc(probs)
        if side:
            self.lane = self.side_lane()
            self.trunc(side)
            self.lane = 0
        # slab updates B_R2 -= (Y_B1 S.L) S.R, C2 likewise (hqr.py:158-159)
        g1, g2 = [], []
        for b in B:
            for (vc1, yc1, ld, ri, kw), (vc2, yc2, _, _, _) in zip(self.slabs(b, v, c1), self.slabs(b, v, c2)):
                zb = self._ph(cap_s * kw)
                g1.append((zb, cap_s, Dim(cap_s, ks[b]), Dim(kw, ri), 0.0,
                           [(sL2[b], m1, 1, 0, yc1, ld, 0, 0, Dim(m1), 1.0)]))
                g2.append((vc2, ld, Dim(m2), Dim(kw, ri), 1.0,
                           [(sR[b], m2, 0, 0, zb, cap_s, 0, 0, Dim(cap_s, ks[b]), -1.0)]))
        if g1:
            self.gemm(g1, ksplit=ks1)
            self.gemm(g2)

    def t_phase(self, v):
        """hqr.py:169-181: T~12 (one recompression of the three-term sum) and
        T12 = -T1 T~12 T2.  Runs on a side lane: only later S-phases (through
        T(c1) of an ancestor) and the output read T12."""
        t = self.tree
        self.cur_level = v[0]
        self.lane = self.side_lane()
        self.lane_bump(R_PHASE).reset()
        c1, c2 = t.children(v)
        m1, m2 = t.size[c1], t.size[c2]
        kc = self.lay.kc[v]
        B = range(self.B)
        D = [self.lay.m[b] for b in B]
        tmp3 = [self._ph(m2 * kc) for _ in B]
        self.happly(c2, "Y", True, [(D[b]["A21U"][v], m2) for b in B], [(tmp3[b], m2) for b in B],
                    (kc, [D[b]["rA21"][v] for b in B]))
        # T~12 = T(T(u1 + u2) + u3) with the plain eps (hqr.py:170-179)
        first = self.first_col(v)
        cur_L = [[(D[b]["YV21"][v], m1, Dim(kc, D[b]["rA21"][v]), 1.0)] for b in B]
        cur_R = [[(tmp3[b], m2, Dim(kc, D[b]["rA21"][v]), 1.0)] for b in B]
        sl = [(self.slabs(b, v, c1), self.slabs(b, v, c2)) for b in B]
        adds = [
            ([[(y1, ld, Dim(kw, ri), 1.0) for (v1, y1, ld, ri, kw) in (sl[b][0][:1] if first else [])] for b in B],
             [[(y2, ld, Dim(kw, ri), 1.0) for (v2, y2, ld, ri, kw) in (sl[b][1][:1] if first else [])] for b in B]),
            ([[(y1, ld, Dim(kw, ri), 1.0) for (v1, y1, ld, ri, kw) in (sl[b][0][1:] if first else sl[b][0])] for b in B],
             [[(y2, ld, Dim(kw, ri), 1.0) for (v2, y2, ld, ri, kw) in (sl[b][1][1:] if first else sl[b][1])] for b in B]),
        ]
        # T(u1 + 0) is still a truncation of the untruncated u1 (kept); an
        # empty last term would only re-truncate (skipped, T(T(x)) = T(x))
        adds = [ad for i, ad in enumerate(adds) if i == 0 or any(ad[0][b] for b in B)]
        for step, (addL, addR) in enumerate(adds):
            last = step == len(adds) - 1
            outL = [self._ph(m1 * kc) for _ in B]
            outR = [self._ph(m2 * kc) for _ in B]
            kk = [D[b]["rT12"][v] if last else self.slots.take() for b in B]
            probs = []
            for b in B:
                probs.append(dict(m=m1, n=m2, L=cur_L[b] + addL[b], R=cur_R[b] + addR[b], eps_slot=-1,
                                  eps_scale=self.eps, U=(outL[b], m1), V=(outR[b], m2), cap=kc,
                                  rank_ri=kk[b]))
            self.trunc(probs)
            cur_L = [[(outL[b], m1, Dim(kc, kk[b]), 1.0)] for b in B]
            cur_R = [[(outR[b], m2, Dim(kc, kk[b]), 1.0)] for b in B]
        tL = [cur_L[b][0][0] for b in B]
        tR = [cur_R[b][0][0] for b in B]
        rT = [D[b]["rT12"][v] for b in B]
        self.happly(c1, "T", False, [(tL[b], m1) for b in B], [(D[b]["T12U"][v], m1) for b in B],
                    (kc, rT), alpha=-1.0)
        self.happly(c2, "T", True, [(tR[b], m2) for b in B], [(D[b]["T12V"][v], m2) for b in B],
                    (kc, rT))
        self.lane = 0


# ---------------------------------------------------------------- packing

PIVOT_CORE = os.environ.get("HQ_PIVOT_CORE", "1") != "0"   # column-pivoted core QR before the Jacobi
CORE_STOP = 1e-3           # pivoted QR stops at ||R22||_F <= CORE_STOP * threshold (the Jacobi's own
                           # level for columns it never rotates against each other)
SVD_SMEM_DOUBLES = 24576   # single-CTA staging capacity (hq_svd_kernel.cuh)
CLUSTER_BUF_DOUBLES = 26880  # per-CTA block buffers (hq_svd_cluster.cuh C_SMEM_DOUBLES)
SVD_SINGLE_MAX_PAIRS = 16     # HQ_SVD_SINGLE_MAX_PAIRS (hq_svd_cluster.cuh)


def qr_cluster(qr_probs):
    """Cluster size for a QR launch: spread few, wide problems over several
    SMs; many problems (or narrow ones) run one CTA each.  Above 48 problems
    one CTA each leaves SMs free for the side streams' work: measured on the
    bench workload (batch 58, profiles/r01_ab_qr_cluster_*.txt) a one-CTA
    launch for 58 problems shortens the step 1195 -> 1170 ms at unchanged QR
    kernel time, while 2-CTA clusters for 75-148 problems lengthen it."""
    n = len(qr_probs)
    kmax = max(p[7].cap for p in qr_probs)
    if kmax < 48 or n > int(os.environ.get("HQ_QR_ONE_CTA_ABOVE", "48")):
        return 1
    if n <= 18:
        return 8
    return 4 if n <= 37 else 2


SVD_BLOCK_MIN = int(os.environ.get("HQ_SVD_BLOCK_MIN", "256"))   # block Jacobi candidates: cores this wide


def svd_use_block(nprob, m, n, G=None):
    """Block Jacobi (hq_svd_block) instead of the scalar kernel: for cores
    the scalar kernel could only run on one CTA from global memory, and for
    wide cores whose clusters would take several waves of the 148 SMs
    (measured, tools/jacobi_ab.py / profiles/r02_jacobi_ab.txt: 56 cores of
    300 columns 27.6 -> 20.2 ms, 450: 189 -> 61 ms, 560: 1466 -> 128 ms;
    below ~250 columns the scalar kernel is faster)."""
    if n <= 0 or m <= 0:
        return False
    if G is None:
        G = svd_cluster_runtime(nprob, m, n)
    scalar_global = G == 1 and not (_svd_fits(1, m, n) and (n + 1) // 2 <= SVD_SINGLE_MAX_PAIRS) \
        and not _svd_fits(2, m, n)
    return scalar_global or (n >= SVD_BLOCK_MIN and nprob * G > 148)


def svd_block_cluster(nprob, n, sms=148):
    """CTAs per problem of a block-Jacobi launch: enough warps (16 per CTA)
    for one pass over a round's ceil(n/16) block pairs, a power of two <= 8,
    as long as the launch still fits the SMs."""
    ntask = -(-(-(-n // 8)) // 2)
    need = max(1, -(-ntask // 16))
    G = 1
    while G < need and G < 8 and nprob * 2 * G <= sms:
        G *= 2
    return G


def svd_cluster(svd_probs):
    """Kernel for a Jacobi launch.  Cores of at least SVD_BLOCK_MIN columns
    run the block Jacobi (hq_svd_block: 16-column Grams and updates on the
    tensor pipe, one CTA per problem); narrower ones the scalar kernel:
    launches with many problems already fill the GPU one CTA each, few-problem
    launches get an 8-CTA cluster and the kernel picks one SM, the cluster,
    or the global-memory path from the run-time core size (capacities
    overstate it)."""
    mmax = max(p[5].cap for p in svd_probs)
    nmax = max(min(p[5].cap, p[6].cap) for p in svd_probs)
    ld = (mmax + 1) // 2 * 2
    if svd_use_block(len(svd_probs), mmax, nmax):
        return dict(cluster=1, max_m=mmax, block=True, bcluster=svd_block_cluster(len(svd_probs), nmax))
    if len(svd_probs) > 18 or mmax > 512:
        return dict(cluster=1, max_m=mmax, block=False)
    if ld * nmax <= SVD_SMEM_DOUBLES and (nmax + 1) // 2 <= SVD_SINGLE_MAX_PAIRS:
        return dict(cluster=1, max_m=mmax, block=False)
    return dict(cluster=8, max_m=mmax, block=False)


SVD_C_SMEM_DOUBLES, SVD_C_MAX_BS = 26880, 64   # hq_svd_cluster.cuh C_SMEM_DOUBLES / C_MAX_BS


def _svd_fits(G, m, n):
    """The cluster kernel's own test (hq_svd_cluster.cuh): G CTAs hold the
    core in 2G column blocks, two buffer sets."""
    if G == 1:
        return (m + 1) // 2 * 2 * n <= SVD_SMEM_DOUBLES
    bs = -(-n // (2 * G))
    return m <= 640 and 4 * bs * ((m + 1) // 2 * 2) <= SVD_C_SMEM_DOUBLES and bs <= SVD_C_MAX_BS


QRCP_SMEM_MAX = 28928   # doubles of dynamic shared memory per CTA (hq_qrcp.cu)


def qrcp_smem(G, m, n, threads):
    """Shared-memory doubles a CTA of a G-CTA hq_qrcp cluster needs to hold
    its column slice of an m x n core (the kernel's own carve-up: norms,
    candidate buffers, the slice with its bank-staggered row stride), or None
    when the slice cannot live there."""
    ncl = -(-n // G)
    tpc = 1
    while tpc < 32 and ncl * tpc * 2 <= threads:
        tpc *= 2
    if ncl * tpc > threads:
        return None
    q = 32 // tpc if tpc >= 4 else 0
    lds = ncl + (q - ncl) % 16
    need = 8 + 2 * ncl + 2 * G * (((m + 1) & ~1) + 4) + m * lds
    return need if need <= QRCP_SMEM_MAX else None


def qrcp_launch(nprob, m, n, sms=148):
    """(cluster size, shared-memory doubles, threads) of a pivoted-QR launch
    whose largest core is m x n: the smallest cluster that holds the core in
    shared memory (a step costs one cluster barrier and G candidate
    broadcasts, so wider is slower: tools/qrcp_micro.py), two CTAs for cores
    of >= 96 columns while the launch fits one wave; 512-thread CTAs when
    every CTA gets its own SM, else 256 so that several share one."""
    if m <= 0 or n <= 0:
        return 1, 64, 256
    for G in (1, 2, 4, 8):
        threads = 512 if nprob * G <= sms else 256
        if G == 1 and n >= 96 and nprob * 2 <= sms and qrcp_smem(2, m, n, 512):
            continue
        need = qrcp_smem(G, m, n, threads)
        if need:
            return G, need, threads
    return 8, QRCP_SMEM_MAX, 512   # reduced in place in global memory


SVD_SMALL_MAX = int(os.environ.get("HQ_SVD_SMALL_MAX", "8192"))   # doubles of staging per small-core CTA


def svd_small_doubles(nprob, m, n, sms=148):
    """Staging doubles for the small-core Jacobi kernel (128-thread CTAs,
    several per SM), or 0 when the launch should not use it: it pays when a
    launch has more problems than SMs (the cluster kernels would run in many
    waves of one CTA per SM) and the cores are small enough for >= 2 CTAs to
    share an SM (tools/svd_small_ab.py, 1482 cores: 48 x 32 9.1 -> 1.6 ms,
    80 x 48 14.9 -> 7.5 ms, 112 x 64 26.4 -> 18.3 ms against 2-CTA clusters)."""
    need = (m + 1) // 2 * 2 * n
    if nprob > sms and m <= 128 and need <= SVD_SMALL_MAX:
        return max(64, need)
    return 0


def svd_cluster_runtime(nprob, m, n, sms=148):
    """Cluster size for a Jacobi launch whose largest core is m x n (run-time
    sizes, e.g. from a previous run of the plan): the smallest cluster whose
    shared memory holds the core (a core that spills to the global-memory
    path is 4-6x slower), widened while the launch still fits one wave."""
    if n <= 0 or m <= 0:
        return 1
    if svd_small_doubles(nprob, m, n, sms):
        return 0
    if _svd_fits(1, m, n) and ((n + 1) // 2 <= SVD_SINGLE_MAX_PAIRS or nprob > sms):
        return 1   # few pairs, or more problems than SMs: one CTA each beats clusters in waves
    fit = [G for G in (2, 4, 8) if _svd_fits(G, m, n)]
    if not fit:
        # too wide for 8 CTAs: a (non-portable) 16-CTA cluster if it fits there
        return 16 if _svd_fits(16, m, n) else 1
    G = fit[0]
    while G < 8 and nprob * 2 * G <= sms:
        G *= 2
    return G


def retune_clusters(builder, rk, margin=1.1):
    """Re-pick every Jacobi launch's cluster size from the core sizes of a
    finished run (rank table rk) with some headroom; the launch records share
    the ops' extra dicts.  Returns the number of launches changed (the caller
    re-captures its graph)."""
    changed = 0
    for kind, probs, extra in builder.ops:
        if kind == "qrcp" and probs:
            mm = max(_dv(p[2], rk) for p in probs)
            nn = max(_dv(p[3], rk) for p in probs)
            m2 = min(int(mm * margin) + 1, max(p[2].cap for p in probs)) if mm else 0
            n2 = min(int(nn * margin) + 1, max(p[3].cap for p in probs)) if nn else 0
            G, smem, threads = qrcp_launch(len(probs), m2, n2)
            if (G, smem, threads) != (extra.get("cluster"), extra.get("smem"), extra.get("threads")):
                extra["cluster"], extra["smem"], extra["threads"] = G, smem, threads
                changed += 1
            continue
        if kind != "svd" or not probs:
            continue
        mm = nn = 0
        for p in probs:
            m, n = _dv(p[5], rk), _dv(p[6], rk)
            if p[12]:
                n = min(n, m)
            mm, nn = max(mm, m), max(nn, n)
        m2 = min(int(mm * margin) + 1, p[5].cap) if mm else 0
        n2 = min(int(nn * margin) + 1, m2) if nn else 0
        G = svd_cluster_runtime(len(probs), m2, n2)
        block = svd_use_block(len(probs), m2, n2, G) if G else False
        bG = svd_block_cluster(len(probs), n2) if block else 1
        small = svd_small_doubles(len(probs), m2, n2) if G == 0 else 0
        if block:
            G = 1
        if (G != extra.get("cluster", 1) or block != extra.get("block", False)
                or bG != extra.get("bcluster", 1) or small != extra.get("small", 0)):
            extra["cluster"] = G
            extra["block"] = block
            extra["bcluster"] = bG
            extra["small"] = small
            changed += 1
    return changed


def _addr(buf, bases, base_ptr):
    if buf is None:
        return 0
    return base_ptr + 8 * (bases[buf.reg] + buf.off)


def op_resources(builder, kind, probs, extra, mem=None):
    """(reads, writes) of one op: allocations touched ('m', region, start),
    rank-table slots ('r', slot) and the scalar table ('scal',).  The rank
    capacity-overflow flag is excluded (it is only ever set).  mem: optional
    Buf -> key map (default: the allocation start after finalize())."""
    R, W = set(), set()
    bumps = builder.bumps

    if mem is None:
        def mem(buf):
            if buf is None:
                return None
            return ("m", buf.reg, bumps[buf.reg].owner(buf.off))

    def rd(buf):
        k = mem(buf)
        if k:
            R.add(k)

    def wr(buf):
        k = mem(buf)
        if k:
            W.add(k)

    def slot(d, write=False):
        ri = d.ri if isinstance(d, Dim) else d
        if ri is not None and ri >= 0 and ri != builder.flag_slot:
            (W if write else R).add(("r", ri))

    if kind == "gemm":
        if extra.get("skip") is not None:
            slot(extra["skip"])
        for (c, ldc, m, n, beta, terms) in probs:
            wr(c)
            if beta != 0.0:
                rd(c)
            slot(m), slot(n)
            for t in terms:
                rd(t[0]), rd(t[4]), slot(t[8])
    elif kind == "zero":
        for (buf, cnt) in probs:
            wr(buf)
    elif kind == "concat":
        for (dst, dst2, rows, kri, pieces) in probs:
            wr(dst), wr(dst2), slot(kri, True)
            for (pp, ld, d, alpha) in pieces:
                rd(pp), slot(d)
    elif kind == "qr":
        for (w, tau, tp, tf, ldw, ldt, m, k) in probs:
            rd(w), wr(w), wr(tau), wr(tp), wr(tf), slot(m), slot(k)
    elif kind == "qrcp":
        for (c, ldc, m, n, rri, es, ssc) in probs:
            rd(c), wr(c), slot(m), slot(n), slot(rri, True)
            if es >= 0:
                R.add(("scal",))
    elif kind == "svd":
        for (c, u, w, ldc, ldu, m, n, cap, rri, fri, es, esc, xf) in probs:
            rd(c), wr(c), wr(u), wr(w), slot(m), slot(n), slot(rri, True)
            if es >= 0:
                R.add(("scal",))
    elif kind == "applyq":
        for (w, tau, tp, x, x0, ldw, ldx, ldx0, m, k, c, r0, tr) in probs:
            rd(w), rd(tau), rd(tp), rd(x0), rd(x), wr(x)
            slot(m), slot(k), slot(c), slot(r0)
    elif kind in ("leaf_gather", "leaf_scatter"):
        for (leaf, panel, nl, ldp, slabs, mri) in probs:
            if kind == "leaf_gather":
                rd(leaf), wr(panel), slot(mri, True)
                for (vv, yv, ld, ldy, kri) in slabs:
                    rd(vv), slot(kri)
            else:
                rd(panel), wr(leaf), slot(mri)
                for (vv, yv, ld, ldy, kri) in slabs:
                    wr(yv), slot(kri)
    elif kind == "power":
        for buf in (builder.PX, builder.PW, builder.PG):
            rd(buf)
        wr(builder.PX)
        R.add(("scal",)), W.add(("scal",))
        for i in range(builder.B):
            slot(builder.power_done + i), slot(builder.power_done + i, True)
        for i in (0, 1):
            slot(builder.all_done + i), slot(builder.all_done + i, True)
    elif kind == "rowblk":
        for (S_, W_, lds, ldw, ch, rt, k, nc, msr, mode) in probs:
            slot(k), slot(nc)
            if mode == 0:
                rd(W_), wr(S_), slot(msr, True)
            else:
                rd(S_), wr(W_)
    elif kind == "copy":
        for (src, dst, rows, cols, lds, ldd, mode) in probs:
            rd(src), wr(dst), slot(cols)
    elif kind == "pack_copy":
        if extra["which"] == 1:
            rd(Buf(R_IN, 0))
            for (buf, rows, cols, *_) in probs:
                wr(buf), slot(cols)
        else:
            wr(Buf(R_OUT, 0)), W.add(("totals",))
            for (buf, rows, cols, *_) in probs:
                rd(buf), slot(cols)
    else:
        raise ValueError(kind)
    return R, W


def schedule(builder):
    """Cross-lane dependencies of the op list (program order = a valid
    topological order).  Returns lanes[i], waits[i] (ops of OTHER lanes op i
    must wait for, latest per lane) and the set of ops that must signal."""
    last_w, readers = {}, {}
    lanes, waits, signal = [], [], set()
    for i, (kind, probs, extra) in enumerate(builder.ops):
        Rs, Ws = op_resources(builder, kind, probs, extra)
        ln = extra.get("lane", 0)
        deps = set()
        for r in Rs | Ws:
            if r in last_w:
                deps.add(last_w[r])
        for r in Ws:
            deps.update(readers.get(r, ()))
        if kind == "pack_copy" and extra.get("which") == 0:
            # the output compaction joins every lane: its region may alias
            # scratch of the side lanes (CompiledPlan), so all of them finish first
            last_in_lane = {}
            for j, lj in enumerate(lanes):
                last_in_lane[lj] = j
            deps.update(last_in_lane.values())
        per_lane = {}
        for d in deps:
            if lanes[d] != ln:
                per_lane[lanes[d]] = max(per_lane.get(lanes[d], -1), d)
        w = sorted(per_lane.values())
        signal.update(w)
        lanes.append(ln)
        waits.append(w)
        for r in Rs:
            readers.setdefault(r, []).append(i)
        for r in Ws:
            last_w[r] = i
            readers[r] = []
    return lanes, waits, signal


class CompiledPlan:
    """Ops packed into one device descriptor buffer; run() launches them."""

    def __init__(self, builder: Builder, device, alias_out: bool = True):
        import torch
        self.b = builder
        self.device = device
        sizes = {r: bp.peak for r, bp in builder.bumps.items()}
        self.region_sizes = sizes
        # the compact output stream is written by the last op only (which joins
        # every lane): it shares the largest scratch region that can hold it
        scratch = [r for r in sizes if r not in (R_PERSIST, R_IN, R_OUT, R_SHARED) and sizes[r] >= sizes.get(R_OUT, 0)]
        self.out_alias = (max(scratch, key=lambda r: sizes[r]) if alias_out and scratch and sizes.get(R_OUT, 0) > 0
                          else None)
        bases, acc = {}, 0
        for r in sorted(sizes):
            if r == R_OUT and self.out_alias is not None:
                continue
            bases[r] = acc
            acc += (sizes[r] + 63) // 64 * 64
        if self.out_alias is not None:
            bases[R_OUT] = bases[self.out_alias]
        self.total_doubles = acc
        self.arena = torch.zeros(max(acc, 1), dtype=torch.float64, device=device)
        self.rank = torch.zeros(max(builder.slots.n, 1), dtype=torch.int32, device=device)
        self.scal = torch.zeros(max(2 * builder.B, 2), dtype=torch.float64, device=device)
        self.totals = torch.zeros(2, dtype=torch.int64, device=device)
        # split-K arrival counters: zero once, every use leaves them zero
        self.counters = torch.zeros(max(builder.n_cnt, 1), dtype=torch.int32, device=device)
        cnt_ptr = self.counters.data_ptr()
        base_ptr = self.arena.data_ptr()
        self.bases = bases
        A = lambda buf: _addr(buf, bases, base_ptr)
        chunks, self.launch = [], []
        off = 0

        def put(arr):
            nonlocal off
            raw = arr.tobytes()
            start = off
            chunks.append((start, raw))
            off = (off + len(raw) + 255) // 256 * 256
            return start

        for kind, probs, extra in builder.ops:
            if kind == "gemm":
                pa = np.zeros(len(probs), _abi.GEMM_PROB)
                nterm = sum(len(p[5]) for p in probs)
                ta = np.zeros(nterm, _abi.GEMM_TERM)
                ti = 0
                wsl = extra.get("ws", [None] * len(probs))
                cnl = extra.get("cnt", [-1] * len(probs))
                for i, (c, ldc, m, n, beta, terms) in enumerate(probs):
                    pa[i] = (A(c), ldc, m.cap, m.ri, n.cap, n.ri, ti, len(terms),
                             extra.get("items", [0] * len(probs))[i], beta, A(wsl[i]),
                             cnt_ptr + 4 * cnl[i] if cnl[i] >= 0 else 0)
                    for (a, lda, tra, ma, bb, ldb, trb, mb, k, alpha) in terms:
                        ta[ti] = (A(a), A(bb), lda, ldb, tra, trb, k.cap, k.ri, ma, mb, alpha)
                        ti += 1
                self.launch.append(("gemm", put(pa), put(ta), len(probs), extra))
            elif kind == "zero":
                ra = np.zeros(2 * len(probs), np.int64)
                mx = 0
                for i, (buf, cnt) in enumerate(probs):
                    ra[2 * i], ra[2 * i + 1] = A(buf), cnt
                    mx = max(mx, cnt)
                self.launch.append(("zero", put(ra), None, len(probs), dict(max_count=mx)))
            elif kind == "concat":
                pa = np.zeros(len(probs), _abi.CONCAT_PROB)
                npc = sum(len(p[4]) for p in probs)
                pc = np.zeros(max(npc, 1), _abi.PIECE)
                pi = 0
                for i, (dst, dst2, rows, kri, pieces) in enumerate(probs):
                    pa[i] = (A(dst), A(dst2), rows, rows, rows, pi, len(pieces), kri)
                    for (p, ld, d, alpha) in pieces:
                        pc[pi] = (A(p), ld, d.cap, d.ri, 0, alpha)
                        pi += 1
                self.launch.append(("concat", put(pa), put(pc), len(probs), extra))
            elif kind == "qr":
                pa = np.zeros(len(probs), _abi.QR_PROB)
                for i, (w, tau, tp, tf, ldw, ldt, m, k) in enumerate(probs):
                    pa[i] = (A(w), A(tau), A(tp), A(tf), ldw, ldt, m.cap, m.ri, k.cap, k.ri)
                self.launch.append(("qr", put(pa), None, len(probs), extra))
            elif kind == "qrcp":
                pa = np.zeros(len(probs), _abi.QRCP_PROB)
                for i, (c, ldc, m, n, rri, es, ssc) in enumerate(probs):
                    pa[i] = (A(c), ldc, m.cap, m.ri, n.cap, n.ri, rri, es, 0, ssc)
                self.launch.append(("qrcp", put(pa), None, len(probs), extra))
            elif kind == "svd":
                pa = np.zeros(len(probs), _abi.SVD_PROB)
                for i, (c, u, w, ldc, ldu, m, n, cap, rri, fri, es, esc, xf) in enumerate(probs):
                    pa[i] = (A(c), A(u), A(w), ldc, ldu, m.cap, m.ri, n.cap, n.ri, cap, rri, fri, es,
                             esc, xf, 0)
                self.launch.append(("svd", put(pa), None, len(probs), extra))
            elif kind == "applyq":
                pa = np.zeros(len(probs), _abi.APPLYQ_PROB)
                for i, (w, tau, tp, x, x0, ldw, ldx, ldx0, m, k, c, r0, tr) in enumerate(probs):
                    pa[i] = (A(w), A(tau), A(tp), A(x), A(x0), ldw, ldx, ldx0, m.cap, m.ri,
                             k.cap, k.ri, c.cap, c.ri, r0.cap, r0.ri, tr)
                self.launch.append(("applyq", put(pa), None, len(probs), extra))
            elif kind in ("leaf_gather", "leaf_scatter"):
                pa = np.zeros(len(probs), _abi.LEAF_PROB)
                ns = sum(len(p[4]) for p in probs)
                sa = np.zeros(max(ns, 1), _abi.SLAB)
                si = 0
                for i, (leaf, panel, nl, ldp, slabs, mri) in enumerate(probs):
                    pa[i] = (A(leaf), A(panel), nl, ldp, si, len(slabs), mri, 0)
                    for (vv, yv, ld, ldy, kri) in slabs:
                        sa[si] = (A(vv), A(yv), ld, ldy, kri, 0)
                        si += 1
                self.launch.append((kind, put(pa), put(sa), len(probs), extra))
            elif kind == "power":
                self.launch.append(("power", None, None, builder.B, extra))
            elif kind == "rowblk":
                pa = np.zeros(len(probs), _abi.ROWBLK_PROB)
                for i, (S_, W_, lds, ldw, ch, rt, k, nc, msr, mode) in enumerate(probs):
                    pa[i] = (A(S_), A(W_), lds, ldw, ch, rt, k.cap, k.ri, nc.cap, nc.ri, msr, mode)
                self.launch.append(("rowblk", put(pa), None, len(probs), extra))
            elif kind == "copy":
                it = np.zeros(len(probs), _abi.COPY_ITEM)
                for i, (src, dst, rows, cols, lds, ldd, mode) in enumerate(probs):
                    it[i] = (A(src), A(dst), rows, cols.cap, cols.ri, lds, ldd, mode)
                self.launch.append(("copy", put(it), None, len(probs), extra))
            elif kind == "pack_copy":
                it = np.zeros(len(probs), _abi.COPY_ITEM)
                for i, (buf, rows, cols, *mode) in enumerate(probs):
                    if extra["which"] == 1:
                        it[i] = (0, A(buf), rows, cols.cap, cols.ri, rows, rows, 0)
                    else:
                        it[i] = (A(buf), 0, rows, cols.cap, cols.ri, rows, rows, mode[0] if mode else 0)
                self.launch.append(("pack_copy", put(it), None, len(probs),
                                    dict(extra, base_ptr=A(extra["base"]))))
            else:
                raise ValueError(kind)
        blob = bytearray(max(off, 256))
        for start, raw in chunks:
            blob[start:start + len(raw)] = raw
        self.desc = torch.frombuffer(blob, dtype=torch.uint8).clone().to(device)
        self.n_launch = len(self.launch)
        self.lanes, self.waits, self.signal = schedule(builder)
        self.n_lanes = max(self.lanes) + 1 if self.lanes else 1
        self.graph = None

    def addr(self, buf):
        return _addr(buf, self.bases, self.arena.data_ptr())

    def launch_one(self, lib, rec, stream_handle):
        self._launch_list([rec], stream_handle, lib)

    def run(self, stream_handle: int, streams=None, events=None, stop=None, start=0):
        """Launch ops start..stop-1 (all by default).  With `streams` (torch
        streams indexed by lane) and an event factory, ops go to their lane's
        stream and cross-lane dependencies become event waits (DAG under graph
        capture); ops before `start` ran on the origin stream beforehand."""
        lib = _abi.load()
        end = len(self.launch) if stop is None else stop
        if streams is None or len(streams) == 1:
            self._launch_list(self.launch[start:end], stream_handle, lib)
            return
        done = {}
        for i in range(start, end):
            rec = self.launch[i]
            ln = self.lanes[i]
            st = streams[ln]
            for j in self.waits[i]:
                if j >= start:
                    st.wait_event(done[j])
            self._launch_list([rec], st.cuda_stream, lib)
            if i in self.signal:
                ev = events()
                ev.record(st)
                done[i] = ev
        # join every side stream back into the origin stream
        for ln in range(1, len(streams)):
            ev = events()
            ev.record(streams[ln])
            streams[0].wait_event(ev)

    def _launch_list(self, launch, stream_handle, lib):
        dp = self.desc.data_ptr()
        rk = self.rank.data_ptr()
        sc = self.scal.data_ptr()
        b = self.b
        for kind, o1, o2, cnt, ex in launch:
            if kind == "gemm":
                skip = rk + 4 * ex["skip"] if ex["skip"] is not None else None
                if ex.get("skinny"):
                    rc = lib.hq_gemm_skinny(stream_handle, dp + o1, cnt, dp + o2, rk, ex["ksplit"], ex["ncmax"],
                                            ex["mode"], ex["max_rows"], skip)
                else:
                    rc = lib.hq_gemm_tiled(stream_handle, dp + o1, cnt, dp + o2, rk, ex["tiles"], ex["ksplit"],
                                           ex.get("tile", 64), skip)
            elif kind == "zero":
                rc = lib.hq_zero(stream_handle, dp + o1, cnt, ex["max_count"])
            elif kind == "concat":
                rc = lib.hq_concat(stream_handle, dp + o1, cnt, dp + o2, rk, ex["max_rows"])
            elif kind == "qr":
                rc = lib.hq_qr(stream_handle, dp + o1, cnt, rk, ex.get("cluster", 1))
            elif kind == "qrcp":
                rc = lib.hq_qrcp(stream_handle, dp + o1, cnt, rk, sc, ex.get("cluster", 1),
                                 ex.get("smem", QRCP_SMEM_MAX), ex.get("threads", 512))
            elif kind == "svd":
                if ex.get("block"):
                    rc = lib.hq_svd_block(stream_handle, dp + o1, cnt, rk, sc, ex.get("bcluster", 1))
                else:
                    rc = lib.hq_svd(stream_handle, dp + o1, cnt, rk, sc, ex.get("cluster", 1), ex.get("max_m", 0),
                                    ex.get("small", 0))
            elif kind == "applyq":
                rc = lib.hq_applyq(stream_handle, dp + o1, cnt, rk, ex.get("max_cols", 0), ex.get("max_rows", 0))
            elif kind == "leaf_gather":
                rc = lib.hq_leaf_gather(stream_handle, dp + o1, cnt, dp + o2, rk, ex["max_nl"])
            elif kind == "leaf_scatter":
                rc = lib.hq_leaf_scatter(stream_handle, dp + o1, cnt, dp + o2, rk, ex["max_nl"])
            elif kind == "rowblk":
                rc = lib.hq_rowblocks(stream_handle, dp + o1, cnt, rk, ex["max_chunks"])
            elif kind == "copy":
                rc = lib.hq_copy(stream_handle, dp + o1, cnt, rk)
            elif kind == "pack_copy":
                rc = lib.hq_pack_offsets(stream_handle, dp + o1, cnt, rk, ex["base_ptr"],
                                         self.totals.data_ptr() + 8 * ex["total"], ex["which"])
                _abi.check(rc, "pack_offsets")
                rc = lib.hq_copy(stream_handle, dp + o1, cnt, rk)
            elif kind == "power":
                rc = lib.hq_power_step(stream_handle, self.addr(b.PX), self.addr(b.PW), self.addr(b.PG),
                                       b.tree.n, 2 if b.tree.n >= 2 else 1, sc, b.eps, b.tol,
                                       rk + 4 * b.power_done, rk + 4 * b.all_done, b.B, ex["final"])
            _abi.check(rc, kind)

    def count_kernels(self):
        return len(self.launch)


# ---------------------------------------------------------------- accounting

def _dv(d, rk):
    return d.cap if d.ri < 0 else int(min(max(int(rk[d.ri]), 0), d.cap))


def op_flops(kind, probs, rk):
    """Algorithmic FP64 flops of one op given the final rank table.
    gemm 2mnk per term; Householder QR 2mk^2 - 2k^3/3 (+ mk^2 when the full
    compact-WY T is formed); applyQ 4mkc - 2k^2c; Jacobi SVD counted as the
    R-SVD estimate 6mn^2 + 20n^3 (Golub-Van Loan, Sigma + U1)."""
    f = 0.0
    if kind == "gemm":
        for (c, ldc, m, n, beta, terms) in probs:
            mm, nn = _dv(m, rk), _dv(n, rk)
            for t in terms:
                f += 2.0 * mm * nn * _dv(t[8], rk)
    elif kind == "qr":
        for (w, tau, tp, tf, ldw, ldt, m, k) in probs:
            mm, kk = _dv(m, rk), _dv(k, rk)
            r = min(mm, kk)
            f += 2.0 * mm * r * kk - (2.0 / 3.0) * r ** 3 if mm >= kk else 2.0 * mm * mm * kk - (2.0 / 3.0) * mm ** 3
            if tf is not None:
                f += mm * r * r
    elif kind == "applyq":
        for p in probs:
            mm, kk, cc = _dv(p[8], rk), _dv(p[9], rk), _dv(p[10], rk)
            r = min(mm, kk)
            f += 4.0 * mm * r * cc - 2.0 * r * r * cc
    elif kind == "qrcp":
        for (c, ldc, m, n, rri, es, ssc) in probs:
            mm, nn, r = _dv(m, rk), _dv(n, rk), int(rk[rri])
            f += 4.0 * (mm * nn * r - (mm + nn) * r * r / 2.0 + r ** 3 / 3.0)
    elif kind == "svd":
        for p in probs:
            mm, nn = _dv(p[5], rk), _dv(p[6], rk)
            a, b = max(mm, nn), min(mm, nn)
            f += 6.0 * a * b * b + 20.0 * b ** 3
    return f


def op_bytes(kind, probs, rk):
    """Compulsory HBM/L2 bytes (read + write once) of data-movement ops."""
    by = 0.0
    if kind == "concat":
        for (dst, dst2, rows, kri, pieces) in probs:
            k = sum(_dv(d, rk) for _, _, d, _ in pieces)
            by += 8.0 * rows * k * (3 if dst2 is not None else 2)
    elif kind == "pack_copy":
        for (buf, rows, cols, *_) in probs:
            by += 16.0 * rows * _dv(cols, rk)
    elif kind in ("leaf_gather", "leaf_scatter"):
        for (leaf, panel, nl, ldp, slabs, mri) in probs:
            by += 16.0 * nl * (nl + sum(int(rk[s[4]]) for s in slabs))
    return by


def kind_key(kind, extra):
    """Kernel class of an op for accounting: the streaming skinny products
    (HBM-bound GEMVs) apart from the DMMA GEMMs, the block Jacobi apart from
    the scalar one."""
    if kind == "gemm" and extra.get("skinny"):
        return "gemv"
    if kind == "svd" and extra.get("block"):
        return "svd_block"
    return kind


def plan_accounting(builder, rk, skipped=None, rk_in=None):
    """Per-kernel-class launches / flops / bytes of a finished run.
    skipped: indices of the ops that were no-ops in that run (the power
    iteration's gated launches after convergence); None: count no gated op.
    rk_in: the rank table as uploaded (the INPUT's ranks): the gated ops --
    the power iteration on the input matrix -- ran before the factorization
    overwrote those slots with the factors' ranks, so their dimensions are
    taken from it (the final table would overcount their bytes severalfold)."""
    acc = {}
    for i, (kind, probs, extra) in enumerate(builder.ops):
        a = acc.setdefault(kind_key(kind, extra), {"launches": 0, "flops": 0.0, "bytes": 0.0})
        a["launches"] += 1
        gated = extra.get("skip") is not None
        if probs is None or (gated and (skipped is None or i in skipped)):
            continue
        r = rk_in if gated and rk_in is not None else rk
        a["flops"] += op_flops(kind, probs, r)
        a["bytes"] += op_bytes(kind, probs, r) if kind != "gemm" or not extra.get("skinny") \
            else gemv_bytes(probs, r)
    return acc


def gemv_bytes(probs, rk):
    """Compulsory bytes of a streaming skinny product: every term's A read
    once, B (k x n, tiny) and C (m x n) once."""
    by = 0.0
    for (c, ldc, m, n, beta, terms) in probs:
        mm, nn = _dv(m, rk), _dv(n, rk)
        for t in terms:
            k = _dv(t[8], rk)
            by += 8.0 * (mm * k + k * nn)
        by += 8.0 * mm * nn * (2 if beta != 0.0 else 1)
    return by
