"""Public hQR API on the B200 (drop-in for reference hodlrqr.hqr).

    f = hqr(a, eps)                 # reference hqr.py:80-92 signature
    f.y, f.t, f.r                   # HodlrMatrix factors, A ~= (I - Y T Y^T) R

The factorization runs entirely on the GPU through libhqb200.so: one plan per
(tree shape, batch, eps mode, rank capacity) is unrolled, packed and captured
as a CUDA graph; each call uploads the matrices (one H2D copy), replays the
graph and downloads the factors (one D2H copy).  There is no CPU fallback:
without a CUDA device or the library this raises.
"""

from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass
from functools import lru_cache

import numpy as np

from . import _abi
from .hodlr import (UNIT_LOWER_TRIANGULAR, UPPER_TRIANGULAR, HodlrMatrix, LowRankBlock,
                    PartitionTree)
from .plan import R_IN, R_OUT, R_PERSIST, Builder, CompiledPlan, retune_clusters


class RankCapacityError(RuntimeError):
    """A truncated rank exceeded the plan's rank capacity (raise kcap)."""


@dataclass
class HodlrQRFactors:
    """A ~= (I - Y T Y^T) R with all three factors sharing A's partition."""
    y: HodlrMatrix
    t: HodlrMatrix
    r: HodlrMatrix


@dataclass
class StructuredColumn:
    """Recursion input [a_tilde; b; c] of hqr_rec (reference hqr.py:38-56):
    an m x m HODLR block, a factorized p x m low-rank block and r2 x m dense
    coupling rows.  b and c may both be empty."""
    a_tilde: HodlrMatrix
    b: LowRankBlock
    c: np.ndarray

    def __post_init__(self):
        m = self.a_tilde.n
        self.c = np.asarray(self.c, dtype=float).reshape(-1, m)
        if self.b.n_cols != m:
            raise ValueError("column counts of a_tilde and b must agree")

    @staticmethod
    def whole_matrix(a: HodlrMatrix) -> "StructuredColumn":
        return StructuredColumn(a, LowRankBlock.zero(0, a.n), np.zeros((0, a.n)))


@dataclass
class StructuredY:
    """Mirror of StructuredColumn for the reflector factor Y (hqr.py:59-68)."""
    y_a: HodlrMatrix
    y_b: LowRankBlock
    y_c: np.ndarray

    def to_dense(self) -> np.ndarray:
        from .hodlr import to_dense as hodlr_to_dense
        return np.vstack([hodlr_to_dense(self.y_a), self.y_b.to_dense(), self.y_c])


def _require_cuda():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1809_10585_b200.hqr needs a CUDA device (B200); no CPU fallback")
    _abi.load()
    return torch


def _start_vectors(n):
    """Deterministic start block of the power method (dense.py:118-121)."""
    rng = np.random.default_rng(0x5EED)
    x = np.column_stack([np.full(n, 1.0 / np.sqrt(n)), rng.standard_normal(n)])
    return np.linalg.qr(x)[0]


_POOL = None
_now = __import__("time").perf_counter


def _pool():
    """Host worker threads for packing / assembling factor streams (numpy
    copies release the GIL)."""
    global _POOL
    if _POOL is None:
        _POOL = ThreadPoolExecutor(max_workers=max(1, min(16, os.cpu_count() or 1)),
                                   thread_name_prefix="hqb200-io")
    return _POOL


@lru_cache(maxsize=8)
def _start_block(n):
    x = _start_vectors(n) if n >= 2 else np.ones((1, 2))
    x = np.asfortranarray(x)
    x.flags.writeable = False
    return x


_CPOOL = None


def _fresh_copy(src, parts):
    """np.array(src) with the copy (and the page faults of the fresh memory)
    split over `parts` threads of a pool separate from the assembly workers."""
    global _CPOOL
    if parts <= 1 or src.size < (1 << 21):
        return np.array(src)
    if _CPOOL is None:
        _CPOOL = ThreadPoolExecutor(max_workers=max(1, min(16, os.cpu_count() or 1)),
                                    thread_name_prefix="hqb200-copy")
    dst = np.empty_like(src)
    step = -(-src.size // parts)
    fs = [_CPOOL.submit(np.copyto, dst[i:i + step], src[i:i + step]) for i in range(0, src.size, step)]
    for f in fs:
        f.result()
    return dst


def _copy_items(dst, items):
    """items: (offset, rows, cols, src); writes src column-major at offset."""
    for o, r, c, src in items:
        np.copyto(dst[o:o + r * c].reshape((r, c), order="F"), src)


def _split_even(items, weight, parts):
    """Consecutive groups of roughly equal total weight."""
    tot = sum(weight(i) for i in items)
    groups, cur, acc = [], [], 0.0
    for it in items:
        cur.append(it)
        acc += weight(it)
        if acc >= tot / parts and len(groups) < parts - 1:
            groups.append(cur)
            cur, acc = [], 0.0
    if cur:
        groups.append(cur)
    return groups


class PlanIO:
    """Host side of a plan: packs inputs into the compact input stream and
    assembles HodlrMatrix factors from the compact output stream (no CUDA).

    Both streams are grouped by matrix (all items of matrix 0, then 1, ...);
    item offsets are prefix sums of rows x (capacity or run-time rank)."""

    def __init__(self, tree: PartitionTree, batch: int = 1, eps: float = 1e-10,
                 absolute: bool = False, kcap: int = 512, builder: Builder = None):
        """builder: an already built plan of these parameters (e.g. a tracked
        one for distributed.py); default: build it."""
        self.tree, self.B, self.eps, self.absolute, self.kcap = tree, batch, eps, absolute, kcap
        self.builder = builder if builder is not None else Builder(tree, batch, eps, absolute, kcap).build()
        bld = self.builder
        self.inbuf = np.zeros(max(bld.bumps[R_IN].peak, 1))
        self.outbuf = np.zeros(max(bld.bumps[R_OUT].peak, 1))
        self.px = np.zeros(2 * bld.tree.n * batch)
        self.rk = np.zeros(max(bld.slots.n, 1), np.int32)
        self.sc = np.zeros(max(2 * batch, 2))
        self.n_in = 0
        self.in_ranges = [(0, 0)] * batch
        oi = bld.out_items
        self._o_rows = np.array([r for _, r, _, _ in oi], np.int64)
        self._o_cap = np.array([c.cap for _, _, c, _ in oi], np.int64)
        self._o_ri = np.array([c.ri for _, _, c, _ in oi], np.int64)
        self._o_per_b = len(oi) // max(batch, 1)
        self._o_key = [(buf.reg, buf.off, mode) for buf, _, _, mode in oi]

    @staticmethod
    def _nodes(a: HodlrMatrix, t):
        """(level, index) -> HodlrMatrix node."""
        out = {}

        def walk(h, v):
            out[v] = h
            if not h.is_leaf:
                c1, c2 = t.children(v)
                walk(h.a11, c1)
                walk(h.a22, c2)
        walk(a, (0, 0))
        return out

    def _sources(self, b, a):
        """Rank-table entries and the input arrays of matrix b in stream order
        (leaves, then per internal node a12.L, a12.R^T, a21.L, a21.R^T; for a
        structured column then B.L, B.R^T and C^T)."""
        bld = self.builder
        t, lay = bld.tree, bld.lay
        col = a if hasattr(a, "a_tilde") else None
        if col is not None:
            a = col.a_tilde
        if tuple(a.leaf_sizes()) != tuple(self.tree.leaf_sizes):
            raise ValueError("matrix does not match the plan's partition tree")
        nodes = self._nodes(a, t)
        d = lay.m[b]
        srcs = [nodes[lf].dense for lf in t.leaves((0, 0))]
        for u in (t.internal_nodes((0, 0)) if t.L > 0 else []):
            h = nodes[u]
            kc = lay.kc[u]
            for blk, slot in ((h.a12, "rA12"), (h.a21, "rA21")):
                if blk.rank > kc:
                    raise RankCapacityError(f"input block rank {blk.rank} exceeds capacity {kc}")
                self.rk[d[slot][u]] = blk.rank
            srcs += [h.a12.L, h.a12.R.T, h.a21.L, h.a21.R.T]
        if bld.root_b is not None or bld.root_c:
            if col is None:
                raise ValueError("this plan factors structured columns [A; B; C]")
            if bld.root_b is not None:
                p_, k_ = bld.root_b
                if col.b.n_rows != p_ or col.b.rank > k_:
                    raise ValueError("B does not match the plan's structured column shape")
                self.rk[d["rBin"]] = col.b.rank
                srcs += [col.b.L, col.b.R.T]
            if bld.root_c:
                if col.c.shape[0] != bld.root_c:
                    raise ValueError("C does not match the plan's structured column shape")
                self.rk[d["rC"]] = bld.root_c
                srcs.append(col.c.T)
        elif col is not None and (col.b.n_rows or col.c.shape[0]):
            raise ValueError("this plan factors whole matrices (empty B and C)")
        return srcs

    def pack_async(self, mats):
        """Fill the rank table, then copy every matrix's factors into the
        compact input stream on the worker threads.  Returns one future per
        matrix (its stream range is self.in_ranges[b])."""
        if len(mats) != self.B:
            raise ValueError(f"expected {self.B} matrices, got {len(mats)}")
        bld = self.builder
        self.rk[:] = 0
        n = bld.tree.n
        x0 = _start_block(n)
        per_mat, off = [], 0
        for b, a in enumerate(mats):
            srcs = self._sources(b, a)
            o0 = off
            items = []
            for s in srcs:
                r, c = s.shape
                items.append((off, r, c, s))
                off += r * c
            self.in_ranges[b] = (o0, off)
            per_mat.append(items)
            self.px[2 * n * b:2 * n * (b + 1)] = x0.ravel(order="F")
        self.n_in = off
        self._ensure_inbuf(off)
        sc = self.sc
        sc[:] = 0.0
        if self.absolute:
            # hqr_rec passes its own threshold for the intermediate sums
            sc[1::2] = self.eps if getattr(self, "eps_abs", None) is None else self.eps_abs
            for b in range(self.B):
                self.rk[bld.power_done + b] = 1
            self.rk[bld.all_done] = 1
        pool = _pool()
        nthr = pool._max_workers
        futs = []
        for items in per_mat:
            groups = _split_even(items, lambda it: it[1] * it[2],
                                 max(1, min(len(items), nthr // max(1, len(per_mat)))))
            futs.append([pool.submit(_copy_items, self.inbuf, g) for g in groups])
        return futs

    def _ensure_inbuf(self, n):
        """The compact input stream buffer (capacity-sized, lazily mapped)."""
        return self.inbuf

    def pack(self, mats):
        """Input ranks -> rank table, factors -> compact input stream."""
        for fs in self.pack_async(mats):
            for f in fs:
                f.result()

    def out_offsets(self, rk):
        """Per-item offsets into the compact output stream for rank table rk;
        returns (offsets[items + 1], per-item column counts)."""
        ri = self._o_ri
        cols = np.where(ri < 0, self._o_cap,
                        np.minimum(np.maximum(rk[np.maximum(ri, 0)], 0), self._o_cap))
        off = np.zeros(len(ri) + 1, np.int64)
        np.cumsum(self._o_rows * cols, out=off[1:])
        return off, cols

    def out_range(self, b, offs):
        i0 = b * self._o_per_b
        return int(offs[0][i0]), int(offs[0][i0 + self._o_per_b])

    def factors(self, b: int, out=None, rk=None, offs=None, copy=True, out_base=0) -> HodlrQRFactors:
        """Assemble the HodlrMatrix factors of matrix b from the compact output
        `out` (holding the stream from position out_base on).  With copy, its
        range is first copied into fresh memory; the blocks are views of it."""
        bld = self.builder
        t = bld.tree
        d = bld.lay.m[b]
        offs = self.out_offsets(rk) if offs is None else offs
        off, cols = offs
        i0 = b * self._o_per_b
        lo, hi = int(off[i0]), int(off[i0 + self._o_per_b])
        parts = max(1, (os.cpu_count() or 1) // max(1, self.B))
        src = out[lo - out_base:hi - out_base]
        base = _fresh_copy(src, parts) if copy else src
        blocks = {}
        for i in range(i0, i0 + self._o_per_b):
            r, c = int(self._o_rows[i]), int(cols[i])
            s = int(off[i]) - lo
            blocks[self._o_key[i]] = base[s:s + r * c].reshape((r, c), order="F")
        get = lambda buf, mode=0: blocks[(buf.reg, buf.off, mode)]

        def build(v, which):
            if t.is_leaf(v):
                # leaves arrive masked (R, T upper; Y unit lower: hq_copy modes)
                if which == "t":
                    return HodlrMatrix(dense=get(d["leafT"][v], 1), shape_tag=UPPER_TRIANGULAR)
                if which == "r":
                    return HodlrMatrix(dense=get(d["leafA"][v], 1), shape_tag=UPPER_TRIANGULAR)
                return HodlrMatrix(dense=get(d["leafA"][v], 2), shape_tag=UNIT_LOWER_TRIANGULAR)
            c1, c2 = t.children(v)
            m1, m2 = t.size[c1], t.size[c2]
            h1, h2 = build(c1, which), build(c2, which)
            zero12, zero21 = LowRankBlock.zero(m1, m2), LowRankBlock.zero(m2, m1)
            if which == "y":
                a21 = LowRankBlock(get(d["A21U"][v]), get(d["YV21"][v]).T, True)
                return HodlrMatrix(a11=h1, a22=h2, a12=zero12, a21=a21, shape_tag=UNIT_LOWER_TRIANGULAR)
            if which == "t":
                a12 = LowRankBlock(get(d["T12U"][v]), get(d["T12V"][v]).T)
            else:
                a12 = LowRankBlock(get(d["A12U"][v]), get(d["A12V"][v]).T, True)
            return HodlrMatrix(a11=h1, a22=h2, a12=a12, a21=zero21, shape_tag=UPPER_TRIANGULAR)

        out = HodlrQRFactors(y=build((0, 0), "y"), t=build((0, 0), "t"), r=build((0, 0), "r"))
        if bld.root_b is not None or bld.root_c:
            n = t.n
            if bld.root_b is not None:
                yb = LowRankBlock(get(d["RB_L"]), get(d["RB_Y"]).T, True)
            else:
                yb = LowRankBlock.zero(0, n)
            yc = get(d["RC_Y"]).T if bld.root_c else np.zeros((0, n))
            out.y_b, out.y_c = yb, yc
        # `build` is a self-referencing closure (a reference cycle): drop the
        # block views it can reach so only the returned factors hold the memory
        blocks.clear()
        return out


class HQREngine(PlanIO):
    """PlanIO + device arena + CUDA graph for batched hQR of same-shape matrices."""

    def __init__(self, tree: PartitionTree, batch: int = 1, eps: float = 1e-10,
                 absolute: bool = False, kcap: int = 512, device=None, use_graph: bool = True,
                 stream_out: bool = False, builder=None):
        """stream_out: keep the compact output stream in its own region and
        run its compaction outside the graph, so factorize_stream() can copy
        one run's factors to the host while the next run computes (costs the
        output region's memory, which otherwise aliases scratch)."""
        torch = _require_cuda()
        super().__init__(tree, batch, eps, absolute, kcap, builder=builder)
        self.torch = torch
        self.device = torch.device(device if device is not None else "cuda")
        self.stream_out = bool(stream_out)
        self.plan = CompiledPlan(self.builder, self.device, alias_out=not self.stream_out)
        last = self.builder.ops[-1]
        assert last[0] == "pack_copy" and last[2].get("which") == 0, "plan must end with the output compaction"
        self._tail = len(self.plan.launch) - 1 if self.stream_out else None
        first = self.builder.ops[0]
        assert first[0] == "pack_copy" and first[2].get("which") == 1, "plan must start with the input restore"
        # streaming engines also run the input restore outside the graph, so the
        # next batch's upload can start as soon as it has consumed the inputs
        self._head = 1 if self.stream_out else 0
        self._d2h_done = None
        self._consumed = None
        self._h2d_ready = None
        self._step = 0
        pin = lambda a: torch.from_numpy(a).pin_memory()
        self.h_rk, self.h_sc, self.h_px = pin(self.rk), pin(self.sc), pin(self.px)
        self.rk, self.sc, self.px = self.h_rk.numpy(), self.h_sc.numpy(), self.h_px.numpy()
        # pinned host staging sized to the actual streams (the device regions
        # are capacity-sized): grown on demand
        in_cap, out_cap = self.inbuf.size, self.outbuf.size
        self.h_in = self.h_out = None
        self.inbuf = self.outbuf = None
        # rank table / totals read back per run: two pinned copies (a stream of
        # runs reads one while the next run's copy lands in the other)
        self._h_rk_outs = [torch.zeros_like(self.h_rk).pin_memory() for _ in range(2)]
        self._h_tots = [torch.zeros(2, dtype=torch.int64).pin_memory() for _ in range(2)]
        self.h_rk_out, self.h_tot = self._h_rk_outs[0], self._h_tots[0]
        p = self.plan
        ib, ob = p.bases[R_IN], p.bases[R_OUT]
        self.d_in = p.arena[ib:ib + in_cap]
        self.d_out = p.arena[ob:ob + out_cap]
        pxo = p.bases[R_PERSIST] + self.builder.PX.off
        self.d_px = p.arena[pxo:pxo + self.px.size]
        # where a run's rank table / scalars / power start are uploaded to:
        # the live buffers, or (streaming) staging copied in at execute()
        if self.stream_out:
            self._src = (torch.empty_like(p.rank), torch.empty_like(p.scal), torch.empty_like(self.d_px))
        else:
            self._src = (p.rank, p.scal, self.d_px)
        self.n_out = 0
        self.use_graph = use_graph
        self.graph = None
        # the chain lane outranks the side lanes: when both have CTAs pending
        # the critical path gets the SMs first (priorities are recorded in
        # the captured graph's kernel nodes)
        prio = -1 if os.environ.get("HQB200_CHAIN_PRIORITY", "1") not in ("0", "") else 0
        self.stream = torch.cuda.Stream(device=self.device, priority=prio)
        self.copy_stream = torch.cuda.Stream(device=self.device)
        self.h2d_stream = torch.cuda.Stream(device=self.device)
        self.side = [torch.cuda.Stream(device=self.device) for _ in range(self.plan.n_lanes - 1)]
        # side streams pay off when a launch leaves most SMs idle (few matrices)
        self.multi_stream = True
        self.autotune = os.environ.get("HQB200_AUTOTUNE", "1") not in ("0", "")
        self._tuned = False
        ms = os.environ.get("HQB200_MULTISTREAM")
        if ms is not None:
            self.multi_stream = ms not in ("0", "")
        self._pins = []
        self._evs = []
        # The plan is tens of millions of small Python objects (one tuple per
        # kernel problem): a full collection of the cyclic GC walks them all
        # (3.4 s for 57 matrices of n = 16384) and fires every few batches,
        # triggered by the result trees' allocations.  They live as long as the
        # engine, so they are moved to the permanent generation.
        if os.environ.get("HQB200_GC_FREEZE", "1") not in ("0", ""):
            import gc
            gc.freeze()

    def _retune(self, rk):
        """After the first run, size the Jacobi clusters from the actual core
        sizes (the plan only knows capacities); the next execute() captures
        a new graph."""
        if self._tuned or not self.autotune:
            return
        self._tuned = True
        if retune_clusters(self.builder, rk):
            self.graph = None

    def _pinned_staging(self, cur, n):
        if cur is not None and cur.numel() >= n:
            return cur
        return self.torch.empty(max(n + n // 4, 1), dtype=self.torch.float64, pin_memory=True)

    def _ensure_inbuf(self, n):
        h = self._pinned_staging(self.h_in, n)
        if h is not self.h_in:
            self.h_in, self.inbuf = h, h.numpy()
        return self.inbuf

    def upload(self):
        """H2D of the compact input stream, the rank table and the scalars."""
        rk, sc, px = self._src
        with self.torch.cuda.stream(self.stream):
            self.d_in[:self.n_in].copy_(self.h_in[:self.n_in], non_blocking=True)
            rk.copy_(self.h_rk, non_blocking=True)
            sc.copy_(self.h_sc, non_blocking=True)
            px.copy_(self.h_px, non_blocking=True)

    def h2d_bytes(self):
        return 8 * (self.n_in + self.px.size + self.sc.size) + 4 * self.rk.size

    def d2h_bytes(self):
        return 8 * (self.n_out + 2) + 4 * self.rk.size

    def restore_device_input(self):
        """Re-arm a run with the input already resident in HBM (device-side
        restore of the rank table / power start; the compact input stream in
        HBM is untouched by a run)."""
        rk, sc, px = self._src
        with self.torch.cuda.stream(self.stream):
            rk.copy_(self.d_rk0, non_blocking=True)
            sc.copy_(self.d_sc0, non_blocking=True)
            px.copy_(self.d_px0, non_blocking=True)

    def snapshot_device_input(self):
        """Keep a device copy of the freshly uploaded run state (call after
        upload(), before execute())."""
        rk, sc, px = self._src
        with self.torch.cuda.stream(self.stream):
            self.d_rk0 = rk.clone()
            self.d_sc0 = sc.clone()
            self.d_px0 = px.clone()

    def _launch(self):
        """Issue the plan: the critical chain on the engine stream, off-chain
        work (R and T coupling blocks, non-spine recompressions) on side
        streams, cross-stream dependencies as events -- a DAG once captured."""
        torch = self.torch
        if not self.side or not self.multi_stream:
            self.plan.run(self.stream.cuda_stream, stop=self._tail, start=self._head)
            return
        self._evs = []

        def mk():
            e = torch.cuda.Event()
            self._evs.append(e)
            return e

        fork = mk()
        fork.record(self.stream)
        for st in self.side:
            st.wait_event(fork)
        self.plan.run(self.stream.cuda_stream, [self.stream] + self.side, mk, stop=self._tail, start=self._head)

    def execute(self, tail: bool = True):
        """Run the factorization on the device (graph replay when captured);
        tail=False leaves the output compaction of a stream_out engine to
        launch_tail()."""
        torch = self.torch
        if self.stream_out:
            # streaming head: the staged run state goes live, then the input
            # restore (the compact input stream is free once it has run)
            p = self.plan
            if self._h2d_ready is not None:
                self.stream.wait_event(self._h2d_ready)
                self._h2d_ready = None
            self.stage_to_live()
            p._launch_list(p.launch[:self._head], self.stream.cuda_stream, _abi.load())
            self._consumed = torch.cuda.Event()
            self._consumed.record(self.stream)
        if not self.use_graph:
            self._launch()
        else:
            if self.graph is None:
                self.stream.synchronize()
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=self.stream):
                    self._launch()
                self.graph = g
            with torch.cuda.stream(self.stream):
                self.graph.replay()
        if tail:
            self.launch_tail()

    def stage_to_live(self):
        """Streaming engines: copy the staged rank table / scalars / power
        start into the buffers the kernels use (engine stream)."""
        p = self.plan
        if self._src[0] is p.rank:
            return
        with self.torch.cuda.stream(self.stream):
            for live, src in zip((p.rank, p.scal, self.d_px), self._src):
                live.copy_(src, non_blocking=True)

    def launch_tail(self):
        """stream_out: the output compaction, outside the graph -- it
        overwrites the output region only once the previous run's factors are
        on the host (event of the last collect's copies)."""
        if self._tail is None:
            return
        if self._d2h_done is not None:
            self.stream.wait_event(self._d2h_done)
        self.plan._launch_list(self.plan.launch[self._tail:], self.stream.cuda_stream, _abi.load())

    def download(self):
        """D2H of the rank table and the compact factor stream."""
        p = self.plan
        with self.torch.cuda.stream(self.stream):
            self.h_tot.copy_(p.totals, non_blocking=True)
            self.h_rk_out.copy_(p.rank, non_blocking=True)
        self.stream.synchronize()
        rk = self.h_rk_out.numpy()
        if int(rk[self.builder.flag_slot]) != 0:
            raise RankCapacityError(f"a truncated rank exceeded the capacity kcap={self.kcap}; "
                                    "retry with a larger kcap")
        self._retune(rk.copy())
        self.n_out = int(self.h_tot.numpy()[1])
        h = self._pinned_staging(self.h_out, self.n_out)
        if h is not self.h_out:
            self.h_out, self.outbuf = h, h.numpy()
        with self.torch.cuda.stream(self.stream):
            self.h_out[:self.n_out].copy_(self.d_out[:self.n_out], non_blocking=True)
        self.stream.synchronize()

    def factors(self, b: int, out=None, rk=None, offs=None, copy=True) -> HodlrQRFactors:
        rk = self.h_rk_out.numpy() if rk is None else rk
        return PlanIO.factors(self, b, self.outbuf if out is None else out, rk, offs, copy)

    def norm_estimate(self, b: int = 0) -> float:
        """||A_b||_2 estimate of the last run (device power iteration)."""
        return float(self.plan.scal[2 * b].item())

    def factorize(self, mats):
        """pack (worker threads) -> H2D per matrix as its range is packed ->
        graph replay -> rank table D2H -> per-matrix D2H of the compact factors,
        each matrix assembled on a worker thread as soon as its copy lands."""
        return self.collect(self.submit(mats))

    def factorize_stream(self, batches):
        """Factor a sequence of batches, yielding each batch's factors: batch
        i+1 is packed, uploaded and launched before batch i's factors are
        copied back, so (with stream_out) the device-to-host traffic of one
        batch overlaps the next batch's device work."""
        if not self.stream_out:   # the output region aliases scratch: no overlap
            for mats in batches:
                yield self.factorize(mats)
            return
        pending = None
        for mats in batches:
            self.launch_main(mats)
            if pending is not None:
                out = self.collect(pending)    # copies overlap this batch's graph
                pending = self.finish()        # its compaction waits for those copies
                yield out
            else:
                pending = self.finish()
        if pending is not None:
            yield self.collect(pending)

    def submit(self, mats):
        """First half of factorize(): pack, upload and launch; returns as soon
        as the replay is enqueued (the device works while the host goes on)."""
        self.launch_main(mats)
        return self.finish()

    def launch_main(self, mats):
        """pack + H2D + the graph (without a stream_out engine's compaction)."""
        torch = self.torch
        self._tr = [("start", _now())]
        if getattr(self, "_h2d_done", None) is not None:
            self._h2d_done.synchronize()   # the staging buffers of the previous run were consumed
        futs = self.pack_async(mats)
        up = self.h2d_stream if self.stream_out else self.stream
        if self.stream_out and self._consumed is not None:
            up.wait_event(self._consumed)   # the previous run's restore read the input region
        rk, sc, px = self._src
        with torch.cuda.stream(up):
            rk.copy_(self.h_rk, non_blocking=True)
            sc.copy_(self.h_sc, non_blocking=True)
            px.copy_(self.h_px, non_blocking=True)
            for b, fs in enumerate(futs):
                for f in fs:
                    f.result()
                lo, hi = self.in_ranges[b]
                if hi > lo:
                    self.d_in[lo:hi].copy_(self.h_in[lo:hi], non_blocking=True)
            self._h2d_done = torch.cuda.Event()
            self._h2d_done.record(up)
            if self.stream_out:
                self._h2d_ready = self._h2d_done
        self._tr.append(("packed", _now()))
        self.execute(tail=False)

    def finish(self):
        """Output compaction, rank-table read-back and the run's done event;
        returns the token collect() takes."""
        torch = self.torch
        p = self.plan
        self.launch_tail()
        par = self._step & 1
        self._step += 1
        self.h_rk_out, self.h_tot = self._h_rk_outs[par], self._h_tots[par]
        with torch.cuda.stream(self.stream):
            self.h_tot.copy_(p.totals, non_blocking=True)
            self.h_rk_out.copy_(p.rank, non_blocking=True)
        done = torch.cuda.Event()
        done.record(self.stream)
        self._tr.append(("replay_enqueued", _now()))
        return (done, self.h_rk_out, self.h_tot, self._tr)

    def collect(self, token=None):
        """Second half of factorize(): wait for the run, then D2H + assembly.
        The copies go on a copy stream, so a run submitted meanwhile keeps
        computing (factorize_stream)."""
        torch = self.torch
        if token is None:
            token = (None, self.h_rk_out, self.h_tot, self._tr)
        done, h_rk, h_tot, tr = token
        if done is None:
            self.stream.synchronize()
        else:
            done.synchronize()
        tr.append(("device_done", _now()))
        rk = h_rk.numpy().copy()
        if int(rk[self.builder.flag_slot]) != 0:
            raise RankCapacityError(f"a truncated rank exceeded the capacity kcap={self.kcap}; "
                                    "retry with a larger kcap")
        offs = self.out_offsets(rk)
        self.n_out = int(offs[0][-1])
        self._retune(rk)
        pool = _pool()
        jobs = []
        cs = self.copy_stream
        if done is not None:
            cs.wait_event(done)
        else:
            cs.wait_stream(self.stream)
        with torch.cuda.stream(cs):
            taken = []
            for b in range(self.B):
                # each matrix's factors land in their own pinned block, recycled
                # once the caller drops every factor that views it
                lo, hi = self.out_range(b, offs)
                hb = self._pinned_block(hi - lo, taken)
                taken.append(hb)
                if hi > lo:
                    hb[:hi - lo].copy_(self.d_out[lo:hi], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(cs)
                jobs.append(pool.submit(self._assemble, b, ev, rk, offs, hb, lo))
            d2h = torch.cuda.Event()
            d2h.record(cs)
            self._d2h_done = d2h
        tr.append(("d2h_enqueued", _now()))
        out = [j.result() for j in jobs]
        tr.append(("assembled", _now()))
        self.last_trace = {k: (t - tr[0][1]) * 1e3 for k, t in tr}
        return out

    def _pinned_block(self, size, taken=()):
        """A pinned host block of >= size doubles that no live result views.
        Returned factors are numpy views whose base is the block's tensor, so
        a block is free again once only the pool references its storage."""
        pool = self._pins
        use = getattr(self.torch._C, "_storage_Use_Count", None)
        best = None
        if use is not None:
            for blk in pool:
                if (blk.numel() >= size and not any(blk is t for t in taken)
                        and use(blk.untyped_storage()._cdata) <= 2):
                    if best is None or blk.numel() < best.numel():
                        best = blk
        if best is not None:
            return best
        self.pin_allocs = getattr(self, "pin_allocs", 0) + 1
        quantum = 1 << 20  # 8 MB granules, +25 % headroom for rank variation
        blk = self.torch.empty(-(-max(size + size // 4, 1) // quantum) * quantum, dtype=self.torch.float64,
                               pin_memory=True)
        if len(pool) < 4 * self.B + 4:
            pool.append(blk)
        return blk

    def _assemble(self, b, ev, rk, offs, hb, lo):
        ev.synchronize()
        return PlanIO.factors(self, b, hb.numpy(), rk, offs, False, lo)


from collections import OrderedDict

# engines of recent (tree, batch, eps, mode, capacity) keys, least recently
# used first.  Each holds a device arena (GBs at n = 16384) and pinned host
# staging, so only a few are kept: a tolerance sweep or a series of matrix
# sizes through hqr() evicts (and frees) the oldest instead of growing.
_ENGINES: "OrderedDict" = OrderedDict()
MAX_ENGINES = int(os.environ.get("HQB200_MAX_ENGINES", "2"))


def clear_engines():
    """Drop every cached engine (their device arenas are freed)."""
    _ENGINES.clear()
    try:
        import torch
        if torch.cuda.is_available():
            torch.cuda.empty_cache()
    except ImportError:  # pragma: no cover
        pass


def _kcap_key(kcap):
    """Hashable form of a rank capacity (an int, or a per-level profile)."""
    return int(kcap) if isinstance(kcap, (int, np.integer)) else tuple(int(k) for k in kcap)


def engine_for(tree: PartitionTree, batch=1, eps=1e-10, absolute=False, kcap=512, use_graph=True):
    key = (tuple(tree.leaf_sizes), batch, float(eps), bool(absolute), _kcap_key(kcap), use_graph)
    eng = _ENGINES.get(key)
    if eng is not None:
        _ENGINES.move_to_end(key)
        return eng
    while len(_ENGINES) >= max(1, MAX_ENGINES):
        _ENGINES.popitem(last=False)
        import torch
        torch.cuda.empty_cache()
    eng = HQREngine(tree, batch, eps, absolute, kcap, use_graph=use_graph)
    _ENGINES[key] = eng
    return eng


def hqr(a: HodlrMatrix, eps: float, n_b: int = 32, absolute: bool = False,
        kcap: int = 512) -> HodlrQRFactors:
    """QR of a square HODLR matrix on the B200 (reference hqr.py:80-92).

    eps is relative (thresholds eps*||A||_2 for intermediate sums, plain eps
    for T's coupling blocks) unless ``absolute``.  ``n_b`` is accepted for
    signature compatibility; the device panel width is fixed (16).
    """
    if n_b < 1:
        raise ValueError("n_b must be >= 1")
    eng = engine_for(a.tree(), 1, eps, absolute, kcap)
    return eng.factorize([a])[0]


def hqr_rec(col, eps_abs: float, eps_plain: float, n_b: int = 32, kcap: int = 512):
    """One recursion on a structured block column [A; B; C] on the B200
    (reference hqr.py:95-194): returns (StructuredY, T, R), Y mirroring the
    column, T and R upper triangular HODLR of A's partition.  Intermediate
    sums are truncated at eps_abs, T's coupling blocks at eps_plain.  B and C
    enter the device plan as the outermost slabs of every compressed column;
    B is left-orthogonalized on the device (SVD basis: the product Y_b is the
    reference's, its factors may differ by an orthogonal change of basis)."""
    if n_b < 1:
        raise ValueError("n_b must be >= 1")
    if not hasattr(col, "a_tilde"):
        raise TypeError("hqr_rec expects a StructuredColumn")
    a = col.a_tilde
    b, c = col.b, np.asarray(col.c, dtype=float).reshape(-1, a.n)
    p = b.n_rows if b.rank > 0 else 0
    eng = _rec_engine(a.tree(), (p, b.rank) if p else None, c.shape[0], eps_plain, kcap)
    eng.eps_abs = float(eps_abs)
    f = eng.factorize([col])[0]
    yb = f.y_b if p else LowRankBlock(np.zeros((b.n_rows, 0)), np.zeros((0, a.n)), True)
    y = StructuredY(f.y, yb, getattr(f, "y_c", np.zeros((0, a.n))))
    return y, f.t, f.r


def _rec_engine(tree, root_b, root_c, eps_plain, kcap):
    key = ("rec", tuple(tree.leaf_sizes), root_b, root_c, float(eps_plain), _kcap_key(kcap))
    eng = _ENGINES.get(key)
    if eng is not None:
        _ENGINES.move_to_end(key)
        return eng
    while len(_ENGINES) >= max(1, MAX_ENGINES):
        _ENGINES.popitem(last=False)
    torch = _require_cuda()
    from .plan import Builder
    bld = Builder(tree, 1, eps_plain, True, kcap, root_b=root_b, root_c=root_c).build()
    eng = HQREngine(tree, 1, eps_plain, True, kcap, builder=bld)
    _ENGINES[key] = eng
    del torch
    return eng


def hqr_batched(mats, eps: float, absolute: bool = False, kcap: int = 512):
    """Factor a batch of same-shape HODLR matrices in one graph replay."""
    if not mats:
        return []
    eng = engine_for(mats[0].tree(), len(mats), eps, absolute, kcap)
    return eng.factorize(list(mats))
