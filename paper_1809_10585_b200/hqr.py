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

import math
from dataclasses import dataclass

import numpy as np

from . import _abi
from .hodlr import (GENERAL, UNIT_LOWER_TRIANGULAR, UPPER_TRIANGULAR, HodlrMatrix, LowRankBlock,
                    PartitionTree)
from .plan import R_PERSIST, Builder, CompiledPlan


class RankCapacityError(RuntimeError):
    """A truncated rank exceeded the plan's rank capacity (raise kcap)."""


@dataclass
class HodlrQRFactors:
    """A ~= (I - Y T Y^T) R with all three factors sharing A's partition."""
    y: HodlrMatrix
    t: HodlrMatrix
    r: HodlrMatrix


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


class PlanIO:
    """Host side of a plan: packs inputs into the persistent-region image and
    assembles HodlrMatrix factors from a downloaded image (no CUDA needed)."""

    def __init__(self, tree: PartitionTree, batch: int = 1, eps: float = 1e-10,
                 absolute: bool = False, kcap: int = 512):
        self.tree, self.B, self.eps, self.absolute, self.kcap = tree, batch, eps, absolute, kcap
        self.builder = Builder(tree, batch, eps, absolute, kcap).build()
        self.n_persist = self.builder.bumps[R_PERSIST].peak
        self.img = np.zeros(self.n_persist)
        self.rk = np.zeros(max(self.builder.slots.n, 1), np.int32)
        self.sc = np.zeros(max(2 * batch, 2))

    # ---------------------------------------------------------------- host image
    def pack(self, mats):
        """Write the input matrices into the pinned host image."""
        if len(mats) != self.B:
            raise ValueError(f"expected {self.B} matrices, got {len(mats)}")
        img, rk = self.img, self.rk
        img[:] = 0.0
        rk[:] = 0
        t = self.builder.tree
        lay = self.builder.lay
        leaves = t.leaves((0, 0))
        for b, a in enumerate(mats):
            if tuple(a.leaf_sizes()) != tuple(self.tree.leaf_sizes):
                raise ValueError("matrix does not match the plan's partition tree")
            d = lay.m[b]

            def put(buf, arr):
                flat = np.asarray(arr, dtype=np.float64).ravel(order="F")
                img[buf.off:buf.off + flat.size] = flat

            def walk(h, v):
                if h.is_leaf:
                    put(d["leafA"][v], h.dense)
                    return
                c1, c2 = t.children(v)
                kc = lay.kc[v]
                for blk, U, V, R in ((h.a12, "A12U", "A12V", "rA12"), (h.a21, "A21U", "A21V", "rA21")):
                    if blk.rank > kc:
                        raise RankCapacityError(f"input block rank {blk.rank} exceeds capacity {kc}")
                    rows = blk.n_rows
                    cols = blk.n_cols
                    buf = d[U][v]
                    img[buf.off:buf.off + rows * blk.rank] = np.asarray(blk.L).ravel(order="F")
                    buf = d[V][v]
                    img[buf.off:buf.off + cols * blk.rank] = np.asarray(blk.R.T).ravel(order="F")
                    rk[d[R][v]] = blk.rank
                walk(h.a11, c1)
                walk(h.a22, c2)

            walk(a, (0, 0))
            n = t.n
            x0 = _start_vectors(n) if n >= 2 else np.ones((1, 2))
            off = self.builder.PX.off + 2 * n * b
            img[off:off + 2 * n] = x0.ravel(order="F")
        sc = self.sc
        sc[:] = 0.0
        if self.absolute:
            sc[1::2] = self.eps
            for b in range(self.B):
                rk[self.builder.power_done + b] = 1
            rk[self.builder.all_done] = 1
        del leaves

    def factors(self, b: int, img=None, rk=None) -> HodlrQRFactors:
        """Assemble the host HodlrMatrix factors of matrix b from an image."""
        t = self.builder.tree
        lay = self.builder.lay
        d = lay.m[b]

        def get(buf, rows, cols):
            return img[buf.off:buf.off + rows * cols].reshape((rows, cols), order="F").copy()

        def build(v, which):
            if t.is_leaf(v):
                nl = t.size[v]
                if which == "t":
                    return HodlrMatrix(dense=np.triu(get(d["leafT"][v], nl, nl)), shape_tag=UPPER_TRIANGULAR)
                full = get(d["leafA"][v], nl, nl)
                if which == "r":
                    return HodlrMatrix(dense=np.triu(full), shape_tag=UPPER_TRIANGULAR)
                y = np.tril(full, -1)
                np.fill_diagonal(y, 1.0)
                return HodlrMatrix(dense=y, shape_tag=UNIT_LOWER_TRIANGULAR)
            c1, c2 = t.children(v)
            m1, m2 = t.size[c1], t.size[c2]
            h1, h2 = build(c1, which), build(c2, which)
            zero12, zero21 = LowRankBlock.zero(m1, m2), LowRankBlock.zero(m2, m1)
            if which == "y":
                k = int(rk[d["rA21"][v]])
                a21 = LowRankBlock(get(d["A21U"][v], m2, k), get(d["YV21"][v], m1, k).T, True)
                return HodlrMatrix(a11=h1, a22=h2, a12=zero12, a21=a21, shape_tag=UNIT_LOWER_TRIANGULAR)
            if which == "t":
                k = int(rk[d["rT12"][v]])
                a12 = LowRankBlock(get(d["T12U"][v], m1, k), get(d["T12V"][v], m2, k).T)
            else:
                k = int(rk[d["rA12"][v]])
                a12 = LowRankBlock(get(d["A12U"][v], m1, k), get(d["A12V"][v], m2, k).T, True)
            return HodlrMatrix(a11=h1, a22=h2, a12=a12, a21=zero21, shape_tag=UPPER_TRIANGULAR)

        return HodlrQRFactors(y=build((0, 0), "y"), t=build((0, 0), "t"), r=build((0, 0), "r"))

class HQREngine(PlanIO):
    """PlanIO + device arena + CUDA graph for batched hQR of same-shape matrices."""

    def __init__(self, tree: PartitionTree, batch: int = 1, eps: float = 1e-10,
                 absolute: bool = False, kcap: int = 512, device=None, use_graph: bool = True):
        torch = _require_cuda()
        super().__init__(tree, batch, eps, absolute, kcap)
        self.torch = torch
        self.device = torch.device(device if device is not None else "cuda")
        self.plan = CompiledPlan(self.builder, self.device)
        pin = lambda a: torch.from_numpy(a).pin_memory()
        self.host_img, self.host_rank, self.host_scal = pin(self.img), pin(self.rk), pin(self.sc)
        self.img, self.rk, self.sc = self.host_img.numpy(), self.host_rank.numpy(), self.host_scal.numpy()
        self.out_img = torch.zeros(self.n_persist, dtype=torch.float64).pin_memory()
        self.out_rank = torch.zeros(self.plan.rank.numel(), dtype=torch.int32).pin_memory()
        self.use_graph = use_graph
        self.graph = None
        self.stream = torch.cuda.Stream(device=self.device)

    # ---------------------------------------------------------------- device
    def _launch(self):
        self.plan.run(self.stream.cuda_stream)

    def upload(self):
        p = self.plan
        with self.torch.cuda.stream(self.stream):
            p.arena[:self.n_persist].copy_(self.host_img, non_blocking=True)
            p.rank.copy_(self.host_rank, non_blocking=True)
            p.scal.copy_(self.host_scal, non_blocking=True)

    def execute(self):
        """Run the factorization on the device (graph replay when captured)."""
        torch = self.torch
        if not self.use_graph:
            self._launch()
            return
        if self.graph is None:
            # warm the library (function attributes) outside capture, then capture
            self.stream.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=self.stream):
                self._launch()
            self.graph = g
        with torch.cuda.stream(self.stream):
            self.graph.replay()

    def download(self):
        p = self.plan
        with self.torch.cuda.stream(self.stream):
            self.out_img.copy_(p.arena[:self.n_persist], non_blocking=True)
            self.out_rank.copy_(p.rank, non_blocking=True)
        self.stream.synchronize()
        if int(self.out_rank.numpy()[self.builder.flag_slot]) != 0:
            raise RankCapacityError(f"a truncated rank exceeded the capacity kcap={self.kcap}; "
                                    "retry with a larger kcap")

    def factors(self, b: int, img=None, rk=None) -> HodlrQRFactors:
        return PlanIO.factors(self, b, self.out_img.numpy() if img is None else img,
                              self.out_rank.numpy() if rk is None else rk)

    def norm_estimate(self, b: int = 0) -> float:
        """||A_b||_2 estimate of the last run (device power iteration)."""
        return float(self.plan.scal[2 * b].item())

    def factorize(self, mats):
        self.pack(mats)
        self.upload()
        self.execute()
        self.download()
        return [self.factors(b) for b in range(self.B)]



_ENGINES: dict = {}


def engine_for(tree: PartitionTree, batch=1, eps=1e-10, absolute=False, kcap=512, use_graph=True):
    key = (tuple(tree.leaf_sizes), batch, float(eps), bool(absolute), int(kcap), use_graph)
    eng = _ENGINES.get(key)
    if eng is None:
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


def hqr_batched(mats, eps: float, absolute: bool = False, kcap: int = 512):
    """Factor a batch of same-shape HODLR matrices in one graph replay."""
    if not mats:
        return []
    eng = engine_for(mats[0].tree(), len(mats), eps, absolute, kcap)
    return eng.factorize(list(mats))
