"""HODLR construction on the B200: the reference's from_dense / compress_block
(pkg/src/hodlrqr/core.py:178-215).

    from_dense(m, tree, tc)     every off-diagonal block of the partition
                                compressed by truncated SVD at tc.eps (absolute),
                                optionally capped at tc.rank_cap
    compress_block(block, tc)   one block: L = U_k (left-orthogonal),
                                R = Sigma_k V_k^T

All blocks of all tree levels are compressed in ONE batched recompression
(plan.Builder.trunc, the same kernels as the hQR truncations): a block B
(rows x cols) enters as the low-rank product B * I, so the pipeline's QR of
the factor stacks, Jacobi SVD of the core and right factor R = U_k^T B give
the truncated SVD of B with the reference's rank rule (sigma > eps).  The
dense matrix is uploaded once; the identity is formed on the device; the
diagonal leaves are the dense input's own diagonal blocks (copied on the host
like the reference's m[:m1, :m1].copy()).  Blocks wider than the device
Jacobi's 1024 columns (min(rows, cols) > 1024, i.e. n > 2048) are rejected.
"""

from __future__ import annotations

import numpy as np

from .hodlr import HodlrMatrix, LowRankBlock, PartitionTree, TruncationControl
from .plan import R_PERSIST, SVD_MAX_N, Builder, CompiledPlan, Dim, Tree


class CompressPlan:
    """Launch plan (buildable without CUDA) compressing sub-blocks
    (r0, c0, rows, cols) of one dense R x C matrix resident at D."""

    def __init__(self, R: int, C: int, blocks, eps: float, rank_cap=None):
        self.R, self.C, self.blocks = int(R), int(C), [tuple(int(x) for x in b) for b in blocks]
        bld = Builder(PartitionTree(0, (1,)), 1, 0.0, True, 1, io=False)
        self.builder = bld
        P = bld.bumps[R_PERSIST]
        self.D = P.alloc(self.R * self.C)
        maxc = max((b[3] for b in self.blocks), default=1)
        for (_, _, rows, cols) in self.blocks:
            if min(rows, cols) > SVD_MAX_N:
                raise ValueError(f"a {rows} x {cols} block is wider than the device SVD ({SVD_MAX_N} columns)")
        self.E = P.alloc(maxc * maxc)
        out = []
        ucap_tot = 0
        for (r0, c0, rows, cols) in self.blocks:
            cap = max(1, min(rows, cols))
            clamp = rank_cap is not None and rank_cap < cap
            if clamp:
                cap = int(rank_cap)
            out.append(dict(r0=r0, c0=c0, rows=rows, cols=cols, cap=cap, clamp=clamp, ri=bld.slots.take(),
                            U=P.alloc(rows * cap), V=P.alloc(cols * cap)))
            ucap_tot += (rows + cols) * cap
        self.out = out
        # identity (maxc x maxc): zero, then the unit-lower copy of itself
        bld.ops = []
        bld.zero([(self.E, maxc * maxc)])
        bld.op("copy", [(self.E, self.E, maxc, Dim(maxc), maxc, maxc, 2)])
        probs = []
        for o in out:
            if o["rows"] == 0 or o["cols"] == 0:
                continue
            probs.append(dict(m=o["rows"], n=o["cols"],
                              L=[(self.D + (o["r0"] + o["c0"] * self.R), self.R, Dim(o["cols"]), 1.0)],
                              R=[(self.E, maxc, Dim(o["cols"]), 1.0)],
                              eps_slot=-1, eps_scale=float(eps), U=(o["U"], o["rows"]), V=(o["V"], o["cols"]),
                              cap=o["cap"], rank_ri=o["ri"],
                              # rank_cap: clamp silently (core.py:210-211); else the
                              # capacity is the full rank and can never overflow
                              flag=-1 if o["clamp"] else bld.flag_slot))
        bld.trunc(probs)
        for b in bld.bumps.values():
            b.finalize()

    def assemble(self, U_of, V_of, rank_of):
        """LowRankBlock per block from accessors of the result buffers."""
        res = []
        for o in self.out:
            k = rank_of(o)
            if o["rows"] == 0 or o["cols"] == 0 or k == 0:
                res.append(LowRankBlock.zero(o["rows"], o["cols"]))
                continue
            res.append(LowRankBlock(U_of(o, k), V_of(o, k).T.copy(), left_orthogonal=True))
        return res


class _CompressEngine:
    def __init__(self, plan: CompressPlan, device=None):
        import torch
        from .hqr import _require_cuda
        _require_cuda()
        self.torch = torch
        self.p = plan
        self.device = torch.device(device if device is not None else "cuda")
        self.cp = CompiledPlan(plan.builder, self.device, alias_out=False)
        self.stream = torch.cuda.Stream(device=self.device)

    def run(self, m: np.ndarray):
        torch = self.torch
        p, cp = self.p, self.cp
        base = cp.bases[R_PERSIST]
        d0 = base + p.D.off
        h = torch.from_numpy(np.asfortranarray(m, dtype=np.float64).ravel(order="F")).pin_memory()
        with torch.cuda.stream(self.stream):
            cp.rank.zero_()
            cp.arena[d0:d0 + h.numel()].copy_(h, non_blocking=True)
            cp.run(self.stream.cuda_stream)
        self.stream.synchronize()
        rk = cp.rank.cpu().numpy()
        if rk[p.builder.flag_slot]:
            raise RuntimeError("rank capacity overflow in compress")   # cannot happen: capacity = full rank
        # one D2H of everything after the dense input (identity, U, V)
        e0 = base + p.E.off
        tail = cp.arena[e0:base + p.builder.bumps[R_PERSIST].peak].cpu().numpy()

        def view(buf, rows, k):
            o = buf.off - p.E.off
            return tail[o:o + rows * k].reshape((rows, k), order="F")
        return p.assemble(lambda o, k: view(o["U"], o["rows"], k).copy(),
                          lambda o, k: view(o["V"], o["cols"], k),
                          lambda o: int(min(max(rk[o["ri"]], 0), o["cap"])))


def _offdiag_blocks(tree: PartitionTree):
    """(node, kind, (r0, c0, rows, cols)) of every off-diagonal block."""
    t = Tree(tree)
    out = []
    for u in (t.internal_nodes((0, 0)) if t.L > 0 else []):
        c1, c2 = t.children(u)
        o1, o2, m1, m2 = t.off[c1], t.off[c2], t.size[c1], t.size[c2]
        out.append((u, "a12", (o1, o2, m1, m2)))
        out.append((u, "a21", (o2, o1, m2, m1)))
    return t, out


def from_dense(m, tree: PartitionTree, tc: TruncationControl, device=None) -> HodlrMatrix:
    """Compress a dense square matrix into HODLR form on the GPU
    (reference core.py:178-200): every off-diagonal block truncated by SVD,
    keeping the smallest rank whose tail singular value is <= tc.eps."""
    m = np.asarray(m, dtype=float)
    if m.ndim != 2 or m.shape[0] != m.shape[1]:
        raise ValueError("from_dense requires a square matrix")
    if m.shape[0] != tree.n:
        raise ValueError(f"matrix size {m.shape[0]} does not match tree size {tree.n}")
    t, blocks = _offdiag_blocks(tree)
    lr = {}
    if blocks:
        plan = CompressPlan(tree.n, tree.n, [b for _, _, b in blocks], tc.eps, tc.rank_cap)
        res = _CompressEngine(plan, device).run(m)
        lr = {(u, kind): r for (u, kind, _), r in zip(blocks, res)}

    def build(v):
        o, s = t.off[v], t.size[v]
        if t.is_leaf(v):
            return HodlrMatrix(dense=m[o:o + s, o:o + s].copy())
        c1, c2 = t.children(v)
        return HodlrMatrix(a11=build(c1), a22=build(c2), a12=lr[(v, "a12")], a21=lr[(v, "a21")])
    return build((0, 0))


def compress_block(block, tc: TruncationControl, device=None) -> LowRankBlock:
    """SVD-truncate a dense block to a left-orthogonal low-rank factorization
    on the GPU (reference core.py:203-215)."""
    block = np.asarray(block, dtype=float)
    rows, cols = block.shape
    if min(rows, cols) == 0:
        return LowRankBlock.zero(rows, cols)
    plan = CompressPlan(rows, cols, [(0, 0, rows, cols)], tc.eps, tc.rank_cap)
    return _CompressEngine(plan, device).run(block)[0]
