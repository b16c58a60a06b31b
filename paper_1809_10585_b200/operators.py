"""Device-resident HODLR operators on the B200: the "apply" half of the
reference API and the accuracy metrics built on it.

    apply_q(f, m)              Q M   = M - Y (T (Y^T M))      reference hqr.py:208-216
    apply_q_transpose(f, m)    Q^T M = M - Y (T^T (Y^T M))    reference hqr.py:197-205
    apply_dense(h, x)          H X                            reference arith.py:35-49
    apply_transpose_dense(h,x) H^T X                          reference arith.py:52-64
    metrics(a, f, estimate=True)  e_orth, e_acc by the reference's power
                               iteration on the implicitly applied operators
                               (bench.py:183-213, _TIGHT = 300 iterations, 1e-6)

A factor set is uploaded ONCE into a device layout (the factorization's own
layout, plan.Layout: leaves, U/V factors per node, rank table) and stays
resident; every apply is an H2D of the block M, one CUDA-graph replay of the
batched HODLR x dense launches (plan.Builder.happly: the V^T X products of
all tree levels in one launch, then one launch over the leaves adding the
U (V^T X) terms) and a D2H of the result.  There is no CPU fallback: without
a CUDA device or libhqb200.so these raise.
"""

from __future__ import annotations

import weakref
from collections import OrderedDict

import numpy as np

from .hodlr import HodlrMatrix
from .plan import R_IN, R_PERSIST, Buf, Builder, CompiledPlan, Dim

# column capacities of the compiled segments: vectors / 2-column blocks go
# through the streaming (HBM-bound) kernels, wider blocks through the DMMA
# GEMM tiles (chunks of WIDE columns)
NARROW, WIDE = 2, 64


def _max_rank(h: HodlrMatrix) -> int:
    if h.is_leaf:
        return 0
    return max(h.a12.rank, h.a21.rank, _max_rank(h.a11), _max_rank(h.a22))


def _nodes(h: HodlrMatrix, t):
    out = {}

    def walk(x, v):
        out[v] = x
        if not x.is_leaf:
            c1, c2 = t.children(v)
            walk(x.a11, c1)
            walk(x.a22, c2)
    walk(h, (0, 0))
    return out


class OperatorPlan:
    """Launch plan (no CUDA needed to build it) of the apply segments for one
    factor layout.

    kinds: "q", "qt" (sets Y and T), "r", "rt" (R), "a", "at" (A: a general
    HODLR matrix).  Factor sets in the layout: "A" (leaves, a12, a21), "Y"
    (unit lower leaves, a21 = A21U YV21^T), "T" (upper leaves in leafT,
    a12 = T12U T12V^T), "R" (upper leaves, a12).  Y and R share the leaf
    buffer (R on and above the diagonal, Y below: the kernels mask).  The
    first op restores the uploaded factor stream into the layout; segment
    (kind, cap) applies the operator to the block in X (cap columns of
    capacity, the run-time count in rank slot col_slot[cap])."""

    KINDS = {"q": ("Y", "T"), "qt": ("Y", "T"), "r": ("R",), "rt": ("R",), "a": ("A",), "at": ("A",)}

    def __init__(self, tree, kcap: int, kinds):
        bld = Builder(tree, 1, 0.0, True, max(1, kcap), io=False)
        self.builder = bld
        t, lay = bld.tree, bld.lay
        n = t.n
        self.n = n
        d = lay.m[0]
        P = bld.bumps[R_PERSIST]
        self.X = P.alloc(n * WIDE)
        self.W1 = P.alloc(n * WIDE)
        self.W2 = P.alloc(n * WIDE)
        self.col_slot = {c: bld.slots.take() for c in (NARROW, WIDE)}
        sets = sorted({s for k in kinds for s in self.KINDS[k]})
        self.sets = sets
        # input items (key, device buffer, rows, Dim cols) in stream order
        items = []
        for lf in t.leaves((0, 0)):
            nl = t.size[lf]
            if {"A", "Y", "R"} & set(sets):
                items.append((("leafA", lf), d["leafA"][lf], nl, Dim(nl)))
            if "T" in sets:
                items.append((("leafT", lf), d["leafT"][lf], nl, Dim(nl)))
        for u in (t.internal_nodes((0, 0)) if t.L > 0 else []):
            c1, c2 = t.children(u)
            m1, m2, kc = t.size[c1], t.size[c2], lay.kc[u]
            if "A" in sets or "R" in sets:
                items += [(("a12L", u), d["A12U"][u], m1, Dim(kc, d["rA12"][u])),
                          (("a12R", u), d["A12V"][u], m2, Dim(kc, d["rA12"][u]))]
            if "A" in sets:
                items += [(("a21L", u), d["A21U"][u], m2, Dim(kc, d["rA21"][u])),
                          (("a21R", u), d["A21V"][u], m1, Dim(kc, d["rA21"][u]))]
            if "Y" in sets:
                items += [(("y21L", u), d["A21U"][u], m2, Dim(kc, d["rA21"][u])),
                          (("y21R", u), d["YV21"][u], m1, Dim(kc, d["rA21"][u]))]
            if "T" in sets:
                items += [(("t12L", u), d["T12U"][u], m1, Dim(kc, d["rT12"][u])),
                          (("t12R", u), d["T12V"][u], m2, Dim(kc, d["rT12"][u]))]
        self.items = items
        bld.bumps[R_IN].alloc(sum(r * c.cap for _, _, r, c in items))
        bld.ops = []
        bld.op("pack_copy", [(buf, rows, cols) for _, buf, rows, cols in items],
               dict(which=1, base=Buf(R_IN, 0), total=0))
        self.segments = {}
        root = (0, 0)
        for kind in kinds:
            for cap in (NARROW, WIDE):
                i0 = len(bld.ops)
                nc = (cap, [self.col_slot[cap]])
                X, W1, W2 = [(self.X, n)], [(self.W1, n)], [(self.W2, n)]
                if kind in ("q", "qt"):
                    # X <- X - Y (T^op (Y^T X))
                    bld.happly(root, "Y", True, X, W1, nc)
                    bld.happly(root, "T", kind == "qt", W1, W2, nc)
                    bld.happly(root, "Y", False, W2, X, nc, alpha=-1.0, beta=1.0)
                    out = self.X
                else:
                    bld.happly(root, "R" if kind[0] == "r" else "A", kind.endswith("t"), X, W1, nc)
                    out = self.W1
                self.segments[(kind, cap)] = (i0, len(bld.ops), out)
        for b in bld.bumps.values():
            b.finalize()

    def pack(self, sources: dict, ranks: dict, rank_table: np.ndarray, dst_alloc):
        """Rank table entries + the packed factor stream (host).  ranks maps
        (slot name, node) -> rank; dst_alloc(total) returns a float64 array
        of >= total doubles to pack into.  Returns (array, total)."""
        lay = self.builder.lay
        d = lay.m[0]
        rank_table[:] = 0
        for (name, u), r in ranks.items():
            if r > lay.kc[u]:
                raise ValueError(f"factor rank {r} exceeds the layout capacity {lay.kc[u]}")
            rank_table[d[name][u]] = r
        cols = [dim.cap if dim.ri < 0 else int(rank_table[dim.ri]) for _, _, _, dim in self.items]
        total = sum(rows * c for (_, _, rows, _), c in zip(self.items, cols))
        hv = dst_alloc(max(total, 1))
        off = 0
        for (key, buf, rows, dim), c in zip(self.items, cols):
            if rows * c:
                np.copyto(hv[off:off + rows * c].reshape((rows, c), order="F"), sources[key])
            off += rows * c
        return hv, total


class _OperatorEngine:
    """An OperatorPlan compiled onto the GPU with its factors resident."""

    def __init__(self, tree, kcap: int, kinds, device=None):
        import torch
        from .hqr import _require_cuda
        _require_cuda()
        self.torch = torch
        self.device = torch.device(device if device is not None else "cuda")
        self.op = OperatorPlan(tree, kcap, kinds)
        self.builder, self.n = self.op.builder, self.op.n
        self.segments, self.col_slot, self.X = self.op.segments, self.op.col_slot, self.op.X
        n = self.n
        self.plan = CompiledPlan(self.builder, self.device, alias_out=False)
        self.stream = torch.cuda.Stream(device=self.device)
        self.graphs = {}
        p = self.plan
        ib = p.bases[R_IN]
        self.d_in = p.arena[ib:ib + max(self.builder.bumps[R_IN].peak, 1)]
        self.h_rank = torch.zeros_like(p.rank, device="cpu").pin_memory()
        self.h_x = torch.empty(n * WIDE, dtype=torch.float64, pin_memory=True)
        self.h_out = torch.empty(n * WIDE, dtype=torch.float64, pin_memory=True)

    # ------------------------------------------------------------------ upload
    def upload(self, sources: dict, ranks: dict):
        """One H2D of the packed factor stream, then the device-side restore
        into the layout (the plan's first op)."""
        torch = self.torch
        holder = {}

        def alloc(total):
            holder["h"] = torch.empty(total, dtype=torch.float64, pin_memory=True)
            return holder["h"].numpy()
        _, total = self.op.pack(sources, ranks, self.h_rank.numpy(), alloc)
        p = self.plan
        with torch.cuda.stream(self.stream):
            p.rank.copy_(self.h_rank, non_blocking=True)
            self.d_in[:total].copy_(holder["h"][:total], non_blocking=True)
            p.run(self.stream.cuda_stream, stop=1)
        self.stream.synchronize()

    # ------------------------------------------------------------------ apply
    def apply(self, kind: str, m: np.ndarray) -> np.ndarray:
        """kind in KINDS; m (n,) or (n, c).  Returns a new numpy array."""
        torch = self.torch
        m = np.asarray(m, dtype=np.float64)
        vec = m.ndim == 1
        x = m[:, None] if vec else m
        if x.ndim != 2 or x.shape[0] != self.n:
            raise ValueError("row counts do not match")
        c = x.shape[1]
        out = np.empty((self.n, c))
        for c0 in range(0, c, WIDE):
            cc = min(WIDE, c - c0)
            cap = NARROW if cc <= NARROW else WIDE
            out[:, c0:c0 + cc] = self._apply_chunk(kind, cap, x[:, c0:c0 + cc])
        return out[:, 0] if vec else out

    def _apply_chunk(self, kind, cap, x):
        torch = self.torch
        n, cc = x.shape
        i0, i1, outbuf = self.segments[(kind, cap)]
        p = self.plan
        hx = self.h_x.numpy()
        np.copyto(hx[:n * cc].reshape((n, cc), order="F"), x)
        rk = self.h_rank.numpy()
        rk[self.col_slot[cap]] = cc
        po = p.addr(outbuf) - p.arena.data_ptr()
        xo = p.addr(self.X) - p.arena.data_ptr()
        with torch.cuda.stream(self.stream):
            p.rank.copy_(self.h_rank, non_blocking=True)
            p.arena[xo // 8:xo // 8 + n * cc].copy_(self.h_x[:n * cc], non_blocking=True)
            g = self.graphs.get((kind, cap))
            if g is None:
                # first use: capture the segment (launch sequence fixed per plan)
                self.stream.synchronize()
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=self.stream):
                    p.run(self.stream.cuda_stream, start=i0, stop=i1)
                self.graphs[(kind, cap)] = g
            g.replay()
            self.h_out[:n * cc].copy_(p.arena[po // 8:po // 8 + n * cc], non_blocking=True)
        self.stream.synchronize()
        return self.h_out.numpy()[:n * cc].reshape((n, cc), order="F").copy()


def qr_sources(f, t_):
    """Factor-stream sources and ranks of hQR factors f for plan tree t_."""
    ny, nt, nr = _nodes(f.y, t_), _nodes(f.t, t_), _nodes(f.r, t_)
    src, ranks = {}, {}
    for lf in t_.leaves((0, 0)):
        src[("leafA", lf)] = np.triu(nr[lf].dense) + np.tril(ny[lf].dense, -1)
        src[("leafT", lf)] = nt[lf].dense
    for u in (t_.internal_nodes((0, 0)) if t_.L > 0 else []):
        ra, ya, ta = nr[u].a12, ny[u].a21, nt[u].a12
        src[("a12L", u)], src[("a12R", u)] = ra.L, ra.R.T
        src[("y21L", u)], src[("y21R", u)] = ya.L, ya.R.T
        src[("t12L", u)], src[("t12R", u)] = ta.L, ta.R.T
        ranks[("rA12", u)], ranks[("rA21", u)], ranks[("rT12", u)] = ra.rank, ya.rank, ta.rank
    return src, ranks


def hodlr_sources(h: HodlrMatrix, t_):
    """Factor-stream sources and ranks of a general HODLR matrix."""
    nd = _nodes(h, t_)
    src, ranks = {}, {}
    for lf in t_.leaves((0, 0)):
        src[("leafA", lf)] = nd[lf].dense
    for u in (t_.internal_nodes((0, 0)) if t_.L > 0 else []):
        a12, a21 = nd[u].a12, nd[u].a21
        src[("a12L", u)], src[("a12R", u)] = a12.L, a12.R.T
        src[("a21L", u)], src[("a21R", u)] = a21.L, a21.R.T
        ranks[("rA12", u)], ranks[("rA21", u)] = a12.rank, a21.rank
    return src, ranks


def qr_kcap(f) -> int:
    if not (f.y.same_structure(f.t) and f.y.same_structure(f.r)):
        raise ValueError("Y, T and R must share one partition tree")
    return max(_max_rank(f.y), _max_rank(f.t), _max_rank(f.r), 1)


class QROperator:
    """Q = I - Y T Y^T and R of an hQR factorization, resident on the GPU."""

    def __init__(self, f, device=None):
        self.n = f.y.n
        self.eng = _OperatorEngine(f.y.tree(), qr_kcap(f), ("q", "qt", "r", "rt"), device)
        self.eng.upload(*qr_sources(f, self.eng.builder.tree))

    def apply_q(self, m):
        return self.eng.apply("q", m)

    def apply_q_transpose(self, m):
        return self.eng.apply("qt", m)

    def apply_r(self, m):
        return self.eng.apply("r", m)

    def apply_r_transpose(self, m):
        return self.eng.apply("rt", m)


class HodlrOperator:
    """A general HODLR matrix resident on the GPU: H X and H^T X."""

    def __init__(self, h: HodlrMatrix, device=None):
        self.n = h.n
        self.eng = _OperatorEngine(h.tree(), max(_max_rank(h), 1), ("a", "at"), device)
        self.eng.upload(*hodlr_sources(h, self.eng.builder.tree))

    def matmat(self, x):
        return self.eng.apply("a", x)

    def rmatmat(self, x):
        return self.eng.apply("at", x)


# ---------------------------------------------------------------- module API
# operators of recently used factor sets / matrices (keyed by object
# identity, dropped when the object is collected or evicted)
_CACHE: "OrderedDict" = OrderedDict()
MAX_CACHED = 3


def _cached(obj, make):
    key = id(obj)
    hit = _CACHE.get(key)
    if hit is not None and hit[0]() is obj:
        _CACHE.move_to_end(key)
        return hit[1]
    op = make(obj)
    try:
        ref = weakref.ref(obj, lambda _r, k=key: _CACHE.pop(k, None))
    except TypeError:  # not weak-referenceable (e.g. __slots__ without __weakref__)
        ref = (lambda o=obj: o)
    _CACHE[key] = (ref, op)
    while len(_CACHE) > MAX_CACHED:
        _CACHE.popitem(last=False)
    return op


def qr_operator(f) -> QROperator:
    """The resident Q/R operator of factors f (uploaded on first use)."""
    return _cached(f, QROperator)


def hodlr_operator(h: HodlrMatrix) -> HodlrOperator:
    return _cached(h, HodlrOperator)


def _check_rows(f, m):
    m = np.asarray(m, dtype=float)
    if m.shape[0] != f.y.n:
        raise ValueError("row counts do not match")
    return m


def apply_q(f, m):
    """Q M = M - Y (T (Y^T M)) on the GPU (reference hqr.py:208-216)."""
    return qr_operator(f).apply_q(_check_rows(f, m))


def apply_q_transpose(f, m):
    """Q^T M = M - Y (T^T (Y^T M)) on the GPU (reference hqr.py:197-205)."""
    return qr_operator(f).apply_q_transpose(_check_rows(f, m))


def apply_dense(h: HodlrMatrix, x):
    """H @ x on the GPU (reference arith.py:35-49)."""
    x = np.asarray(x, dtype=float)
    if x.shape[0] != h.n:
        raise ValueError(f"dimension mismatch: {h.n} vs {x.shape[0]}")
    return hodlr_operator(h).matmat(x)


def apply_transpose_dense(h: HodlrMatrix, x):
    """H.T @ x on the GPU (reference arith.py:52-64)."""
    x = np.asarray(x, dtype=float)
    if x.shape[0] != h.n:
        raise ValueError(f"dimension mismatch: {h.n} vs {x.shape[0]}")
    return hodlr_operator(h).rmatmat(x)


def spectral_norm_estimate_block(apply_block, apply_t_block, n, max_iter=50, tol=1e-3):
    """||op||_2 by the reference's two-vector block power iteration on
    op^T op (dense.py:102-141): same start block, same Ritz-residual stop;
    both vectors go through the operator as one 2-column block."""
    if n <= 0:
        return 0.0
    rng = np.random.default_rng(0x5EED)
    x = np.linalg.qr(np.column_stack([np.full(n, 1.0 / np.sqrt(n)), rng.standard_normal(n)]))[0]
    est = 0.0
    for _ in range(max_iter):
        y = apply_block(x)
        lam, vecs = np.linalg.eigh(y.T @ y)
        theta = float(lam[-1])
        est = np.sqrt(max(theta, 0.0))
        if est == 0.0:
            return 0.0
        w = apply_t_block(y)
        g = vecs[:, -1]
        if np.linalg.norm(w @ g - theta * (x @ g)) <= 2.0 * tol * theta:
            return est
        q, _ = np.linalg.qr(w)
        if q.shape[1] < x.shape[1]:
            return est
        x = q
    return est


TIGHT = dict(max_iter=300, tol=1e-6)   # reference bench.py:180


def metrics(a, f, eps: float = 1e-10, estimate: bool = True, dense_limit: int = 4096) -> dict:
    """e_orth = ||Q^T Q - I||_2 and e_acc = ||Q R - A||_2 of factors f of a
    (reference bench.py:183-213).  estimate=True: the reference's power
    iteration (_TIGHT) on the operators applied on the GPU; estimate=False:
    dense evaluation on the host (n <= dense_limit), as the reference does."""
    n = f.y.n
    out = {"kappa2": float("nan"), "e_orth": float("nan"), "e_acc": float("nan")}
    if estimate:
        if not isinstance(a, HodlrMatrix):
            raise ValueError("estimate mode needs the HODLR input matrix")
        qo = qr_operator(f)
        ao = hodlr_operator(a)

        def qtq(v):
            return qo.apply_q_transpose(qo.apply_q(v)) - v

        def resid(v):
            return qo.apply_q(qo.apply_r(v)) - ao.matmat(v)

        def resid_t(v):
            return qo.apply_r_transpose(qo.apply_q_transpose(v)) - ao.rmatmat(v)

        out["e_orth"] = spectral_norm_estimate_block(qtq, qtq, n, **TIGHT)
        out["e_acc"] = spectral_norm_estimate_block(resid, resid_t, n, **TIGHT)
        return out
    if n > dense_limit:
        raise ValueError(f"n = {n} exceeds the densification limit {dense_limit}; pass estimate=True")
    from .hodlr import to_dense
    ad = to_dense(a) if isinstance(a, HodlrMatrix) else np.asarray(a, dtype=float)
    yd, td, rd = to_dense(f.y), to_dense(f.t), to_dense(f.r)
    q = np.eye(n) - yd @ td @ yd.T
    out["e_orth"] = float(np.linalg.norm(q.T @ q - np.eye(n), 2))
    out["e_acc"] = float(np.linalg.norm(q @ rd - ad, 2))
    out["kappa2"] = float(np.linalg.cond(ad, 2))
    return out
