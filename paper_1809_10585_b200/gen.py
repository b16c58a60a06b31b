"""Seeded synthetic HODLR inputs for the five BASELINE.json configurations.

These are input generators (host numpy), not part of the factorization path.
Every leaf and every off-diagonal block draws from its own PCG64 stream
spawned from ``SeedSequence(seed)`` in HDLR1 serialization order (a11
subtree, a21 block, a12 block, a22 subtree), following the reproducibility
rule of the reference generator (pkg/src/hodlrqr/bench.py:75-104).

Configs (BASELINE.json "configs"):
  0  random  n=1024  leaf 64   rank 8,  leaves N(0,1)+8I,  tol 1e-10
  1  logker  n=8192  leaf 256  A_ij = log|x_i - y_j| compressed by SVD at 1e-10*||A||
  2  illcond n=16384 leaf 256  rank 16, A = D B, D = diag(logspace(0,-14,n)) permuted
  3  large   n=65536 leaf 256  rank 32, leaves N(0,1)+16I, tol 1e-8
  4  batch   64 x n=4096 leaf 128 rank 16, seeds 0..63, tol 1e-10
"""

from __future__ import annotations

import numpy as np

from .hodlr import (HodlrMatrix, LowRankBlock, PartitionTree, TruncationControl,
                    build_partition)

CONFIGS = {
    0: dict(name="random_n1024", kind="random", n=1024, leaf=64, rank=8, diag=8.0, tol=1e-10),
    1: dict(name="logkernel_n8192", kind="logkernel", n=8192, leaf=256, tol=1e-10),
    2: dict(name="illcond_n16384", kind="illcond", n=16384, leaf=256, rank=16, diag=8.0, tol=1e-10),
    3: dict(name="large_n65536", kind="random", n=65536, leaf=256, rank=32, diag=16.0, tol=1e-8),
    4: dict(name="batch64_n4096", kind="random", n=4096, leaf=128, rank=16, diag=8.0, tol=1e-10,
            batch=64),
}


def _streams(seed):
    root = np.random.SeedSequence(seed)
    return lambda: np.random.Generator(np.random.PCG64(root.spawn(1)[0]))


def gen_random_hodlr(n: int, leaf: int, rank: int, diag: float, seed: int = 0) -> HodlrMatrix:
    """Leaves N(0,1) + diag*I; off-diagonal U V^T of the given rank with
    U, V i.i.d. N(0,1)/sqrt(block size)."""
    nxt = _streams(seed)

    def build(tr: PartitionTree) -> HodlrMatrix:
        if tr.level == 0:
            return HodlrMatrix(dense=nxt().standard_normal((tr.n, tr.n)) + diag * np.eye(tr.n))
        t1, t2 = tr.split()
        a11 = build(t1)
        g = nxt()
        a21 = LowRankBlock(g.standard_normal((t2.n, rank)) / np.sqrt(t2.n),
                           (g.standard_normal((t1.n, rank)) / np.sqrt(t1.n)).T)
        g = nxt()
        a12 = LowRankBlock(g.standard_normal((t1.n, rank)) / np.sqrt(t1.n),
                           (g.standard_normal((t2.n, rank)) / np.sqrt(t2.n)).T)
        a22 = build(t2)
        return HodlrMatrix(a11=a11, a22=a22, a12=a12, a21=a21)

    return build(build_partition(n, leaf))


def row_scale(h: HodlrMatrix, d: np.ndarray) -> HodlrMatrix:
    """D*H for diagonal D: scales leaves row-wise and the U (left) factors."""
    def sc(node, o):
        if node.is_leaf:
            return HodlrMatrix(dense=node.dense * d[o:o + node.n, None])
        m1 = node.a11.n
        return HodlrMatrix(
            a11=sc(node.a11, o), a22=sc(node.a22, o + m1),
            a12=LowRankBlock(node.a12.L * d[o:o + m1, None], node.a12.R),
            a21=LowRankBlock(node.a21.L * d[o + m1:o + node.n, None], node.a21.R))
    return sc(h, 0)


def gen_illcond_hodlr(n: int, leaf: int, rank: int, diag: float, seed: int = 0) -> HodlrMatrix:
    """A = D B, B random as gen_random_hodlr, D = diag(logspace(0,-14,n))
    in a seeded random order (condition number ~1e14)."""
    b = gen_random_hodlr(n, leaf, rank, diag, seed)
    perm = np.random.Generator(np.random.PCG64(np.random.SeedSequence([seed, 0xD1A6]))).permutation(n)
    return row_scale(b, np.logspace(0.0, -14.0, n)[perm])


def compress_dense_block(block: np.ndarray, eps_abs: float) -> LowRankBlock:
    """Truncated SVD factorization L = U_k, R = S_k V_k^T (sigma > eps_abs)."""
    if min(block.shape) == 0:
        return LowRankBlock.zero(*block.shape)
    u, s, vt = np.linalg.svd(block, full_matrices=False)
    k = int(np.sum(s > eps_abs))
    return LowRankBlock(u[:, :k].copy(), s[:k, None] * vt[:k], True)


def gen_logkernel_hodlr(n: int, leaf: int, tol: float = 1e-10) -> HodlrMatrix:
    """A_ij = log|x_i - y_j|, x_i = i/n, y_j = (j+0.5)/n; off-diagonal blocks
    compressed by truncated SVD at tol * ||A||_2 (||A||_2 from the dense
    matrix's power iteration -- a few matvecs)."""
    x = np.arange(n) / n
    y = (np.arange(n) + 0.5) / n

    def entries(r0, r1, c0, c1):
        return np.log(np.abs(x[r0:r1, None] - y[None, c0:c1]))

    # spectral norm of the full operator by power iteration on row blocks
    v = np.ones(n) / np.sqrt(n)
    est = 0.0
    for _ in range(30):
        w = np.concatenate([entries(i, min(i + 1024, n), 0, n) @ v for i in range(0, n, 1024)])
        wt = np.zeros(n)
        for i in range(0, n, 1024):
            wt += entries(i, min(i + 1024, n), 0, n).T @ w[i:i + 1024]
        new = np.sqrt(np.linalg.norm(wt))
        v = wt / np.linalg.norm(wt)
        if abs(new - est) <= 1e-6 * new:
            est = new
            break
        est = new
    eps_abs = tol * est

    def build(tr: PartitionTree, o: int) -> HodlrMatrix:
        if tr.level == 0:
            return HodlrMatrix(dense=entries(o, o + tr.n, o, o + tr.n))
        t1, t2 = tr.split()
        m = o + t1.n
        return HodlrMatrix(a11=build(t1, o), a22=build(t2, m),
                           a12=compress_dense_block(entries(o, m, m, o + tr.n), eps_abs),
                           a21=compress_dense_block(entries(m, o + tr.n, o, m), eps_abs))

    return build(build_partition(n, leaf), 0)


def gen_config(idx: int, seed: int = 0, n: int | None = None) -> HodlrMatrix:
    """Matrix of BASELINE config ``idx`` (optionally at a reduced size n)."""
    c = CONFIGS[idx]
    size = n if n is not None else c["n"]
    if c["kind"] == "logkernel":
        return gen_logkernel_hodlr(size, c["leaf"], c["tol"])
    if c["kind"] == "illcond":
        return gen_illcond_hodlr(size, c["leaf"], c["rank"], c["diag"], seed)
    return gen_random_hodlr(size, c["leaf"], c["rank"], c["diag"], seed)
