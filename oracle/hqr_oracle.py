"""numpy restatement of the reference hQR algorithm -- TEST INFRASTRUCTURE ONLY.

Restates (not copies) reference ``hodlrqr`` (pkg/src/hodlrqr/) on the host
containers of ``paper_1809_10585_b200.hodlr``.  Each function cites the
reference lines it follows.  Used as the parity checker for the CUDA path and
as the CPU baseline timed by bench.py; never used by the product path.
"""

from __future__ import annotations

import numpy as np

from paper_1809_10585_b200.hodlr import (UNIT_LOWER_TRIANGULAR, UPPER_TRIANGULAR,
                                         HodlrMatrix, LowRankBlock, hodlr_identity)


# ---------------------------------------------------------------- dense.py

def householder(v):
    """Reflector I - gamma y y^T with y[0] = 1 mapping v to rho e1,
    rho = -sign(v0)||v||, sign(0) = +1, zero vector -> gamma = 0.
    Follows dense.py:45-68 (scaled by max|v| against over/underflow)."""
    v = np.asarray(v, dtype=np.float64).ravel()
    if v.size == 0:
        raise ValueError("empty vector")
    y = np.zeros_like(v)
    y[0] = 1.0
    big = np.abs(v).max()
    if big == 0.0:
        return y, 0.0, 0.0
    w = v / big
    nw = np.sqrt(w @ w)
    s = -1.0 if v[0] < 0 else 1.0
    head = w[0] + s * nw
    y[1:] = w[1:] / head
    return y, 2.0 / (1.0 + y[1:] @ y[1:]), -s * big * nw


def svd_rank(sigma, eps):
    """Number of singular values strictly above eps (dense.py:93-99)."""
    return int(np.count_nonzero(np.asarray(sigma) > eps))


def norm2_estimate(op, op_t, n, max_iter=50, tol=1e-3):
    """Two-vector block power iteration on A^T A with Ritz-residual stop
    (dense.py:102-141): start = [ones/sqrt(n), PCG64(0x5EED) normal]."""
    if n <= 0:
        return 0.0
    g = np.random.default_rng(0x5EED)
    x = np.linalg.qr(np.column_stack([np.full(n, n ** -0.5), g.standard_normal(n)]))[0]
    est = 0.0
    for _ in range(max_iter):
        y = np.column_stack([op(x[:, i]) for i in range(x.shape[1])])
        lam, vec = np.linalg.eigh(y.T @ y)
        theta = float(lam[-1])
        est = np.sqrt(max(theta, 0.0))
        if est == 0.0:
            return 0.0
        w = np.column_stack([op_t(y[:, i]) for i in range(y.shape[1])])
        top = vec[:, -1]
        if np.linalg.norm(w @ top - theta * (x @ top)) <= 2.0 * tol * theta:
            return est
        q = np.linalg.qr(w)[0]
        if q.shape[1] < x.shape[1]:
            return est
        x = q
    return est


# ---------------------------------------------------------------- wy.py

def block_qr(a, nb=32):
    """Householder QR A = (I - Y T Y^T)[R; 0] with compact WY (Y, T).
    Same factors as wy.py:55-96 (Elmroth-Gustavson recursion); restated here as
    a left-to-right panel sweep: each panel of nb columns is reduced by the
    unblocked loop of wy.py:17-40, the trailing columns are updated with
    Q_p^T, and T is merged by T12 = -T1 (Y1^T Y2) T2 (wy.py:53)."""
    a = np.array(a, dtype=np.float64)
    m, n = a.shape
    if m < n or n < 1 or nb < 1:
        raise ValueError("block_qr requires rows >= cols >= 1 and nb >= 1")
    Y = np.zeros((m, n))
    T = np.zeros((n, n))
    for p in range(0, n, nb):
        q = min(p + nb, n)
        for j in range(p, q):
            y, gamma, rho = householder(a[j:, j])
            a[j, j] = rho
            a[j + 1:, j] = 0.0
            if gamma != 0.0 and j + 1 < q:
                a[j:, j + 1:q] -= gamma * np.outer(y, y @ a[j:, j + 1:q])
            Y[j:, j] = y
            T[p:j, j] = -gamma * (T[p:j, p:j] @ (Y[:, p:j].T @ Y[:, j]))
            T[j, j] = gamma
        if q < n:  # trailing update with Q_p^T = I - Y_p T_p^T Y_p^T
            yp = Y[:, p:q]
            a[:, q:] -= yp @ (T[p:q, p:q].T @ (yp.T @ a[:, q:]))
        if p > 0:
            T[:p, p:q] = -T[:p, :p] @ ((Y[:, :p].T @ Y[:, p:q]) @ T[p:q, p:q])
    return Y, T, np.triu(a[:n, :n])


# ---------------------------------------------------------------- core.py

def truncate(L, R, eps, left_orth=True):
    """Recompression T_eps: QR of L and R^T, SVD of R1 R2^T, keep sigma > eps
    (core.py:239-258).  Returns (L', R') with L' orthonormal."""
    L = np.asarray(L, dtype=np.float64)
    R = np.asarray(R, dtype=np.float64)
    if L.shape[1] == 0:
        return L, R
    q1, r1 = np.linalg.qr(L)
    q2, r2 = np.linalg.qr(R.T)
    u, s, vt = np.linalg.svd(r1 @ r2.T, full_matrices=False)
    k = svd_rank(s, eps)
    return q1 @ u[:, :k], (s[:k, None] * vt[:k]) @ q2.T


def left_orth(b: LowRankBlock) -> LowRankBlock:
    """Economy QR of L with R absorbed (core.py:229-236)."""
    if b.left_orthogonal or b.rank == 0:
        return b
    q, r = np.linalg.qr(b.L)
    return LowRankBlock(q, r @ b.R, True)


def trunc_block(b: LowRankBlock, eps) -> LowRankBlock:
    if b.rank == 0:
        return LowRankBlock(b.L, b.R, True)
    L, R = truncate(b.L, b.R, eps)
    return LowRankBlock(L, R, True)


# ---------------------------------------------------------------- arith.py

def happly(h: HodlrMatrix, x, trans=False):
    """H x (or H^T x) by recursive descent through the low-rank factors
    (arith.py:35-64)."""
    x = np.asarray(x, dtype=np.float64)
    if h.is_leaf:
        return (h.dense.T if trans else h.dense) @ x
    m1 = h.a11.n
    x1, x2 = x[:m1], x[m1:]
    if trans:
        top = happly(h.a11, x1, True) + h.a21.R.T @ (h.a21.L.T @ x2)
        bot = h.a12.R.T @ (h.a12.L.T @ x1) + happly(h.a22, x2, True)
    else:
        top = happly(h.a11, x1) + h.a12.L @ (h.a12.R @ x2)
        bot = h.a21.L @ (h.a21.R @ x1) + happly(h.a22, x2)
    return np.concatenate([top, bot], axis=0)


def hnorm2(h: HodlrMatrix, max_iter=50, tol=1e-3):
    """||H||_2 estimate with HODLR matvecs (arith.py:293-298)."""
    return norm2_estimate(lambda v: happly(h, v[:, None])[:, 0],
                          lambda v: happly(h, v[:, None], True)[:, 0], h.n, max_iter, tol)


def _add_trunc(b1: LowRankBlock, L2, R2, eps) -> LowRankBlock:
    if b1.rank == 0 and L2.shape[1] == 0:
        return b1
    return trunc_block(LowRankBlock(np.hstack([b1.L, L2]), np.vstack([b1.R, R2])), eps)


def lr_update(h: HodlrMatrix, u, v, eps) -> HodlrMatrix:
    """H + u v^T split over the tree, every touched block recompressed
    (arith.py:126-145)."""
    if u.shape[1] == 0:
        return h
    if h.is_leaf:
        return HodlrMatrix(dense=h.dense + u @ v.T)
    m1 = h.a11.n
    return HodlrMatrix(a11=lr_update(h.a11, u[:m1], v[:m1], eps),
                       a22=lr_update(h.a22, u[m1:], v[m1:], eps),
                       a12=_add_trunc(h.a12, u[:m1], v[m1:].T, eps),
                       a21=_add_trunc(h.a21, u[m1:], v[:m1].T, eps))


# ---------------------------------------------------------------- hqr.py

def _sum_trunc(terms, eps):
    """Left-to-right sum of low-rank terms, truncating after every addition
    (hqr.py:137-147 and 170-179)."""
    L, R = terms[0]
    for L2, R2 in terms[1:]:
        L, R = truncate(np.hstack([L, L2]), np.vstack([R, R2]), eps)
    return L, R


def hqr_rec(a: HodlrMatrix, b: LowRankBlock, c, eps_abs, eps_plain, nb=32):
    """One recursion of Algorithm 2 on the structured column [a; b; c]
    (hqr.py:95-194).  Returns ((y_a, y_b, y_c), t, r)."""
    b = left_orth(b)
    m = a.n
    c = np.asarray(c, dtype=np.float64).reshape(-1, m)
    k1 = b.rank
    if a.is_leaf:  # compressed column [A; B_R; C] (hqr.py:110-119)
        Y, T, R = block_qr(np.vstack([a.dense, b.R, c]), nb)
        return ((HodlrMatrix(dense=Y[:m], shape_tag=UNIT_LOWER_TRIANGULAR),
                 LowRankBlock(b.L, Y[m:m + k1], b.left_orthogonal), Y[m + k1:]),
                HodlrMatrix(dense=T, shape_tag=UPPER_TRIANGULAR),
                HodlrMatrix(dense=R, shape_tag=UPPER_TRIANGULAR))
    m1 = a.a11.n
    br1, br2 = b.R[:, :m1], b.R[:, m1:]
    c1, c2 = c[:, :m1], c[:, m1:]
    (ya11, ya21, yc_1), t1, r11 = hqr_rec(a.a11, a.a21, np.vstack([br1, c1]),
                                         eps_abs, eps_plain, nb)
    ybr1, yc1 = yc_1[:k1], yc_1[k1:]
    a12, a22 = a.a12, a.a22
    # S~ = Y1^T [A12; A22; B_R2; C2] as four low-rank terms (hqr.py:136-147)
    sL, sR = _sum_trunc([(happly(ya11, a12.L, True), a12.R),
                         (ya21.R.T, happly(a22, ya21.L, True).T),
                         (ybr1.T, br2), (yc1.T, c2)], eps_abs)
    sL = happly(t1, sL, True)                                   # S = T1^T S~
    a12_new = trunc_block(LowRankBlock(np.hstack([a12.L, -happly(ya11, sL)]),
                                       np.vstack([a12.R, sR])), eps_abs)
    cross = ya21.L @ (ya21.R @ sL)
    a22_new = lr_update(a22, -cross, sR.T, eps_abs)
    br2_new = br2 - (ybr1 @ sL) @ sR
    c2_new = c2 - (yc1 @ sL) @ sR
    (ya22, _, yc_2), t2, r22 = hqr_rec(a22_new, LowRankBlock.zero(0, a22_new.n),
                                       np.vstack([br2_new, c2_new]), eps_abs, eps_plain, nb)
    ybr2, yc2 = yc_2[:k1], yc_2[k1:]
    tL, tR = _sum_trunc([(ya21.R.T, happly(ya22, ya21.L, True).T),
                         (ybr1.T, ybr2), (yc1.T, yc2)], eps_plain)   # hqr.py:170-179
    t12 = LowRankBlock(-happly(t1, tL), happly(t2, tR.T, True).T)
    z = lambda r, cc: LowRankBlock.zero(r, cc)
    t = HodlrMatrix(a11=t1, a22=t2, a12=t12, a21=z(t2.n, t1.n), shape_tag=UPPER_TRIANGULAR)
    r = HodlrMatrix(a11=r11, a22=r22, a12=a12_new, a21=z(r22.n, r11.n), shape_tag=UPPER_TRIANGULAR)
    ya = HodlrMatrix(a11=ya11, a22=ya22, a21=ya21, a12=z(m1, ya22.n),
                     shape_tag=UNIT_LOWER_TRIANGULAR)
    return ((ya, LowRankBlock(b.L, np.hstack([ybr1, ybr2]), b.left_orthogonal),
             np.hstack([yc1, yc2])), t, r)


def hqr(a: HodlrMatrix, eps: float, nb: int = 32, absolute: bool = False):
    """(Y, T, R) with A ~= (I - Y T Y^T) R; thresholds eps*||A||_2 for the
    intermediate sums, plain eps for T's coupling blocks (hqr.py:80-92)."""
    eps_abs = eps if absolute else eps * hnorm2(a)
    (ya, _, _), t, r = hqr_rec(a, LowRankBlock.zero(0, a.n), np.zeros((0, a.n)),
                              eps_abs, eps, nb)
    return ya, t, r


def apply_qt(y, t, x):
    """Q^T X = X - Y T^T Y^T X (hqr.py:197-205)."""
    return x - happly(y, happly(t, happly(y, x, True), True))


def apply_q(y, t, x):
    """Q X = X - Y T Y^T X (hqr.py:208-216)."""
    return x - happly(y, happly(t, happly(y, x, True)))


def dense_metrics(a_dense, y, t, r):
    """e_orth = ||Q^T Q - I||_2, e_acc = ||QR - A||_2 (bench.py:219-223)."""
    from paper_1809_10585_b200.hodlr import to_dense
    n = a_dense.shape[0]
    yd = to_dense(y)
    q = np.eye(n) - yd @ to_dense(t) @ yd.T
    return (float(np.linalg.norm(q.T @ q - np.eye(n), 2)),
            float(np.linalg.norm(q @ to_dense(r) - a_dense, 2)))


__all__ = ["householder", "svd_rank", "norm2_estimate", "block_qr", "truncate",
           "left_orth", "happly", "hnorm2", "lr_update", "hqr_rec", "hqr",
           "apply_q", "apply_qt", "dense_metrics", "hodlr_identity"]
