"""Each CUDA kernel of libhqb200.so against a numpy statement of its
contract (include/hodlrqr_b200.h), on odd / ragged / degenerate shapes."""

import numpy as np
import pytest

from emu import Emu  # noqa: F401  (numpy semantics reference lives in emu)
from paper_1809_10585_b200 import _abi

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    return torch, _abi.load()


def colmajor(torch, a):
    a = np.asarray(a, dtype=np.float64)
    return torch.tensor(a.T.copy(), device="cuda").contiguous()  # storage = a in column-major


def back(t, rows, cols):
    return t.cpu().numpy().reshape(cols, rows).T


def put(torch, arr):
    raw = np.frombuffer(arr.tobytes(), np.uint8)
    return torch.tensor(raw, device="cuda")


@pytest.mark.parametrize("tile", [32, 64])
@pytest.mark.parametrize("m,n,k,ta,tb", [(25, 3, 25, 0, 0), (25, 25, 6, 1, 0), (7, 33, 65, 0, 1),
                                         (130, 70, 19, 1, 1), (1, 1, 1, 0, 0), (257, 129, 300, 0, 0),
                                         (64, 64, 64, 1, 1)])
def test_gemm(dev, m, n, k, ta, tb, tile):
    torch, lib = dev
    rng = np.random.default_rng(m * 100 + n)
    A = rng.standard_normal((k, m) if ta else (m, k))
    B = rng.standard_normal((n, k) if tb else (k, n))
    C = rng.standard_normal((m, n))
    dA, dB, dC = colmajor(torch, A), colmajor(torch, B), colmajor(torch, C)
    rank = torch.zeros(4, dtype=torch.int32, device="cuda")
    terms = np.zeros(1, _abi.GEMM_TERM)
    terms[0] = (dA.data_ptr(), dB.data_ptr(), A.shape[0], B.shape[0], ta, tb, k, -1, 0, 0, -0.5)
    probs = np.zeros(1, _abi.GEMM_PROB)
    probs[0] = (dC.data_ptr(), m, m, -1, n, -1, 0, 1, 0, 2.0, 0, 0)
    dt, dp = put(torch, terms), put(torch, probs)
    tiles = -(-m // tile) * -(-n // tile)
    assert lib.hq_gemm_tiled(None, dp.data_ptr(), 1, dt.data_ptr(), rank.data_ptr(), tiles, 1, tile, None) == 0
    torch.cuda.synchronize()
    ref = 2.0 * C - 0.5 * ((A.T if ta else A) @ (B.T if tb else B))
    assert np.allclose(back(dC, m, n), ref, atol=1e-12 * max(1, np.abs(ref).max()))


def split_buffers(torch, slots, per, counters):
    """K-split workspace (slots x per doubles, NaN-filled: every slot a
    launch reads must have been written) and zeroed arrival counters."""
    ws = torch.full((max(slots * per, 1),), float("nan"), dtype=torch.float64, device="cuda")
    cnt = torch.zeros(max(counters, 1), dtype=torch.int32, device="cuda")
    return ws, cnt


@pytest.mark.parametrize("tile", [32, 64])
@pytest.mark.parametrize("m,n,k,ta,tb,ks,masks", [(100, 70, 300, 0, 0, 1, (1, 0)), (33, 90, 257, 1, 0, 3, (2, 0)),
                                                  (130, 20, 40, 0, 1, 1, (0, 1)), (64, 64, 512, 1, 1, 4, (0, 2)),
                                                  (40, 36, 4000, 1, 0, 16, (0, 0))])
def test_gemm_terms_masks(dev, m, n, k, ta, tb, ks, masks, tile):
    """hq_gemm_tiled: two terms (k-tiles of both stream through one pipeline),
    triangular masks, alpha, beta; K split into slices whose partial sums
    the last slice adds in slice order (bit-identical reruns, counters left
    at zero)."""
    torch, lib = dev
    rng = np.random.default_rng(m + 3 * n + 7 * k)
    A = rng.standard_normal((k, m) if ta else (m, k))
    B = rng.standard_normal((n, k) if tb else (k, n))
    A2 = rng.standard_normal((m, 21))
    B2 = rng.standard_normal((21, n))
    C = rng.standard_normal((m, n))
    dA, dB, dA2, dB2, dC = (colmajor(torch, x) for x in (A, B, A2, B2, C))
    rank = torch.zeros(4, dtype=torch.int32, device="cuda")
    terms = np.zeros(2, _abi.GEMM_TERM)
    terms[0] = (dA.data_ptr(), dB.data_ptr(), A.shape[0], B.shape[0], ta, tb, k, -1, masks[0], masks[1], 0.75)
    terms[1] = (dA2.data_ptr(), dB2.data_ptr(), m, 21, 0, 0, 21, -1, 0, 0, -1.0)
    tiles = -(-m // tile) * -(-n // tile)
    nkt = -(-k // 16) + -(-21 // 16)
    ks_cap = min(ks, max(1, nkt // 8))
    ws, cnt = split_buffers(torch, tiles * ks_cap, tile * tile, tiles)
    probs = np.zeros(1, _abi.GEMM_PROB)
    beta = 0.5
    probs[0] = (dC.data_ptr(), m, m, -1, n, -1, 0, 2, 0, beta, ws.data_ptr(), cnt.data_ptr())
    dt, dp = put(torch, terms), put(torch, probs)
    outs = []
    for _ in range(2):
        dC.copy_(colmajor(torch, C))
        assert lib.hq_gemm_tiled(None, dp.data_ptr(), 1, dt.data_ptr(), rank.data_ptr(), tiles, ks, tile, None) == 0
        torch.cuda.synchronize()
        outs.append(back(dC, m, n).copy())
    assert np.array_equal(outs[0], outs[1])
    assert int(cnt.abs().sum().item()) == 0

    def mask(x, mk):
        if mk == 1:
            return np.triu(x)
        if mk == 2:
            y = np.tril(x, -1)
            np.fill_diagonal(y, 1.0)
            return y
        return x
    opA = (mask(A, masks[0])).T if ta else mask(A, masks[0])
    opB = (mask(B, masks[1])).T if tb else mask(B, masks[1])
    ref = beta * C + 0.75 * (opA @ opB) - A2 @ B2
    assert np.allclose(outs[0], ref, atol=1e-11 * max(1, np.abs(ref).max()))


@pytest.mark.parametrize("mode", [0, 1, 2, 3, 4, 5])
@pytest.mark.parametrize("m,n,k,ta,tb,ks,masks", [(16, 2, 8192, 1, 0, 32, (0, 0)), (2, 2, 5000, 1, 0, 19, (0, 0)),
                                                  (256, 2, 256, 0, 0, 1, (1, 0)), (37, 3, 300, 1, 1, 1, (2, 0)),
                                                  (70, 4, 900, 0, 1, 4, (0, 0)), (5, 1, 3, 1, 0, 1, (0, 0)),
                                                  (600, 2, 40, 1, 0, 1, (0, 2)), (130, 2, 20000, 1, 0, 16, (0, 0))])
def test_gemm_skinny(dev, m, n, k, ta, tb, ks, masks, mode):
    """hq_gemm_skinny: two terms, masks, transposes, beta; split K with the
    deterministic slice-order reduction (bit-identical reruns)."""
    torch, lib = dev
    rng = np.random.default_rng(m * 7 + n + k)
    A = rng.standard_normal((k, m) if ta else (m, k))
    B = rng.standard_normal((n, k) if tb else (k, n))
    if (mode == 3 and ta) or (mode == 4 and not ta):
        pytest.skip("layout-specialised mode: every term must match it")
    if mode == 5 and not ta:
        pytest.skip("mode 5 problems are op(A) = A^T")
    ta2 = 1 if mode in (4, 5) else 0   # second term's layout (modes 4/5: all op(A) = A^T)
    A2 = rng.standard_normal((m, 5))
    B2 = rng.standard_normal((5, n))
    if mode == 1:
        ks = 1
    C = rng.standard_normal((m, n))
    dA, dB, dA2, dB2, dC = (colmajor(torch, x) for x in (A, B, A2.T if ta2 else A2, B2, C))
    rank = torch.zeros(4, dtype=torch.int32, device="cuda")
    terms = np.zeros(2, _abi.GEMM_TERM)
    terms[0] = (dA.data_ptr(), dB.data_ptr(), A.shape[0], B.shape[0], ta, tb, k, -1, masks[0], masks[1], 0.75)
    terms[1] = (dA2.data_ptr(), dB2.data_ptr(), 5 if ta2 else m, 5, ta2, 0, 5, -1, 0, 0, -1.0)
    nc = 2 if n <= 2 else 4
    if mode == 0:
        ws, cnt = split_buffers(torch, ks, m * n, 1)
    elif mode == 5:
        ws, cnt = split_buffers(torch, ks, m * nc, 1)
    else:
        ks_cap = min(ks, max(1, (k + 5) // 512))
        from paper_1809_10585_b200.plan import gv_rows
        R = gv_rows(m)   # output rows per CTA (launch max_rows = m)
        ws, cnt = split_buffers(torch, -(-m // R) * ks_cap, R * nc, -(-m // R))
    probs = np.zeros(1, _abi.GEMM_PROB)
    beta = 0.5
    probs[0] = (dC.data_ptr(), m, m, -1, n, -1, 0, 2, 0, beta, ws.data_ptr(), cnt.data_ptr())
    dt, dp = put(torch, terms), put(torch, probs)
    outs = []
    for _ in range(2):
        dC.copy_(colmajor(torch, C))
        assert lib.hq_gemm_skinny(None, dp.data_ptr(), 1, dt.data_ptr(), rank.data_ptr(), ks, n, mode, m, None) == 0
        torch.cuda.synchronize()
        outs.append(back(dC, m, n).copy())
    assert np.array_equal(outs[0], outs[1])
    assert int(cnt.abs().sum().item()) == 0

    def mask(x, mk):
        if mk == 1:
            return np.triu(x)
        if mk == 2:
            y = np.tril(x, -1)
            np.fill_diagonal(y, 1.0)
            return y
        return x
    opA = (mask(A, masks[0])).T if ta else mask(A, masks[0])
    opB = (mask(B, masks[1])).T if tb else mask(B, masks[1])
    ref = beta * C + 0.75 * (opA @ opB) - A2 @ B2
    assert np.allclose(outs[0], ref, atol=1e-11 * max(1, np.abs(ref).max()))


@pytest.mark.parametrize("cl", [1, 2, 8])
@pytest.mark.parametrize("m,k", [(25, 25), (28, 25), (9, 6), (300, 40), (50, 70), (1200, 17), (200, 200), (60, 57),
                                 (352, 256)])
def test_qr_and_applyq(dev, m, k, cl):
    torch, lib = dev
    rng = np.random.default_rng(m + 7 * k)
    A = rng.standard_normal((m, k))
    A[:, min(2, k - 1)] = 0.0  # a zero column
    dW = colmajor(torch, A)
    r = min(m, k)
    tau = torch.zeros(max(r, 1), dtype=torch.float64, device="cuda")
    tp = torch.zeros(((r + 15) // 16) * 256 + 2 * r * 16 + 256, dtype=torch.float64, device="cuda")
    tf = torch.full((r * r + 32 * r,), float("nan"), dtype=torch.float64, device="cuda")
    rank = torch.zeros(4, dtype=torch.int32, device="cuda")
    q = np.zeros(1, _abi.QR_PROB)
    q[0] = (dW.data_ptr(), tau.data_ptr(), tp.data_ptr(), tf.data_ptr(), m, r, m, -1, k, -1)
    dq = put(torch, q)
    assert lib.hq_qr(None, dq.data_ptr(), 1, rank.data_ptr(), cl) == 0
    torch.cuda.synchronize()
    W = back(dW, m, k)
    R = np.triu(W[:r])
    Y = np.tril(W[:, :r], -1)
    Y[np.arange(r), np.arange(r)] = 1.0
    assert torch.isnan(tf[r * r:]).all(), "QR wrote past the end of the T factor"
    T = np.triu(np.nan_to_num(back(tf[:r * r], r, r)))
    Q = np.eye(m) - Y @ T @ Y.T
    assert np.linalg.norm(Q.T @ Q - np.eye(m)) <= 1e-13 * m
    assert np.linalg.norm(Q[:, :r] @ R - A) <= 1e-13 * max(1, np.linalg.norm(A))
    # reference sign convention: R_jj = -sign(x0) * ||x||
    from oracle.hqr_oracle import block_qr
    Yr, Tr, Rr = block_qr(A, 32) if m >= k else (None, None, None)
    if Rr is not None:
        assert np.abs(R - Rr).max() <= 1e-11 * max(1, np.abs(Rr).max())
    # applyq: Q [X0; 0]
    c = 5
    X0 = rng.standard_normal((r, c))
    dX0 = colmajor(torch, X0)
    dX = torch.zeros(m * c, dtype=torch.float64, device="cuda")
    ap = np.zeros(1, _abi.APPLYQ_PROB)
    ap[0] = (dW.data_ptr(), tau.data_ptr(), tp.data_ptr(), dX.data_ptr(), dX0.data_ptr(), m, m, r,
             m, -1, k, -1, c, -1, r, -1, 0)
    da = put(torch, ap)
    assert lib.hq_applyq(None, da.data_ptr(), 1, rank.data_ptr(), c, m if cl != 2 else 0) == 0
    torch.cuda.synchronize()
    ref = Q[:, :r] @ X0
    assert np.abs(back(dX, m, c) - ref).max() <= 1e-12 * max(1, np.abs(ref).max())


@pytest.mark.parametrize("rows,ld,off,two", [(256, 256, 0, True), (255, 256, 0, False), (300, 302, 1, True),
                                             (64, 64, 2, False), (1, 2, 0, True)])
def test_concat(dev, rows, ld, off, two):
    """hq_concat: dst = [a1 P1 | a2 P2] (and the optional second copy), K into
    the rank table; 16-byte path (even rows / leading dims, aligned bases) and
    the element path (odd rows, odd offsets)."""
    torch, lib = dev
    rng = np.random.default_rng(rows + ld)
    c1, c2 = 5, 3
    P1 = rng.standard_normal((rows, c1)); P2 = rng.standard_normal((rows, c2))

    def dev_cols(x):
        buf = np.full(off + ld * x.shape[1] + 4, -3.0)
        for j in range(x.shape[1]):
            buf[off + j * ld: off + j * ld + rows] = x[:, j]
        return torch.tensor(buf, device="cuda")
    d1, d2 = dev_cols(P1), dev_cols(P2)
    dst = torch.full((off + ld * (c1 + c2) + 4,), -3.0, dtype=torch.float64, device="cuda")
    dst2 = torch.full((off + ld * (c1 + c2) + 4,), -3.0, dtype=torch.float64, device="cuda")
    rank = torch.zeros(4, dtype=torch.int32, device="cuda")
    rank[1] = c2
    pieces = np.zeros(2, _abi.PIECE)
    pieces[0] = (d1.data_ptr() + 8 * off, ld, c1, -1, 0, 0.5)
    pieces[1] = (d2.data_ptr() + 8 * off, ld, 7, 1, 0, -2.0)   # capacity 7, run-time 3 columns
    pr = np.zeros(1, _abi.CONCAT_PROB)
    pr[0] = (dst.data_ptr() + 8 * off, dst2.data_ptr() + 8 * off if two else 0, ld, ld, rows, 0, 2, 2)
    assert lib.hq_concat(None, put(torch, pr).data_ptr(), 1, put(torch, pieces).data_ptr(), rank.data_ptr(), rows) == 0
    torch.cuda.synchronize()
    assert int(rank[2].item()) == c1 + c2
    ref = np.concatenate([0.5 * P1, -2.0 * P2], axis=1)
    for d in ((dst, dst2) if two else (dst,)):
        o = d.cpu().numpy()
        got = np.stack([o[off + j * ld: off + j * ld + rows] for j in range(c1 + c2)], axis=1)
        assert np.array_equal(got, ref)
        o2 = o.copy()
        for j in range(c1 + c2):
            o2[off + j * ld: off + j * ld + rows] = -3.0
        assert (o2 == -3.0).all()


@pytest.mark.parametrize("trans,max_rows", [(0, None), (1, None), (0, 0), (1, 1024)])
@pytest.mark.parametrize("m,k,c,ldx,off", [(64, 48, 40, 64, 0), (65, 33, 7, 66, 0), (65, 33, 7, 65, 0),
                                            (200, 150, 70, 202, 1), (200, 150, 70, 200, 2), (2, 2, 3, 2, 0),
                                            (1, 1, 2, 2, 0), (511, 100, 33, 512, 0), (700, 40, 20, 700, 0)])
def test_applyq_in_place(dev, m, k, c, ldx, off, trans, max_rows):
    """X := Q X / Q^T X in place (x0 = NULL): the staged path moves the columns
    of X and of every reflector panel with bulk copies when their starts are
    16-byte aligned (even ld, even offset) and with element copies otherwise;
    odd row counts, rows > 512 (X left in global memory)."""
    # max_rows: the launch's row bound (None: exact; 0: unknown -> 512, taller
    # problems run from global memory; 1024: 8-column chunks, one panel buffer)
    max_rows = m if max_rows is None else max_rows
    torch, lib = dev
    rng = np.random.default_rng(m * 31 + k + c)
    A = rng.standard_normal((m, k))
    dW = colmajor(torch, A)
    r = min(m, k)
    tau = torch.zeros(max(r, 1), dtype=torch.float64, device="cuda")
    tp = torch.zeros(((r + 15) // 16) * 256 + 2 * r * 16 + 256, dtype=torch.float64, device="cuda")
    tf = torch.zeros(r * r + 32 * r, dtype=torch.float64, device="cuda")
    rank = torch.zeros(4, dtype=torch.int32, device="cuda")
    q = np.zeros(1, _abi.QR_PROB)
    q[0] = (dW.data_ptr(), tau.data_ptr(), tp.data_ptr(), tf.data_ptr(), m, r, m, -1, k, -1)
    assert lib.hq_qr(None, put(torch, q).data_ptr(), 1, rank.data_ptr(), 1) == 0
    torch.cuda.synchronize()
    W = back(dW, m, k)
    Y = np.tril(W[:, :r], -1)
    Y[np.arange(r), np.arange(r)] = 1.0
    T = np.triu(back(tf[:r * r], r, r))
    Q = np.eye(m) - Y @ T @ Y.T
    X = rng.standard_normal((m, c))
    buf = np.full(off + ldx * c + 8, 7.5)
    for j in range(c):
        buf[off + j * ldx: off + j * ldx + m] = X[:, j]
    dX = torch.tensor(buf, device="cuda")
    ap = np.zeros(1, _abi.APPLYQ_PROB)
    ap[0] = (dW.data_ptr(), tau.data_ptr(), tp.data_ptr(), dX.data_ptr() + 8 * off, 0, m, ldx, 0,
             m, -1, k, -1, c, -1, 0, -1, trans)
    assert lib.hq_applyq(None, put(torch, ap).data_ptr(), 1, rank.data_ptr(), c, max_rows) == 0
    torch.cuda.synchronize()
    out = dX.cpu().numpy()
    ref = (Q.T if trans else Q) @ X
    got = np.stack([out[off + j * ldx: off + j * ldx + m] for j in range(c)], axis=1)
    assert np.abs(got - ref).max() <= 1e-12 * max(1, np.abs(ref).max())
    # nothing outside the m x c block was touched
    out2 = out.copy()
    for j in range(c):
        out2[off + j * ldx: off + j * ldx + m] = 7.5
    assert (out2 == 7.5).all()


@pytest.mark.parametrize("xform,CL", [(0, 1), (1, 1), (1, 2), (1, 4), (1, 8), (1, 16), (0, 0), (1, 0)])
@pytest.mark.parametrize("m,n,keep", [(6, 6, 3), (25, 25, 25), (40, 13, 7), (13, 40, 9), (150, 150, 60),
                                      (200, 190, 120), (256, 256, 200), (130, 128, 128), (448, 448, 300),
                                      (600, 300, 250), (640, 200, 150), (48, 32, 20), (112, 36, 30),
                                      (128, 64, 50)])
def test_svd_truncation(dev, m, n, keep, xform, CL):
    if xform == 0 and m >= 150:
        pytest.skip("unpreconditioned Jacobi is not used by the plan at this size")
    if CL == 16 and m < 256:
        pytest.skip("16-CTA clusters carry only the widest cores")
    if CL == 0 and m > 256:
        pytest.skip("the small-core kernel carries cores of at most 128 rows (larger ones only as a fallback)")
    # CL = 0: the 128-thread small-core kernel; staging for cores of up to 4096
    # doubles, larger ones take its global-memory path
    SMALL = 4096
    # cluster launches pick one SM / the cluster / the global-memory path from
    # the run-time size, so every (size, cluster) combination must be exact
    MM = m
    torch, lib = dev
    rng = np.random.default_rng(m * n)
    u = np.linalg.qr(rng.standard_normal((m, min(m, n))))[0]
    v = np.linalg.qr(rng.standard_normal((n, min(m, n))))[0]
    s = np.logspace(0, -14, min(m, n))
    C = (u * s) @ v.T
    # threshold between sigma_keep-1 and sigma_keep (geometric mid-point: the
    # smallest kept sigma is ~1e-12 here, known to eps ||C|| absolutely)
    thr = float(np.sqrt(s[keep - 1] * s[keep])) if keep < len(s) else 0.0
    # xform=1 feeds R of C^T = Q R (the LQ preconditioner); X = R^T
    dC = colmajor(torch, np.linalg.qr(C.T)[1] if xform else C)
    ldc = min(m, n) if xform else m
    dW = torch.zeros(m * n, dtype=torch.float64, device="cuda")
    dU = torch.zeros(m * min(m, n), dtype=torch.float64, device="cuda")
    rank = torch.zeros(4, dtype=torch.int32, device="cuda")
    scal = torch.zeros(2, dtype=torch.float64, device="cuda")
    p = np.zeros(1, _abi.SVD_PROB)
    p[0] = (dC.data_ptr(), dU.data_ptr(), dW.data_ptr(), ldc, m, m, -1, n, -1, min(m, n), 0, 1, -1, thr, xform, 0)
    dp = put(torch, p)
    assert lib.hq_svd(None, dp.data_ptr(), 1, rank.data_ptr(), scal.data_ptr(), CL, MM, SMALL) == 0
    torch.cuda.synchronize()
    k = int(rank[0].item())
    assert k == min(keep, len(s))
    U = back(dU, m, min(m, n))[:, :k]
    assert np.linalg.norm(U.T @ U - np.eye(k)) <= 1e-12 * max(k, 1)
    # projection error of C onto span(U) equals the dropped tail (<= thr)
    err = np.linalg.norm(C - U @ (U.T @ C), 2)
    assert err <= thr * 1.0001 + 1e-12 * np.linalg.norm(C, 2)


@pytest.mark.parametrize("G,threads,smem", [(1, 256, None), (1, 512, None), (2, 512, None), (4, 256, None),
                                             (8, 512, None), (2, 512, "hdr"), (1, 256, "hdr")])
@pytest.mark.parametrize("m,n,keep", [(6, 6, 3), (25, 25, 25), (40, 13, 7), (13, 40, 9), (150, 150, 60),
                                      (200, 190, 120), (208, 208, 112), (97, 33, 30), (17, 17, 1),
                                      (300, 280, 150)])
def test_qrcp_then_svd(dev, m, n, keep, G, threads, smem):
    """hq_qrcp (pivoted R of the core, stopped at 1e-3 thr) followed by the
    xform-2 Jacobi on its rows: rank, orthogonality and projection error as
    for the unpivoted path; every cluster size, both thread counts, and the
    in-place global-memory mode (shared memory holds only the norms and the
    candidate buffers, which the caller must always provide)."""
    from paper_1809_10585_b200.plan import QRCP_SMEM_MAX, qrcp_smem
    torch, lib = dev
    rng = np.random.default_rng(m * n + 1)
    kk = min(m, n)
    u = np.linalg.qr(rng.standard_normal((m, kk)))[0]
    v = np.linalg.qr(rng.standard_normal((n, kk)))[0]
    s = np.logspace(0, -14, kk)
    C = (u * s) @ v.T                      # m x n; left singular vectors wanted
    thr = float(np.sqrt(s[keep - 1] * s[keep])) if keep < len(s) else 0.0
    # the pivoted QR works on C^T (n x m): its R rows transposed are X (m x r)
    dC = colmajor(torch, C.T.copy())
    need = qrcp_smem(G, n, m, threads)
    sm = need or QRCP_SMEM_MAX
    if smem == "hdr":   # room for the norms and candidates only: the slice stays in global memory
        sm = 8 + 2 * -(-m // G) + 2 * G * (((n + 1) & ~1) + 4) + 8
    dW = torch.zeros(((m + 1) // 2 * 2) * kk, dtype=torch.float64, device="cuda")
    dU = torch.zeros(m * kk, dtype=torch.float64, device="cuda")
    rank = torch.zeros(4, dtype=torch.int32, device="cuda")
    scal = torch.zeros(2, dtype=torch.float64, device="cuda")
    q = np.zeros(1, _abi.QRCP_PROB)
    q[0] = (dC.data_ptr(), n, n, -1, m, -1, 2, -1, 0, 1e-3 * thr)
    dq = put(torch, q)
    assert lib.hq_qrcp(None, dq.data_ptr(), 1, rank.data_ptr(), scal.data_ptr(), G, sm, threads) == 0
    torch.cuda.synchronize()
    r = int(rank[2].item())
    assert min(keep, kk) <= r <= kk
    p = np.zeros(1, _abi.SVD_PROB)
    p[0] = (dC.data_ptr(), dU.data_ptr(), dW.data_ptr(), n, m, m, -1, kk, 2, kk, 0, 1, -1, thr, 2, 0)
    dp = put(torch, p)
    assert lib.hq_svd(None, dp.data_ptr(), 1, rank.data_ptr(), scal.data_ptr(), 1, m, 0) == 0
    torch.cuda.synchronize()
    k = int(rank[0].item())
    assert k == min(keep, kk)
    U = back(dU, m, kk)[:, :k]
    assert np.linalg.norm(U.T @ U - np.eye(k)) <= 1e-12 * max(k, 1)
    err = np.linalg.norm(C - U @ (U.T @ C), 2)
    assert err <= thr * 1.001 + 1e-12 * np.linalg.norm(C, 2)
    # the rows kept are R of a pivoted QR: singular values of C up to the dropped block
    Rk = back(dC, n, m)[:r, :]
    sv = np.linalg.svd(Rk, compute_uv=False)
    assert np.abs(sv[:k] - s[:k]).max() <= 2e-3 * max(thr, 1e-13) + 1e-13


@pytest.mark.parametrize("xform,G", [(0, 1), (1, 1), (1, 2), (1, 4), (1, 8)])
@pytest.mark.parametrize("m,n,keep", [(6, 6, 3), (25, 25, 25), (40, 13, 7), (13, 40, 9), (150, 150, 60),
                                      (200, 190, 120), (256, 256, 200), (130, 128, 128), (448, 448, 300),
                                      (600, 300, 250), (640, 200, 150), (97, 33, 30), (17, 17, 1)])
def test_svd_block_truncation(dev, m, n, keep, xform, G):
    """hq_svd_block (block Jacobi on the tensor pipe): same contract as
    hq_svd -- rank by the threshold, orthonormal U_k spanning the kept
    singular subspace -- on graded spectra down to 1e-14."""
    if xform == 0 and m >= 150:
        pytest.skip("unpreconditioned cores this large are not issued by the plan")
    torch, lib = dev
    rng = np.random.default_rng(m * n + 11)
    u = np.linalg.qr(rng.standard_normal((m, min(m, n))))[0]
    v = np.linalg.qr(rng.standard_normal((n, min(m, n))))[0]
    s = np.logspace(0, -14, min(m, n))
    C = (u * s) @ v.T
    # threshold between sigma_keep-1 and sigma_keep (geometric mid-point: the
    # smallest kept sigma is ~1e-12 here, known to eps ||C|| absolutely)
    thr = float(np.sqrt(s[keep - 1] * s[keep])) if keep < len(s) else 0.0
    dC = colmajor(torch, np.linalg.qr(C.T)[1] if xform else C)
    ldc = min(m, n) if xform else m
    k_cols = min(m, n) if xform else n
    dW = torch.full((((m + 1) // 2 * 2) * k_cols,), float("nan"), dtype=torch.float64, device="cuda")
    dU = torch.zeros(m * min(m, n), dtype=torch.float64, device="cuda")
    rank = torch.zeros(4, dtype=torch.int32, device="cuda")
    scal = torch.zeros(2, dtype=torch.float64, device="cuda")
    p = np.zeros(1, _abi.SVD_PROB)
    p[0] = (dC.data_ptr(), dU.data_ptr(), dW.data_ptr(), ldc, m, m, -1, n, -1, min(m, n), 0, 1, -1, thr, xform, 0)
    dp = put(torch, p)
    assert lib.hq_svd_block(None, dp.data_ptr(), 1, rank.data_ptr(), scal.data_ptr(), G) == 0
    torch.cuda.synchronize()
    k = int(rank[0].item())
    assert int(rank[1].item()) == 0, "capacity flag"
    assert k == min(keep, len(s))
    U = back(dU, m, min(m, n))[:, :k]
    assert np.linalg.norm(U.T @ U - np.eye(k)) <= 1e-12 * max(k, 1)
    err = np.linalg.norm(C - U @ (U.T @ C), 2)
    assert err <= thr * 1.0001 + 1e-12 * np.linalg.norm(C, 2)
    # deterministic: a second launch gives the same U bit for bit
    U1 = back(dU, m, min(m, n)).copy()
    assert lib.hq_svd_block(None, dp.data_ptr(), 1, rank.data_ptr(), scal.data_ptr(), G) == 0
    torch.cuda.synchronize()
    assert np.array_equal(back(dU, m, min(m, n)), U1)
