"""Edge cases of the reference's own test suite, run on the GPU through the
public API (pkg/tests/test_hqr.py, pkg/tests/test_acceptance.py):

  identity HODLR, every off-diagonal block rank 0     test_hqr.py:33
  dense equivalence at eps = 1e-15                    test_hqr.py:43, test_acceptance.py:45
  robustness to ill-conditioning (kappa up to 1e10)   test_hqr.py:227
  absolute thresholds (hqr(..., absolute=True))       hqr.py:80-92
  single leaf matrix (block_qr of the leaf)           test_hqr.py:82
"""

import numpy as np
import pytest

from oracle import hqr_oracle as O
from paper_1809_10585_b200 import gen
from paper_1809_10585_b200.hodlr import (HodlrMatrix, LowRankBlock, build_partition, hodlr_identity, stats,
                                         to_dense, validate_structure)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def hqr_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_1809_10585_b200 import hqr
    return hqr


def dense_q(f):
    y, t = to_dense(f.y), to_dense(f.t)
    return np.eye(y.shape[0]) - y @ t @ y.T


def plain_random_hodlr(n, n_min, rank, seed):
    """The reference bench generator's distribution (bench.py:75-104):
    N(0,1) leaves, off-diagonal blocks outer products of N(0,1) factors of
    the given rank, one PCG64 stream per block in HDLR1 order."""
    root = np.random.SeedSequence(seed)
    nxt = lambda: np.random.Generator(np.random.PCG64(root.spawn(1)[0]))

    def build(tr):
        if tr.level == 0:
            return HodlrMatrix(dense=nxt().standard_normal((tr.n, tr.n)))
        t1, t2 = tr.split()
        a11 = build(t1)
        g = nxt()
        a21 = LowRankBlock(g.standard_normal((t2.n, rank)), g.standard_normal((rank, t1.n)))
        g = nxt()
        a12 = LowRankBlock(g.standard_normal((t1.n, rank)), g.standard_normal((rank, t2.n)))
        return HodlrMatrix(a11=a11, a22=build(t2), a12=a12, a21=a21)

    return build(build_partition(n, n_min))


def host_from_dense(m, tree, eps):
    """Input construction (test side): per-block truncated SVD at eps."""
    if tree.level == 0:
        return HodlrMatrix(dense=m.copy())
    t1, t2 = tree.split()
    m1 = t1.n
    return HodlrMatrix(a11=host_from_dense(m[:m1, :m1], t1, eps), a22=host_from_dense(m[m1:, m1:], t2, eps),
                       a12=gen.compress_dense_block(m[:m1, m1:], eps),
                       a21=gen.compress_dense_block(m[m1:, :m1], eps))


def test_identity_rank_zero_blocks(hqr_gpu):
    n = 128
    f = hqr_gpu(hodlr_identity(build_partition(n, 32)), 1e-15)
    u = np.finfo(float).eps
    q = dense_q(f)
    assert np.linalg.norm(q.T @ q - np.eye(n), 2) <= n * u
    assert np.max(np.abs(np.abs(to_dense(f.r)) - np.eye(n))) <= n * u
    for h in (f.y, f.t, f.r):
        validate_structure(h)
        assert stats(h)["max_offdiag_rank"] == 0


@pytest.mark.parametrize("n,seed", [(256, 31), (128, 0), (128, 3), (256, 4), (512, 7), (512, 9)])
def test_dense_equivalence_eps_1e15(hqr_gpu, n, seed):
    """hqr at eps = 1e-15 reproduces the dense block QR's R (up to the
    diagonal signs): gap <= 1e-11 ||A||_2 (test_hqr.py:43) and the
    acceptance criterion's 1e-10 (test_acceptance.py:45)."""
    a = plain_random_hodlr(n, 32, 1, seed)
    d = to_dense(a)
    norm = np.linalg.norm(d, 2)
    f = hqr_gpu(a, 1e-15)
    _, _, r_ref = O.block_qr(d)
    gap = np.max(np.abs(np.abs(to_dense(f.r)) - np.abs(r_ref))) / norm
    assert gap <= 1e-11, gap


def test_robust_to_ill_conditioning(hqr_gpu):
    """Orthogonality does not grow with the condition number (kappa 1e2, 1e6,
    1e10): max e_orth <= 1e-10 and max/min <= 1e3 (test_hqr.py:227)."""
    rng = np.random.default_rng(40)
    n = 256
    tree = build_partition(n, 64)
    e_orths = []
    for kappa in (1e2, 1e6, 1e10):
        u = np.linalg.qr(rng.standard_normal((n, n)))[0]
        v = np.linalg.qr(rng.standard_normal((n, n)))[0]
        m = (u * np.logspace(0, -np.log10(kappa), n)) @ v.T
        h = host_from_dense(m, tree, 1e-13)
        f = hqr_gpu(h, 1e-13)
        q = dense_q(f)
        e_orths.append(np.linalg.norm(q.T @ q - np.eye(n), 2))
        e_acc = np.linalg.norm(q @ to_dense(f.r) - to_dense(h), 2)
        assert e_acc <= 1e-11, (kappa, e_acc)
    assert max(e_orths) <= 1e-10, e_orths
    assert max(e_orths) / min(e_orths) <= 1e3, e_orths


@pytest.mark.parametrize("eps", [1e-9, 1e-12])
def test_absolute_thresholds(hqr_gpu, eps):
    a = gen.gen_random_hodlr(512, 64, 8, 8.0, seed=11)
    f = hqr_gpu(a, eps, absolute=True)
    y, t, r = O.hqr(a, eps, absolute=True)
    rd, rr = to_dense(f.r), to_dense(r)
    assert np.linalg.norm(rd - rr) <= 100 * eps * np.linalg.norm(rr)
    assert abs(stats(f.r)["max_offdiag_rank"] - stats(r)["max_offdiag_rank"]) <= 2
    e_orth, e_acc = O.dense_metrics(to_dense(a), f.y, f.t, f.r)
    assert e_orth <= 1e-12 and e_acc <= 10 * eps * np.sqrt(512)


def test_single_leaf_matrix(hqr_gpu):
    m = np.random.default_rng(1234).standard_normal((48, 48))
    f = hqr_gpu(HodlrMatrix(dense=m), 1e-14)
    y_ref, t_ref, r_ref = O.block_qr(m)
    assert np.allclose(to_dense(f.r), r_ref)
    assert np.allclose(to_dense(f.y), y_ref)
    assert np.allclose(to_dense(f.t), t_ref)


def test_extreme_magnitudes_reflector_scaling(hqr_gpu):
    """Columns with entries near 1e-160 / 1e+160: the reflector scales by
    max|x| like the reference (dense.py:54-60) instead of under/overflowing."""
    for s in (1e-160, 1e160):
        m = np.random.default_rng(5).standard_normal((32, 32)) * s
        f = hqr_gpu(HodlrMatrix(dense=m), 1e-14, absolute=True)
        _, _, r_ref = O.block_qr(m)
        rd = to_dense(f.r)
        assert np.all(np.isfinite(rd))
        assert np.allclose(rd / s, r_ref / s, rtol=1e-12, atol=1e-12 * np.abs(r_ref / s).max())
