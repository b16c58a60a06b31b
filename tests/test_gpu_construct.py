"""GPU construction (from_dense / compress_block, reference core.py:178-215)
against host truncated SVDs, and the reference's ill-conditioning test
(test_hqr.py:227) built end to end on the GPU: from_dense -> hqr -> metrics."""

import numpy as np
import pytest

from paper_1809_10585_b200 import gen
from paper_1809_10585_b200.hodlr import TruncationControl, build_partition, stats, to_dense

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def api():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1809_10585_b200 as P
    return P


def host_blocks(h, out=None):
    out = [] if out is None else out
    if not h.is_leaf:
        out += [h.a12, h.a21]
        host_blocks(h.a11, out)
        host_blocks(h.a22, out)
    return out


@pytest.mark.parametrize("n,leaf,eps", [(256, 32, 1e-10), (1024, 64, 1e-8), (200, 24, 1e-12)])
def test_from_dense_matches_truncated_svd(api, n, leaf, eps):
    rng = np.random.default_rng(n)
    x = np.arange(n) / n
    m = np.log(np.abs(x[:, None] - (x[None, :] + 0.5 / n))) + 0.01 * rng.standard_normal((n, n)) * (eps * 1e3)
    tree = build_partition(n, leaf)
    h = api.from_dense(m, tree, TruncationControl(eps))
    assert h.tree().leaf_sizes == tree.leaf_sizes
    assert np.array_equal(to_dense(h)[:leaf, :leaf], m[:leaf, :leaf])
    # every block: the reference's rank rule and the truncated SVD's error
    ref = []

    def walk(o, s, t):
        if t.level == 0:
            return
        t1, t2 = t.split()
        ref.append(gen.compress_dense_block(m[o:o + t1.n, o + t1.n:o + s], eps))
        ref.append(gen.compress_dense_block(m[o + t1.n:o + s, o:o + t1.n], eps))
        walk(o, t1.n, t1)
        walk(o + t1.n, t2.n, t2)
    walk(0, n, tree)
    got = host_blocks(h)
    assert len(got) == len(ref)
    for g, r in zip(got, ref):
        assert abs(g.rank - r.rank) <= 1, (g.rank, r.rank)   # a sigma within rounding of eps may flip
        assert g.left_orthogonal
        if g.rank:
            assert np.allclose(g.L.T @ g.L, np.eye(g.rank), atol=1e-12)
    assert np.linalg.norm(to_dense(h) - m, 2) <= tree.level * eps * 1.01 + 1e-13 * np.linalg.norm(m, 2)


def test_compress_block_rank_cap(api):
    blk = np.random.default_rng(2).standard_normal((70, 50))
    lr = api.compress_block(blk, TruncationControl(1e-12, rank_cap=7))
    s = np.linalg.svd(blk, compute_uv=False)
    assert lr.rank == 7
    assert np.isclose(np.linalg.norm(blk - lr.to_dense(), 2), s[7], rtol=1e-9)


def test_ill_conditioning_end_to_end_on_gpu(api):
    """test_hqr.py:227 with the construction on the GPU too."""
    rng = np.random.default_rng(40)
    n = 256
    tree = build_partition(n, 64)
    e_orths = []
    for kappa in (1e2, 1e6, 1e10):
        u = np.linalg.qr(rng.standard_normal((n, n)))[0]
        v = np.linalg.qr(rng.standard_normal((n, n)))[0]
        m = (u * np.logspace(0, -np.log10(kappa), n)) @ v.T
        h = api.from_dense(m, tree, TruncationControl(1e-13))
        f = api.hqr(h, 1e-13)
        e_orths.append(api.metrics(h, f, estimate=False)["e_orth"])
    assert max(e_orths) <= 1e-10, e_orths
    assert max(e_orths) / min(e_orths) <= 1e3, e_orths
