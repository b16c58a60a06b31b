"""GPU construction plans (paper_1809_10585_b200.construct: from_dense /
compress_block, reference core.py:178-215) checked without a GPU through the
numpy kernel emulator."""

import numpy as np
import pytest
import torch

from emu import Emu
from paper_1809_10585_b200 import gen
from paper_1809_10585_b200.construct import CompressPlan, _offdiag_blocks
from paper_1809_10585_b200.hodlr import TruncationControl, build_partition
from paper_1809_10585_b200.plan import R_PERSIST, CompiledPlan


def emulate_compress(m, blocks, eps, rank_cap=None):
    p = CompressPlan(m.shape[0], m.shape[1], blocks, eps, rank_cap)
    cp = CompiledPlan(p.builder, torch.device("cpu"), alias_out=False)
    A = cp.arena.numpy()
    base = cp.bases[R_PERSIST]
    A[base + p.D.off:base + p.D.off + m.size] = m.ravel(order="F")
    Emu(cp).run()
    rk = cp.rank.numpy()

    def view(buf, rows, k):
        o = base + buf.off
        return A[o:o + rows * k].reshape((rows, k), order="F")
    return p.assemble(lambda o, k: view(o["U"], o["rows"], k).copy(), lambda o, k: view(o["V"], o["cols"], k),
                      lambda o: int(min(rk[o["ri"]], o["cap"])))


@pytest.mark.parametrize("eps", [1e-8, 1e-12])
def test_from_dense_blocks_match_truncated_svd(eps):
    rng = np.random.default_rng(0)
    n = 128
    u = np.linalg.qr(rng.standard_normal((n, n)))[0]
    v = np.linalg.qr(rng.standard_normal((n, n)))[0]
    m = (u * np.logspace(0, -12, n)) @ v.T
    tree = build_partition(n, 16)
    t, blocks = _offdiag_blocks(tree)
    res = emulate_compress(m, [b for _, _, b in blocks], eps)
    for (_, _, (r0, c0, rows, cols)), lr in zip(blocks, res):
        blk = m[r0:r0 + rows, c0:c0 + cols]
        ref = gen.compress_dense_block(blk, eps)
        assert lr.rank == ref.rank
        assert lr.left_orthogonal
        if lr.rank:
            assert np.allclose(lr.L.T @ lr.L, np.eye(lr.rank), atol=1e-12)
            # same truncated matrix (singular vector signs may differ)
            assert np.linalg.norm(lr.to_dense() - ref.to_dense(), 2) <= 1e-12 * np.linalg.norm(blk, 2)
            s = np.linalg.svd(blk, compute_uv=False)
            assert np.linalg.norm(blk - lr.to_dense(), 2) <= max(s[lr.rank] if lr.rank < len(s) else 0, 1e-15) * 1.0001


def test_rank_cap_clamps():
    rng = np.random.default_rng(1)
    blk = rng.standard_normal((40, 30))
    (lr,) = emulate_compress(blk, [(0, 0, 40, 30)], 1e-12, rank_cap=5)
    assert lr.rank == 5
    s = np.linalg.svd(blk, compute_uv=False)
    assert np.isclose(np.linalg.norm(blk - lr.to_dense(), 2), s[5], rtol=1e-10)


def test_zero_block_has_rank_zero():
    (lr,) = emulate_compress(np.zeros((20, 12)), [(0, 0, 20, 12)], 1e-12)
    assert lr.rank == 0 and lr.L.shape == (20, 0) and lr.R.shape == (0, 12)
