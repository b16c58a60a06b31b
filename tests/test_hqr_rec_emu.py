"""hqr_rec on a general structured column [A; B; C] (reference hqr.py:95-194)
through the planner and the kernel emulator, against the reference's golden
vectors (tests/golden/make_golden.py ran hodlrqr.hqr_rec) and the oracle."""

import numpy as np
import pytest
import torch

from conftest import load_golden
from emu import Emu
from oracle import hqr_oracle as O
from paper_1809_10585_b200 import gen
from paper_1809_10585_b200.hodlr import HodlrMatrix, LowRankBlock, to_dense, validate_structure
from paper_1809_10585_b200.hqr import PlanIO, StructuredColumn, StructuredY
from paper_1809_10585_b200.plan import R_IN, R_OUT, R_PERSIST, Builder, CompiledPlan


def emulate_rec(col, eps_abs, eps_plain, kcap=512):
    a = col.a_tilde
    p = col.b.n_rows if col.b.rank > 0 else 0
    bld = Builder(a.tree(), 1, eps_plain, True, kcap, root_b=(p, col.b.rank) if p else None,
                  root_c=col.c.shape[0]).build()
    io = PlanIO(a.tree(), 1, eps_plain, True, kcap, builder=bld)
    io.eps_abs = eps_abs
    plan = CompiledPlan(bld, torch.device("cpu"))
    io.pack([col])
    A = plan.arena.numpy()
    ib, ob = plan.bases[R_IN], plan.bases[R_OUT]
    A[ib:ib + io.n_in] = io.inbuf[:io.n_in]
    pxo = plan.bases[R_PERSIST] + bld.PX.off
    A[pxo:pxo + io.px.size] = io.px
    plan.rank.numpy()[:] = io.rk
    plan.scal.numpy()[:] = io.sc
    Emu(plan).run()
    rk = plan.rank.numpy().copy()
    assert not rk[bld.flag_slot]
    out = A[ob:ob + int(plan.totals.numpy()[1])].copy()
    f = io.factors(0, out, rk)
    yb = f.y_b if p else LowRankBlock(np.zeros((col.b.n_rows, 0)), np.zeros((0, a.n)), True)
    return StructuredY(f.y, yb, getattr(f, "y_c", np.zeros((0, a.n)))), f.t, f.r


def reconstruction(col, y, t, r):
    stacked = np.vstack([to_dense(col.a_tilde), col.b.to_dense(), col.c])
    yd = y.to_dense()
    rows = stacked.shape[0]
    q = np.eye(rows) - yd @ to_dense(t) @ yd.T
    rebuilt = q @ np.vstack([to_dense(r), np.zeros((rows - col.a_tilde.n, col.a_tilde.n))])
    return stacked, q, rebuilt


def test_structured_column_matches_reference_golden():
    g = load_golden("structured_col")
    h = gen.gen_random_hodlr(64, 16, 2, 8.0, seed=7)
    col = StructuredColumn(h, LowRankBlock(g["bl"], g["br"]), g["c"])
    y, t, r = emulate_rec(col, 1e-14, 1e-14)
    validate_structure(y.y_a)
    validate_structure(t)
    validate_structure(r)
    assert np.linalg.norm(to_dense(r) - g["R"]) <= 1e-12 * np.linalg.norm(g["R"])
    assert np.linalg.norm(y.to_dense() - g["Y"]) <= 1e-11 * np.linalg.norm(g["Y"])
    assert np.linalg.norm(to_dense(t) - g["T"]) <= 1e-11 * np.linalg.norm(g["T"])


@pytest.mark.parametrize("m,p,k,r2,leaf", [(64, 3, 5, 0, 16), (64, 0, 0, 11, 16), (200, 35, 2, 9, 100),
                                           (40, 0, 0, 0, 40), (128, 20, 1, 6, 32)])
def test_structured_column_reconstruction(m, p, k, r2, leaf):
    """The reference's hqr_rec cases: overcomplete B (p < k), empty B with
    coupling rows, B and C together, the void column (= block_qr of the
    leaf): Q [R; 0] rebuilds [A; B; C] and Q is orthogonal."""
    rng = np.random.default_rng(m + p + r2)
    h = gen.gen_random_hodlr(m, leaf, 2, 0.0, seed=m)
    b = LowRankBlock(rng.standard_normal((p, k)), rng.standard_normal((k, m))) if p else \
        LowRankBlock(np.zeros((0, 0)), np.zeros((0, m)))
    col = StructuredColumn(h, b, rng.standard_normal((r2, m)))
    y, t, r = emulate_rec(col, 1e-14, 1e-14)
    stacked, q, rebuilt = reconstruction(col, y, t, r)
    norm = np.linalg.norm(stacked, 2)
    assert np.linalg.norm(q.T @ q - np.eye(q.shape[0]), 2) <= 1e-12
    assert np.linalg.norm(rebuilt - stacked, 2) <= 1e-11 * norm
    assert y.y_b.n_rows == p and y.y_c.shape == (r2, m)
    # against the oracle's hqr_rec (same recursion, numpy)
    yo, to, ro = O.hqr_rec(h, b, col.c, 1e-14, 1e-14)
    assert np.max(np.abs(np.abs(to_dense(r)) - np.abs(to_dense(ro)))) <= 1e-11 * norm
