"""The apply plans of paper_1809_10585_b200.operators checked without a GPU:
the packed launch sequence runs through the numpy kernel emulator and is
compared with the oracle's apply_q / apply_qt / happly (reference
hqr.py:197-216, arith.py:35-64)."""

import numpy as np
import pytest
import torch

from emu import Emu
from oracle import hqr_oracle as O
from paper_1809_10585_b200 import gen
from paper_1809_10585_b200.operators import (NARROW, WIDE, OperatorPlan, hodlr_sources, qr_kcap, qr_sources,
                                             _max_rank, spectral_norm_estimate_block)
from paper_1809_10585_b200.plan import R_IN, CompiledPlan


class EmuOperator:
    """OperatorPlan + CPU CompiledPlan + emulator (test harness)."""

    def __init__(self, tree, kcap, kinds, sources, ranks):
        self.op = OperatorPlan(tree, kcap, kinds)
        self.plan = CompiledPlan(self.op.builder, torch.device("cpu"), alias_out=False)
        A = self.plan.arena.numpy()
        ib = self.plan.bases[R_IN]
        rk = self.plan.rank.numpy()
        self.op.pack(sources, ranks, rk, lambda total: A[ib:ib + total])
        self.emu = Emu(self.plan)
        self.emu.run_ops(self.plan.launch[:1])

    def apply(self, kind, x):
        x = np.asarray(x, dtype=float)
        n, c = x.shape
        cap = NARROW if c <= NARROW else WIDE
        i0, i1, out = self.op.segments[(kind, cap)]
        p = self.plan
        p.rank.numpy()[self.op.col_slot[cap]] = c
        A = p.arena.numpy()
        xo = (p.addr(self.op.X) - p.arena.data_ptr()) // 8
        A[xo:xo + n * c] = x.ravel(order="F")
        self.emu.run_ops(p.launch[i0:i1])
        oo = (p.addr(out) - p.arena.data_ptr()) // 8
        return A[oo:oo + n * c].reshape((n, c), order="F").copy()


@pytest.fixture(scope="module")
def case():
    from emu import emulate
    a = gen.gen_random_hodlr(256, 32, 4, 8.0, seed=0)
    (f,), _, _ = emulate([a], 1e-10)
    return a, f


@pytest.mark.parametrize("c", [1, 2, 5])
def test_apply_q_and_qt_match_oracle(case, c):
    a, f = case
    tree = f.y.tree()
    from paper_1809_10585_b200.plan import Tree
    src, ranks = qr_sources(f, Tree(tree))
    op = EmuOperator(tree, qr_kcap(f), ("q", "qt", "r", "rt"), src, ranks)
    x = np.random.default_rng(c).standard_normal((a.n, c))
    for kind, ref in (("q", O.apply_q(f.y, f.t, x)), ("qt", O.apply_qt(f.y, f.t, x)),
                      ("r", O.happly(f.r, x)), ("rt", O.happly(f.r, x, True))):
        got = op.apply(kind, x)
        assert np.allclose(got, ref, atol=1e-12 * np.abs(ref).max()), kind
    # Q^T Q x = x and Q^T A x = R x (the factorization's contract)
    assert np.allclose(op.apply("qt", op.apply("q", x)), x, atol=1e-12)
    assert np.allclose(op.apply("qt", O.happly(a, x)), O.happly(f.r, x), atol=1e-8)


def test_hodlr_apply_matches_oracle(case):
    a, _ = case
    from paper_1809_10585_b200.plan import Tree
    src, ranks = hodlr_sources(a, Tree(a.tree()))
    op = EmuOperator(a.tree(), max(_max_rank(a), 1), ("a", "at"), src, ranks)
    x = np.random.default_rng(7).standard_normal((a.n, 3))
    assert np.allclose(op.apply("a", x), O.happly(a, x), atol=1e-11)
    assert np.allclose(op.apply("at", x), O.happly(a, x, True), atol=1e-11)


def test_block_power_iteration_matches_reference_rule(case):
    """Both vectors through the operator as one block give the reference's
    column-by-column estimate (dense.py:102-141)."""
    a, _ = case
    ref = O.norm2_estimate(lambda v: O.happly(a, v[:, None])[:, 0], lambda v: O.happly(a, v[:, None], True)[:, 0],
                           a.n, max_iter=300, tol=1e-6)
    got = spectral_norm_estimate_block(lambda x: O.happly(a, x), lambda x: O.happly(a, x, True), a.n,
                                       max_iter=300, tol=1e-6)
    assert abs(got - ref) <= 1e-12 * ref
