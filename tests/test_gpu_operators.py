"""GPU apply_q / apply_q_transpose / apply_dense and metrics(estimate=True)
against the oracle and the reference's own test cases
(pkg/tests/test_hqr.py:184-205, pkg/src/hodlrqr/bench.py:183-213)."""

import numpy as np
import pytest

from conftest import load_golden
from oracle import hqr_oracle as O
from paper_1809_10585_b200 import gen
from paper_1809_10585_b200.hodlr import HodlrMatrix, LowRankBlock, build_partition, to_dense

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def api():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1809_10585_b200 as P
    return P


def rank1_pair(n, n_min, seed):
    """N(0,1) leaves and rank-1 off-diagonal blocks, with the dense matrix."""
    rng = np.random.default_rng(seed)

    def build(tr):
        if tr.level == 0:
            return HodlrMatrix(dense=rng.standard_normal((tr.n, tr.n)))
        t1, t2 = tr.split()
        a11 = build(t1)
        a21 = LowRankBlock(rng.standard_normal((t2.n, 1)), rng.standard_normal((1, t1.n)))
        a12 = LowRankBlock(rng.standard_normal((t1.n, 1)), rng.standard_normal((1, t2.n)))
        return HodlrMatrix(a11=a11, a22=build(t2), a12=a12, a21=a21)

    h = build(build_partition(n, n_min))
    return h, to_dense(h)


def test_apply_q_transpose_reduces_a(api):
    h, dense = rank1_pair(192, 48, 36)
    f = api.hqr(h, 1e-13)
    reduced = api.apply_q_transpose(f, dense)
    assert np.linalg.norm(reduced - to_dense(f.r), 2) <= 1e-10 * np.linalg.norm(dense, 2)


def test_apply_q_transpose_zero(api):
    h, _ = rank1_pair(64, 16, 37)
    f = api.hqr(h, 1e-13)
    assert np.array_equal(api.apply_q_transpose(f, np.zeros((64, 2))), np.zeros((64, 2)))


def test_apply_q_matches_dense_q(api):
    n = 512
    h, _ = rank1_pair(n, 64, 38)
    f = api.hqr(h, 1e-13)
    y, t = to_dense(f.y), to_dense(f.t)
    q = np.eye(n) - y @ t @ y.T
    v = np.random.default_rng(1234).standard_normal(n)
    assert np.allclose(api.apply_q(f, v), q @ v, atol=1e-11 * np.linalg.norm(v))
    assert np.allclose(api.apply_q_transpose(f, v), q.T @ v, atol=1e-11 * np.linalg.norm(v))
    assert api.apply_q(f, v).shape == (n,)


@pytest.mark.parametrize("c", [1, 2, 3, 64, 70])
def test_apply_matches_oracle(api, c):
    a = gen.gen_config(0)
    f = api.hqr(a, 1e-10)
    x = np.random.default_rng(c).standard_normal((a.n, c))
    for got, ref in ((api.apply_q(f, x), O.apply_q(f.y, f.t, x)),
                     (api.apply_q_transpose(f, x), O.apply_qt(f.y, f.t, x)),
                     (api.apply_dense(a, x), O.happly(a, x)),
                     (api.apply_transpose_dense(a, x), O.happly(a, x, True))):
        assert np.allclose(got, ref, atol=1e-12 * max(1.0, np.abs(ref).max()))


def test_metrics_estimate_on_gpu(api):
    """metrics(estimate=True): the reference's power-iteration metrics with
    every operator applied on the GPU, against the dense metrics (n = 1024)
    and the reference's golden values for the same input."""
    a = gen.gen_config(0)
    f = api.hqr(a, 1e-10)
    m = api.metrics(a, f, estimate=True)
    e_orth, e_acc = O.dense_metrics(to_dense(a), f.y, f.t, f.r)
    # a power iteration bounds the norm from below, up to the rounding of the
    # operator applications themselves -- which for e_orth (1.5e-14 here, a
    # rounding-level quantity) is a few per cent of the value: tolerance 10 %
    assert m["e_orth"] <= 1.10 * e_orth and m["e_orth"] >= 0.5 * e_orth
    assert m["e_acc"] <= 1.10 * e_acc and m["e_acc"] >= 0.5 * e_acc
    g = load_golden("full_cfg0")
    assert m["e_orth"] <= 10 * max(float(g["e_orth"]), 1e-14)
    assert m["e_acc"] <= 10 * float(g["e_acc"])
