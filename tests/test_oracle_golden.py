"""Pin the CPU oracle against the reference's own outputs (golden vectors made
by tests/golden/make_golden.py from the reference package) and against the
reference tests' known-answer examples."""

import numpy as np
import pytest

from conftest import load_golden
from oracle import hqr_oracle as O
from paper_1809_10585_b200 import gen
from paper_1809_10585_b200.hodlr import LowRankBlock, stats, to_dense

BUILDERS = {
    "random_n256": lambda: gen.gen_random_hodlr(256, 32, 4, 8.0, seed=0),
    "illcond_n256": lambda: gen.gen_illcond_hodlr(256, 32, 4, 8.0, seed=1),
    "logkernel_n256": lambda: gen.gen_logkernel_hodlr(256, 32, 1e-10),
    "ragged_n200": lambda: gen.gen_random_hodlr(200, 24, 3, 8.0, seed=2),
    "leaf_n48": lambda: gen.gen_random_hodlr(48, 64, 1, 8.0, seed=3),
    "cfg0_n1024": lambda: gen.gen_config(0),
    "cfg4_n1024": lambda: gen.gen_random_hodlr(1024, 128, 16, 8.0, seed=5),
}


def test_householder_known_answers():
    # reference tests/test_dense_kernels.py: [3,4] -> y=[1,.5], gamma=1.6, rho=-5
    y, g, rho = O.householder([3.0, 4.0])
    assert np.allclose(y, [1.0, 0.5]) and g == pytest.approx(1.6) and rho == pytest.approx(-5.0)
    y, g, rho = O.householder([-3.0, 4.0])
    assert rho == pytest.approx(5.0)
    y, g, rho = O.householder(np.zeros(4))
    assert g == 0.0 and rho == 0.0
    assert O.householder([7.0])[2] == pytest.approx(-7.0)


def test_truncation_rank_known_answers():
    assert O.svd_rank([5, 1, 1e-12], 1e-10) == 2
    assert O.svd_rank([5], 10) == 0
    assert O.svd_rank([5, 1e-10], 1e-10) == 1   # ties truncate


def test_block_qr_matches_reference():
    g = load_golden("block_qr")
    Y, T, R = O.block_qr(g["A"], 8)
    s = np.linalg.norm(g["A"], 2)
    assert np.max(np.abs(R - g["R"])) <= 1e-13 * s
    assert np.max(np.abs(Y - g["Y"])) <= 1e-12
    assert np.max(np.abs(T - g["T"])) <= 1e-12


def test_block_qr_single_column():
    Y, T, R = O.block_qr(np.array([[3.0], [4.0]]))
    assert R[0, 0] == pytest.approx(-5.0) and T[0, 0] == pytest.approx(1.6)
    assert np.allclose(Y[:, 0], [1.0, 0.5])


def test_structured_column_matches_reference():
    g = load_golden("structured_col")
    h = gen.gen_random_hodlr(64, 16, 2, 8.0, seed=7)
    (ya, yb, yc), t, r = O.hqr_rec(h, LowRankBlock(g["bl"], g["br"]), g["c"], 1e-14, 1e-14)
    ydense = np.vstack([to_dense(ya), yb.to_dense(), yc])
    assert np.max(np.abs(to_dense(r) - g["R"])) <= 1e-11 * np.abs(g["R"]).max()
    assert np.max(np.abs(ydense - g["Y"])) <= 1e-10
    assert np.max(np.abs(to_dense(t) - g["T"])) <= 1e-10


@pytest.mark.parametrize("name", sorted(BUILDERS))
def test_hqr_oracle_matches_reference(name):
    g = load_golden(name)
    a = BUILDERS[name]()
    ad = to_dense(a)
    assert np.linalg.norm(ad) == pytest.approx(float(g["input_dense_fro"]), rel=1e-12)
    eps = float(g["eps"])
    assert O.hnorm2(a) == pytest.approx(float(g["norm_est"]), rel=1e-9)
    y, t, r = O.hqr(a, eps)
    rd = to_dense(r)
    # R agrees with the reference's R to 100*tol relative Frobenius (north star)
    if "R" in g:
        rel = np.linalg.norm(rd - g["R"]) / np.linalg.norm(g["R"])
        assert rel <= 100 * eps
        assert np.max(np.abs(to_dense(y) - g["Y"])) <= 1e3 * eps
    else:
        assert np.max(np.abs(np.diag(rd) - g["r_diag"])) <= 100 * eps * np.abs(g["r_diag"]).max()
    e_orth, e_acc = O.dense_metrics(ad, y, t, r)
    assert e_orth <= 10 * max(float(g["e_orth"]), 1e-15)
    assert e_acc <= 10 * max(float(g["e_acc"]), 1e-15)
    assert stats(y)["max_offdiag_rank"] == int(g["rank_y"])
    assert stats(r)["max_offdiag_rank"] == int(g["rank_r"])
    assert stats(t)["max_offdiag_rank"] == int(g["rank_t"])
