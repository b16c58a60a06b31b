"""Full-size BASELINE configurations on the GPU against the reference's own
results (tests/golden/make_golden_full.py ran the reference on the same
inputs): e_orth and e_acc within 10x the reference's, R within 100*tol
(relative Frobenius error of the sketch R @ G), all at full n."""

import os

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import hqr_oracle as O
from paper_1809_10585_b200 import gen

pytestmark = pytest.mark.gpu


def golden_full(ci):
    p = os.path.join(GOLDEN, f"golden_full_cfg{ci}.npz")
    if not os.path.exists(p):
        pytest.skip(f"no golden vectors for config {ci}")
    return dict(np.load(p))


def estimate_metrics(a, f):
    """e_orth = ||Q^T Q - I||_2 and e_acc = ||QR - A||_2 by the reference's
    two-vector power iteration on HODLR applies (bench.py:196-213)."""
    n = a.n

    def qtq(v):
        x = v[:, None]
        return (O.apply_qt(f.y, f.t, O.apply_q(f.y, f.t, x)) - x)[:, 0]

    def res(v):
        x = v[:, None]
        return (O.apply_q(f.y, f.t, O.happly(f.r, x)) - O.happly(a, x))[:, 0]

    def res_t(v):
        x = v[:, None]
        return (O.happly(f.r, O.apply_qt(f.y, f.t, x), True) - O.happly(a, x, True))[:, 0]

    e_orth = O.norm2_estimate(qtq, qtq, n, max_iter=100, tol=1e-4)
    e_acc = O.norm2_estimate(res, res_t, n, max_iter=100, tol=1e-4)
    return e_orth, e_acc


@pytest.mark.parametrize("ci", [0, 1, 2, 3, 4])
def test_full_config_vs_reference(ci):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_1809_10585_b200 import hqr
    from paper_1809_10585_b200.hodlr import stats
    g = golden_full(ci)
    c = gen.CONFIGS[ci]
    a = gen.gen_config(ci, seed=0)
    f = hqr(a, c["tol"])
    G = np.random.default_rng(0x5C37).standard_normal((a.n, 8))
    rg = O.happly(f.r, G)
    rel = np.linalg.norm(rg - g["RG"]) / np.linalg.norm(g["RG"])
    # north star: R within 100*tol of the reference's R.  Where the reference
    # itself is not reproducible to that level (config 2, kappa ~1e17: its
    # numpy restatement differs by r_sketch_floor, tests/golden/oracle_floor.py)
    # the GPU must stay within 10x that rounding floor.
    bound = max(100 * c["tol"], 10 * float(g.get("r_sketch_floor", 0.0)))
    assert rel <= bound, (rel, bound)
    e_orth, e_acc = estimate_metrics(a, f)
    assert e_orth <= 10 * max(float(g["e_orth"]), 1e-14), (e_orth, float(g["e_orth"]))
    assert e_acc <= 10 * max(float(g["e_acc"]), 1e-14 * float(g["norm_est"])), (e_acc, float(g["e_acc"]))
    # ranks of the factors stay within a few of the reference's
    for k, ref_rank in (("y", g["rank_y"]), ("t", g["rank_t"]), ("r", g["rank_r"])):
        assert stats(getattr(f, k))["max_offdiag_rank"] <= int(ref_rank) + 8
