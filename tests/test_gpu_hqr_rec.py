"""hqr_rec on general structured columns [A; B; C] on the GPU (reference
hqr.py:95-194; cases of pkg/tests/test_hqr.py:85-170): the reference's golden
vectors, reconstruction and orthogonality, and the oracle's R."""

import numpy as np
import pytest

from conftest import load_golden
from oracle import hqr_oracle as O
from paper_1809_10585_b200 import gen
from paper_1809_10585_b200.hodlr import LowRankBlock, to_dense, validate_structure

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def api():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1809_10585_b200 as P
    return P


def test_golden_structured_column(api):
    g = load_golden("structured_col")
    h = gen.gen_random_hodlr(64, 16, 2, 8.0, seed=7)
    col = api.StructuredColumn(h, LowRankBlock(g["bl"], g["br"]), g["c"])
    y, t, r = api.hqr_rec(col, 1e-14, 1e-14)
    for x in (y.y_a, t, r):
        validate_structure(x)
    assert np.linalg.norm(to_dense(r) - g["R"]) <= 1e-12 * np.linalg.norm(g["R"])
    assert np.linalg.norm(y.to_dense() - g["Y"]) <= 1e-11 * np.linalg.norm(g["Y"])
    assert np.linalg.norm(to_dense(t) - g["T"]) <= 1e-11 * np.linalg.norm(g["T"])


@pytest.mark.parametrize("m,p,k,r2,leaf", [(64, 3, 5, 0, 16), (64, 0, 0, 11, 16), (200, 35, 2, 9, 100),
                                           (40, 0, 0, 0, 40), (128, 20, 1, 6, 32), (1024, 40, 8, 16, 64)])
def test_structured_column_reconstruction(api, m, p, k, r2, leaf):
    rng = np.random.default_rng(m + p + r2)
    h = gen.gen_random_hodlr(m, leaf, 2, 0.0, seed=m)
    b = LowRankBlock(rng.standard_normal((p, k)), rng.standard_normal((k, m))) if p else \
        LowRankBlock(np.zeros((0, 0)), np.zeros((0, m)))
    col = api.StructuredColumn(h, b, rng.standard_normal((r2, m)))
    y, t, r = api.hqr_rec(col, 1e-14, 1e-14)
    stacked = np.vstack([to_dense(h), b.to_dense(), col.c])
    yd = y.to_dense()
    rows = stacked.shape[0]
    q = np.eye(rows) - yd @ to_dense(t) @ yd.T
    rebuilt = q @ np.vstack([to_dense(r), np.zeros((rows - m, m))])
    norm = np.linalg.norm(stacked, 2)
    assert np.linalg.norm(q.T @ q - np.eye(rows), 2) <= 1e-12
    assert np.linalg.norm(rebuilt - stacked, 2) <= 1e-11 * norm
    assert y.y_b.n_rows == p and y.y_c.shape == (r2, m)
    yo, to, ro = O.hqr_rec(h, b, col.c, 1e-14, 1e-14)
    assert np.max(np.abs(np.abs(to_dense(r)) - np.abs(to_dense(ro)))) <= 1e-11 * norm
