"""The CPU oracle against the reference's own full-size results
(tests/golden/make_golden_full.py): the sketch R @ G of the oracle's R within
100*tol of the reference's, ranks within a few.  Configs 0 and 4 (n = 1024,
4096) run in seconds; the larger ones are covered on the GPU side
(test_gpu_fullsize.py) against the same golden files."""

import os

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import hqr_oracle as O
from paper_1809_10585_b200 import gen
from paper_1809_10585_b200.hodlr import stats


@pytest.mark.parametrize("ci", [0, 4])
def test_oracle_full_config_vs_reference(ci):
    g = dict(np.load(os.path.join(GOLDEN, f"golden_full_cfg{ci}.npz")))
    c = gen.CONFIGS[ci]
    a = gen.gen_config(ci, seed=0)
    y, t, r = O.hqr(a, c["tol"])
    G = np.random.default_rng(0x5C37).standard_normal((a.n, 8))
    rel = np.linalg.norm(O.happly(r, G) - g["RG"]) / np.linalg.norm(g["RG"])
    assert rel <= 100 * c["tol"], rel
    for f, key in ((y, "rank_y"), (t, "rank_t"), (r, "rank_r")):
        assert abs(stats(f)["max_offdiag_rank"] - int(g[key])) <= 4
