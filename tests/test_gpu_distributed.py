"""The partitioned single-matrix executor (distributed.py) on the GPU.  The
box has one GPU, so the world is one rank here: every op goes through the
executor's op-by-op path (same descriptors as the graph, no transfers) and
must reproduce hqr(); the 2-rank exchange itself is covered on CPU by
tests/test_distributed_gloo.py."""

import numpy as np
import pytest

from paper_1809_10585_b200 import gen
from paper_1809_10585_b200.hodlr import to_dense

pytestmark = pytest.mark.gpu


def test_dist_engine_one_rank_matches_hqr():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_1809_10585_b200 import hqr
    from paper_1809_10585_b200.distributed import DistEngine
    a = gen.gen_random_hodlr(1024, 64, 8, 8.0, seed=2)
    eng = DistEngine(a.tree(), 1e-10)
    assert not eng.sched.transfers()
    f = eng.factorize(a)
    ref = hqr(a, 1e-10)
    rd, rr = to_dense(f.r), to_dense(ref.r)
    assert np.linalg.norm(rd - rr) <= 1e-10 * np.linalg.norm(rr)
    f2 = eng.factorize(a)
    assert np.array_equal(to_dense(f2.r), rd)
