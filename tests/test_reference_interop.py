"""hqr accepts the reference package's own HodlrMatrix objects (duck-typed
boundary); checked here through the CPU kernel emulator.  Skipped where the
reference package is not mounted (it never is on the GPU box)."""

import os
import sys

import numpy as np
import pytest

from emu import emulate
from oracle import hqr_oracle as O
from paper_1809_10585_b200 import gen
from paper_1809_10585_b200.hodlr import to_dense

REF = "/root/reference/pkg/src"


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference package not mounted")
def test_reference_hodlr_matrix_is_accepted():
    sys.path.insert(0, REF)
    import hodlrqr as ref
    sys.path.insert(0, os.path.join(os.path.dirname(__file__), "golden"))
    from make_golden import to_ref
    a = gen.gen_random_hodlr(128, 32, 3, 8.0, seed=9)
    ra = to_ref(a)
    (f,), _, _ = emulate([ra], 1e-10)
    rf = ref.hqr(ra, 1e-10)
    rel = np.linalg.norm(to_dense(f.r) - ref.to_dense(rf.r)) / np.linalg.norm(ref.to_dense(rf.r))
    assert rel <= 1e-8
    e_orth, e_acc = O.dense_metrics(to_dense(a), f.y, f.t, f.r)
    assert e_orth <= 1e-13 and e_acc <= 1e-11
