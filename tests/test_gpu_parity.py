"""GPU parity: the CUDA path (libhqb200.so through the public API) against the
CPU oracle and the reference's golden vectors."""

import numpy as np
import pytest

from conftest import load_golden
from oracle import hqr_oracle as O
from paper_1809_10585_b200 import gen
from paper_1809_10585_b200.hodlr import stats, to_dense, validate_structure

pytestmark = pytest.mark.gpu

CASES = {
    "random_n256": (lambda: gen.gen_random_hodlr(256, 32, 4, 8.0, seed=0), 1e-10),
    "illcond_n256": (lambda: gen.gen_illcond_hodlr(256, 32, 4, 8.0, seed=1), 1e-10),
    "logkernel_n256": (lambda: gen.gen_logkernel_hodlr(256, 32, 1e-10), 1e-10),
    "ragged_n200": (lambda: gen.gen_random_hodlr(200, 24, 3, 8.0, seed=2), 1e-12),
    "leaf_n48": (lambda: gen.gen_random_hodlr(48, 64, 1, 8.0, seed=3), 1e-14),
    "cfg0_n1024": (lambda: gen.gen_config(0), 1e-10),
    "cfg4_n1024": (lambda: gen.gen_random_hodlr(1024, 128, 16, 8.0, seed=5), 1e-10),
}


@pytest.fixture(scope="module")
def hqr_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_1809_10585_b200 import hqr
    return hqr


@pytest.mark.parametrize("name", sorted(CASES))
def test_gpu_matches_reference_golden(hqr_gpu, name):
    build, eps = CASES[name]
    g = load_golden(name)
    a = build()
    ad = to_dense(a)
    f = hqr_gpu(a, eps)
    validate_structure(f.y)
    validate_structure(f.t)
    validate_structure(f.r)
    e_orth, e_acc = O.dense_metrics(ad, f.y, f.t, f.r)
    # north star: within 10x the reference's value and at the tolerance's order
    assert e_orth <= 10 * max(float(g["e_orth"]), 1e-14)
    assert e_acc <= 10 * max(float(g["e_acc"]), 1e-14 * np.linalg.norm(ad, 2))
    rd = to_dense(f.r)
    if "R" in g:
        # dense R within 100*tol relative Frobenius of the reference's R
        assert np.linalg.norm(rd - g["R"]) / np.linalg.norm(g["R"]) <= 100 * eps
    else:
        assert np.max(np.abs(np.diag(rd) - g["r_diag"])) <= 100 * eps * np.abs(g["r_diag"]).max()


@pytest.mark.parametrize("name", ["random_n256", "illcond_n256", "cfg0_n1024"])
def test_gpu_matches_oracle(hqr_gpu, name):
    build, eps = CASES[name]
    a = build()
    f = hqr_gpu(a, eps)
    y, t, r = O.hqr(a, eps)
    rel = np.linalg.norm(to_dense(f.r) - to_dense(r)) / np.linalg.norm(to_dense(r))
    assert rel <= 100 * eps
    # truncation ranks agree with the oracle's to within a few
    for mine, ref in ((f.y, y), (f.t, t), (f.r, r)):
        assert abs(stats(mine)["max_offdiag_rank"] - stats(ref)["max_offdiag_rank"]) <= 4


def test_gpu_batched_results_independent_and_persistent(hqr_gpu):
    """A batch factorization returns each matrix's own factors (equal to the
    single-matrix run), and results stay valid across later calls that reuse
    the engine's pinned result blocks."""
    from paper_1809_10585_b200 import hqr_batched
    mats = [gen.gen_random_hodlr(512, 64, 8, 8.0, seed=s) for s in range(4)]
    fb = hqr_batched(mats, 1e-10)
    snap = [to_dense(f.r).copy() for f in fb]
    for a, f, rd in zip(mats, fb, snap):
        single = to_dense(hqr_gpu(a, 1e-10).r)
        assert np.linalg.norm(rd - single) <= 1e-12 * np.linalg.norm(single)
    for _ in range(3):  # later calls must not overwrite live results
        other = hqr_batched([gen.gen_random_hodlr(512, 64, 8, 8.0, seed=s + 10) for s in range(4)], 1e-10)
        del other
        fb2 = hqr_batched(mats, 1e-10)
        for f, rd in zip(fb, snap):
            assert np.array_equal(to_dense(f.r), rd)
        del fb2
    for i in range(3):
        assert np.linalg.norm(snap[i] - snap[i + 1]) > 1e-3 * np.linalg.norm(snap[i])


def test_gpu_factorize_stream_matches_factorize(hqr_gpu):
    """A stream_out engine's factorize_stream (batch i's copies overlapping
    batch i+1's device work) returns exactly the factors of separate
    factorize calls, for a sequence of different batches.  Both engines are
    warmed on the same batch first: an engine re-sizes its Jacobi / pivoted-QR
    launches once, from its first run's core sizes, and the launch shape fixes
    the summation orders (results are bit-identical per launch configuration)."""
    from paper_1809_10585_b200.hqr import HQREngine
    batches = [[gen.gen_random_hodlr(512, 64, 8, 8.0, seed=10 * i + s) for s in range(3)] for i in range(4)]
    ref_eng = HQREngine(batches[0][0].tree(), 3, 1e-10)
    ref_eng.factorize(batches[0])
    ref = [[to_dense(f.r) for f in ref_eng.factorize(bt)] for bt in batches]
    eng = HQREngine(batches[0][0].tree(), 3, 1e-10, stream_out=True)
    eng.factorize(batches[0])
    outs = list(eng.factorize_stream(batches))
    assert len(outs) == len(batches)
    for fs, rs in zip(outs, ref):
        for f, rd in zip(fs, rs):
            validate_structure(f.r)
            assert np.array_equal(to_dense(f.r), rd)
    # and again (graphs captured, pinned blocks recycled)
    outs2 = list(eng.factorize_stream(batches[::-1]))
    for fs, rs in zip(outs2, ref[::-1]):
        for f, rd in zip(fs, rs):
            assert np.array_equal(to_dense(f.r), rd)
