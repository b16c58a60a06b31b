"""Parity of exactly what bench.py times (config 2, n = 16384): the engine is
built by bench.build_engine -- the automatic batch (as many matrices as fit,
<= 74), the per-level rank capacity profile (bench.kcap_profile, at most 192),
streaming output, Jacobi / pivoted-QR clusters re-tuned after the first run
and the graph re-captured -- and its results are checked:

* matrix 0 against the reference's own full-size results
  (tests/golden/golden_full_cfg2.npz, produced by running hodlrqr): the R
  sketch within 10x the reference's own rounding floor (its n_b = 16 vs
  n_b = 32 variation, tests/golden/golden_floor_ref.json), e_orth and e_acc
  within 10x the reference's, estimated with the reference's _TIGHT power
  iteration (bench.py:180) on the GPU operators;
* other matrices of the batch against single-matrix runs of hqr();
* two replays of the timed graph are bit-identical (deterministic
  reductions), and factorize_stream (the e2e path) returns those factors.
"""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN
from paper_1809_10585_b200 import gen

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def bench_engine():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import bench
    from paper_1809_10585_b200 import clear_engines
    clear_engines()
    torch.cuda.empty_cache()
    eng, mats, kcap, _ = bench.build_engine(torch, 2, gen.CONFIGS[2]["n"])
    yield torch, eng, mats, kcap
    del eng
    torch.cuda.empty_cache()


def _floor():
    with open(os.path.join(GOLDEN, "golden_floor_ref.json")) as fh:
        return json.load(fh)["2"]


def test_timed_replays_are_bit_identical(bench_engine):
    torch, eng, mats, kcap = bench_engine
    assert max(np.atleast_1d(kcap)) == 192 and len(mats) >= 2
    assert any(ex.get("cluster", 1) != 1 for k, _, ex in eng.builder.ops if k == "svd")
    outs = []
    for _ in range(2):
        eng.restore_device_input()
        eng.execute()
        eng.download()
        outs.append(eng.h_out[:eng.n_out].clone())
    assert outs[0].numel() > 0
    assert torch.equal(outs[0], outs[1])


def test_timed_workload_matches_reference(bench_engine):
    torch, eng, mats, kcap = bench_engine
    import bench
    from paper_1809_10585_b200 import metrics
    from paper_1809_10585_b200.hodlr import stats
    g = dict(np.load(os.path.join(GOLDEN, "golden_full_cfg2.npz")))
    fs = next(iter(eng.factorize_stream([mats])))
    f0 = fs[0]
    rel = bench.r_sketch_error(f0, 2)
    floor = _floor()
    print(f"config 2 (bench engine, batch {len(mats)}): R-sketch rel. error {rel:.3e} "
          f"(reference n_b=16 vs 32: {floor['r_sketch_nb16_vs_nb32']:.3e})")
    assert rel <= max(100 * 1e-10, 10 * floor["r_sketch_nb16_vs_nb32"]), rel
    m = metrics(mats[0], f0, estimate=True)
    print(f"e_orth {m['e_orth']:.3e} (ref {float(g['e_orth']):.3e}), e_acc {m['e_acc']:.3e} "
          f"(ref {float(g['e_acc']):.3e})")
    assert m["e_orth"] <= 10 * max(float(g["e_orth"]), 1e-14)
    assert m["e_acc"] <= 10 * float(g["e_acc"])
    for k, ref_rank in (("y", g["rank_y"]), ("t", g["rank_t"]), ("r", g["rank_r"])):
        assert stats(getattr(f0, k))["max_offdiag_rank"] <= int(ref_rank) + 8


def test_other_matrices_match_single_runs(bench_engine):
    """Matrices 1 and B-1 of the timed batch equal their own batch-1 runs
    through hqr() to within the reference's rounding floor (the batch-1 plan
    picks other cluster sizes, i.e. other rounding)."""
    torch, eng, mats, kcap = bench_engine
    from paper_1809_10585_b200 import clear_engines, hqr
    from paper_1809_10585_b200.operators import QROperator
    fs = next(iter(eng.factorize_stream([mats])))
    G = np.random.default_rng(3).standard_normal((mats[0].n, 4))
    floor = _floor()["r_sketch_nb16_vs_nb32"]
    for i in sorted({1, len(mats) - 1}):
        rb = QROperator(fs[i]).apply_r(G)
        single = hqr(mats[i], gen.CONFIGS[2]["tol"], kcap=kcap)
        rs = QROperator(single).apply_r(G)
        clear_engines()
        rel = np.linalg.norm(rb - rs) / np.linalg.norm(rs)
        assert rel <= 10 * floor, (i, rel)
