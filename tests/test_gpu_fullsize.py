"""Full-size BASELINE configurations on the GPU against the reference's own
results (tests/golden/make_golden_full.py ran the reference on the same
inputs): e_orth and e_acc within 10x the reference's, R within 100*tol
(relative Frobenius error of the sketch R @ G), all at full n."""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN
from paper_1809_10585_b200 import gen

pytestmark = pytest.mark.gpu


def golden_full(ci):
    p = os.path.join(GOLDEN, f"golden_full_cfg{ci}.npz")
    if not os.path.exists(p):
        pytest.skip(f"no golden vectors for config {ci}")
    return dict(np.load(p))


def ref_floor(ci):
    """The reference's own R reproducibility (n_b = 16 vs its default 32,
    tests/golden/make_floor_ref.py ran the reference)."""
    with open(os.path.join(GOLDEN, "golden_floor_ref.json")) as fh:
        return json.load(fh).get(str(ci), {}).get("r_sketch_nb16_vs_nb32", 0.0)


def log_result(rec):
    """Achieved errors of every full-size run: printed, and appended to
    gpurun_out/parity_fullsize.jsonl when that scratch directory exists."""
    print(json.dumps(rec))
    d = os.path.join(os.path.dirname(GOLDEN), "..", "gpurun_out")
    if os.path.isdir(d):
        with open(os.path.join(d, "parity_fullsize.jsonl"), "a") as fh:
            fh.write(json.dumps(rec) + "\n")


@pytest.mark.parametrize("ci", [0, 1, 2, 3, 4])
def test_full_config_vs_reference(ci):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_1809_10585_b200 import clear_engines, hqr, metrics
    from paper_1809_10585_b200.hodlr import stats
    from paper_1809_10585_b200.operators import QROperator
    g = golden_full(ci)
    c = gen.CONFIGS[ci]
    a = gen.gen_config(ci, seed=0)
    clear_engines()
    f = hqr(a, c["tol"])
    G = np.random.default_rng(0x5C37).standard_normal((a.n, 8))
    rg = QROperator(f).apply_r(G)
    rel = np.linalg.norm(rg - g["RG"]) / np.linalg.norm(g["RG"])
    # north star: R within 100*tol of the reference's R.  Where the reference
    # itself is not reproducible to that level (config 2, kappa ~1e17: its
    # own n_b = 16 and n_b = 32 runs differ by ~2e-3) the GPU must stay within
    # 10x the reference's own variation.
    floor = ref_floor(ci)
    bound = max(100 * c["tol"], 10 * floor)
    # e_orth / e_acc with the reference's _TIGHT estimator (bench.py:180) on
    # the GPU operators -- the same estimator that produced the golden values
    m = metrics(a, f, estimate=True)
    ranks = {k: stats(getattr(f, k))["max_offdiag_rank"] for k in ("y", "t", "r")}
    log_result(dict(config=ci, r_sketch_rel=float(rel), bound=bound, ref_floor=floor, e_orth=m["e_orth"],
                    e_orth_ref=float(g["e_orth"]), e_acc=m["e_acc"], e_acc_ref=float(g["e_acc"]), ranks=ranks,
                    ranks_ref=[int(g["rank_y"]), int(g["rank_t"]), int(g["rank_r"])]))
    assert rel <= bound, (rel, bound)
    assert m["e_orth"] <= 10 * max(float(g["e_orth"]), 1e-14), (m["e_orth"], float(g["e_orth"]))
    assert m["e_acc"] <= 10 * max(float(g["e_acc"]), 1e-14 * float(g["norm_est"])), (m["e_acc"], float(g["e_acc"]))
    # ranks of the factors stay within a few of the reference's
    for k, ref_rank in (("y", g["rank_y"]), ("t", g["rank_t"]), ("r", g["rank_r"])):
        assert ranks[k] <= int(ref_rank) + 8
    clear_engines()


def test_config3_retuned_engine_matches_reference():
    """Config 3 (n = 65536) factored twice through the same engine: the
    second run uses the Jacobi clusters re-tuned from the first run's core
    sizes (incl. 16-CTA clusters for the widest cores) and must still match
    the reference's R sketch."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_1809_10585_b200 import clear_engines
    from paper_1809_10585_b200.hqr import engine_for
    from paper_1809_10585_b200.operators import QROperator
    g = golden_full(3)
    c = gen.CONFIGS[3]
    a = gen.gen_config(3, seed=0)
    clear_engines()
    eng = engine_for(a.tree(), 1, c["tol"], False, 512)
    eng.factorize([a])
    clusters = [ex.get("cluster", 1) for k, _, ex in eng.builder.ops if k == "svd"]
    f = eng.factorize([a])[0]
    G = np.random.default_rng(0x5C37).standard_normal((a.n, 8))
    rel = np.linalg.norm(QROperator(f).apply_r(G) - g["RG"]) / np.linalg.norm(g["RG"])
    log_result(dict(config=3, retuned=True, r_sketch_rel=float(rel), clusters=sorted(set(clusters))))
    assert rel <= max(100 * c["tol"], 10 * ref_floor(3)), rel
    clear_engines()
