"""Host-side planner checked without a GPU: the packed launch sequence is
interpreted by the numpy kernel emulator (tests/emu.py) and compared with the
CPU oracle / reference golden vectors."""

import numpy as np
import pytest

from conftest import load_golden
from emu import emulate
from oracle import hqr_oracle as O
from paper_1809_10585_b200 import gen
from paper_1809_10585_b200.hodlr import stats, to_dense, validate_structure

CASES = {
    "random_n256": (lambda: gen.gen_random_hodlr(256, 32, 4, 8.0, seed=0), 1e-10),
    "illcond_n256": (lambda: gen.gen_illcond_hodlr(256, 32, 4, 8.0, seed=1), 1e-10),
    "ragged_n200": (lambda: gen.gen_random_hodlr(200, 24, 3, 8.0, seed=2), 1e-12),
    "leaf_n48": (lambda: gen.gen_random_hodlr(48, 64, 1, 8.0, seed=3), 1e-14),
}


@pytest.mark.parametrize("name", sorted(CASES))
def test_plan_matches_golden(name):
    build, eps = CASES[name]
    g = load_golden(name)
    a = build()
    (f,), io, plan = emulate([a], eps)
    for h in (f.y, f.t, f.r):
        validate_structure(h)
    rd = to_dense(f.r)
    assert np.linalg.norm(rd - g["R"]) / np.linalg.norm(g["R"]) <= 100 * eps
    e_orth, e_acc = O.dense_metrics(to_dense(a), f.y, f.t, f.r)
    assert e_orth <= 10 * max(float(g["e_orth"]), 1e-15)
    assert e_acc <= 10 * max(float(g["e_acc"]), 1e-15)
    assert stats(f.r)["max_offdiag_rank"] == int(g["rank_r"])
    assert stats(f.y)["max_offdiag_rank"] == int(g["rank_y"])


def test_plan_batched_matches_single():
    mats = [gen.gen_random_hodlr(128, 32, 3, 8.0, seed=s) for s in range(3)]
    fs, io, plan = emulate(mats, 1e-10)
    for a, f in zip(mats, fs):
        y, t, r = O.hqr(a, 1e-10)
        rel = np.linalg.norm(to_dense(f.r) - to_dense(r)) / np.linalg.norm(to_dense(r))
        assert rel <= 1e-8


def test_plan_absolute_eps():
    a = gen.gen_random_hodlr(128, 32, 3, 8.0, seed=4)
    (f,), io, plan = emulate([a], 1e-9, absolute=True)
    y, t, r = O.hqr(a, 1e-9, absolute=True)
    assert stats(f.r)["max_offdiag_rank"] == stats(r)["max_offdiag_rank"]
    assert np.linalg.norm(to_dense(f.r) - to_dense(r)) <= 1e-7 * np.linalg.norm(to_dense(r))


def test_rank_capacity_overflow_raises():
    a = gen.gen_random_hodlr(128, 32, 4, 8.0, seed=5)
    with pytest.raises(Exception):
        emulate([a], 1e-14, kcap=2)


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_multistream_schedule_is_hazard_free(seed):
    """Random interleavings allowed by the lane/event schedule give the same
    factorization as program order (a missed dependency would not)."""
    a = gen.gen_random_hodlr(256, 32, 4, 8.0, seed=0)
    (f0,), _, _ = emulate([a], 1e-10)
    (f1,), _, plan = emulate([a], 1e-10, interleave_seed=seed)
    assert plan.n_lanes > 1
    for k in ("y", "t", "r"):
        d0, d1 = to_dense(getattr(f0, k)), to_dense(getattr(f1, k))
        assert np.abs(d0 - d1).max() <= 1e-12 * max(1.0, np.abs(d0).max())


def test_tsqr_path_for_tall_factor_stacks(monkeypatch):
    """Force the one-level TSQR branch (chunk QRs, stacked R's, Q applied in
    two stages) on a small case and compare with the oracle."""
    import paper_1809_10585_b200.plan as PL
    monkeypatch.setattr(PL, "TALL_ROWS", 40)
    monkeypatch.setattr(PL, "TSQR_CH", 24)
    a = gen.gen_random_hodlr(256, 32, 4, 8.0, seed=0)
    (f,), io, plan = emulate([a], 1e-10)
    assert any(op[0] == "rowblk" for op in plan.launch)
    y, t, r = O.hqr(a, 1e-10)
    assert np.linalg.norm(to_dense(f.r) - to_dense(r)) <= 1e-8 * np.linalg.norm(to_dense(r))
    e_orth, e_acc = O.dense_metrics(to_dense(a), f.y, f.t, f.r)
    assert e_orth <= 1e-13 and e_acc <= 1e-11


def test_svd_cluster_sizes_from_runtime_sizes():
    """Cluster choice of a Jacobi launch (plan.svd_cluster_runtime): tiny
    cores stay on one CTA, a core goes to the smallest cluster whose shared
    memory holds it, widened while the launch fits one wave of 148 SMs."""
    from paper_1809_10585_b200.plan import _svd_fits, svd_cluster_runtime
    assert svd_cluster_runtime(1, 24, 24) == 1            # few pairs: one SM
    assert svd_cluster_runtime(1, 200, 200) == 8           # one core: widest cluster
    assert svd_cluster_runtime(32, 200, 200) == 4          # 32 x 4 CTAs = one wave
    assert svd_cluster_runtime(64, 120, 120) == 2
    assert svd_cluster_runtime(64, 700, 300) == 1          # beyond the cluster path (m > 640)
    assert svd_cluster_runtime(1, 440, 440) == 16          # too wide for 8 CTAs: a 16-CTA cluster
    for G in (2, 4, 8):
        n = 8
        while _svd_fits(G, n + 8, n + 8):
            n += 8
        assert svd_cluster_runtime(1000, n, n) == G        # many problems: the smallest fitting cluster


def test_retune_clusters_uses_the_rank_table():
    """After a run the Jacobi launches are re-sized from the core sizes in the
    rank table (not the capacities), and only the svd and pivoted-QR ops change."""
    from paper_1809_10585_b200.plan import retune_clusters
    a = gen.gen_random_hodlr(1024, 128, 16, 8.0, seed=0)
    (f,), io, plan = emulate([a], 1e-10)
    rk = plan.rank.numpy().copy()
    before = [dict(ex) for _, _, ex in io.builder.ops]
    retune_clusters(io.builder, rk)
    for (kind, probs, ex), old in zip(io.builder.ops, before):
        if kind == "qrcp":
            assert ex["cluster"] in (1, 2, 4, 8) and ex["threads"] in (256, 512)
            assert {k: v for k, v in ex.items() if k not in ("cluster", "smem", "threads")} == \
                {k: v for k, v in old.items() if k not in ("cluster", "smem", "threads")}
        elif kind != "svd":
            assert ex == old
        else:
            assert ex["cluster"] in (0, 1, 2, 4, 8)
