#!/usr/bin/env python
"""Benchmark: HODLR QR factorizations/s (FP64) on the B200.

Workload (BASELINE.json metric "at n=16384"): config 2, the ill-conditioned
HODLR matrix, n = 16384, leaf 256, off-diagonal rank 16, A = D B with
D = diag(logspace(0,-14,n)) permuted, tol 1e-10 relative.  One step = one
batch of B independent such matrices (seeds B*rank .. B*rank+B-1; B = 64, or fewer
if they do not fit 85 % of the free HBM) factorized
by one graph replay: power iteration for ||A||_2, the unrolled Algorithm 2,
compaction of Y, T, R.  `latency_ms_single_matrix` reports one matrix alone.

  value  factorizations/s with the input resident in HBM (graph replay of the
         whole factorization; CUDA events on the launching stream, max over
         ranks); the working set (~GBs of factor storage) exceeds the 126 MB L2.
  e2e    the same metric through the public API with host buffers: pack,
         H2D of the compact input stream, replay, D2H of the compact factors,
         and assembly of the HodlrMatrix factors -- all inside the timed region.
Under torchrun each rank factors its own matrix (seed = rank): independent
HODLR matrices shard with no collective (weak scaling).

--impl reference times the CPU oracle port (oracle/hqr_oracle.py, a numpy
restatement of the reference hodlrqr.hqr pinned to its golden vectors) on the
host cores, on the same configuration.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "hodlr_qr_factorizations_per_s"
UNIT = "factorizations/s"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", type=int, default=2)
    p.add_argument("--n", type=int, default=None, help="override n (smoke runs)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--kcap", type=int, default=None,
                   help="rank capacity of the plan (overflow raises RankCapacityError, never truncates)")
    p.add_argument("--no-instrument", action="store_true")
    p.add_argument("--batch", type=int, default=None,
                   help="matrices per step per GPU (config 2 default: 64 or what fits; config 4 is the fixed 64-batch)")
    return p.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def config_dict(cfg, n, extra=None):
    from paper_1809_10585_b200.gen import CONFIGS
    c = dict(CONFIGS[cfg])
    d = {"workload": f"config{cfg}:{c['name']}", "n": n if n else c["n"], "leaf": c["leaf"],
         "tol": c["tol"], "offdiag_rank": c.get("rank"), "matrices_per_step_per_gpu": 1,
         "l2": "working set > 126 MB L2 (factor storage in HBM); no flush needed"}
    if extra:
        d.update(extra)
    return d


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index, self.samples, self.proc = index, [], None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm = [float(s[0]) for s in self.samples if len(s) >= 6 and s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if len(s) >= 6 and s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples if len(s) >= 6
                          for i in range(4) if "Active" in s[2 + i] and "Not" not in s[2 + i]})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def _oracle_one(job):
    """Worker: generate and factor one workload matrix with the CPU oracle
    (single-threaded BLAS); returns the factorization's seconds."""
    cfg, n, seed = job
    from oracle import hqr_oracle as O
    from paper_1809_10585_b200.gen import CONFIGS, gen_config
    a = gen_config(cfg, seed=seed, n=n)
    t0 = time.perf_counter()
    O.hqr(a, CONFIGS[cfg]["tol"])
    return time.perf_counter() - t0


def host_threads():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_throughput(cfg, n, rounds=1, seed0=0, procs=None):
    """The CPU oracle on all host threads: `procs` single-threaded worker
    processes each factor their own matrix (independent matrices, like the
    GPU batch), `rounds` times.  Returns (factorizations/s, procs, matrices)."""
    import multiprocessing as mp
    procs = procs or host_threads()
    env = {k: os.environ.get(k) for k in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS")}
    for k in env:
        os.environ[k] = "1"
    try:
        ctx = mp.get_context("spawn")
        with ctx.Pool(procs) as pool:
            pool.map(_oracle_one, [(cfg, min(n, 1024), seed0 + 1000 + i) for i in range(procs)])  # warm-up: imports
            t0 = time.perf_counter()
            for r in range(rounds):
                pool.map(_oracle_one, [(cfg, n, seed0 + r * procs + i) for i in range(procs)])
            wall = time.perf_counter() - t0
    finally:
        for k, v in env.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    return rounds * procs / wall, procs, rounds * procs


def run_reference(args):
    """--impl reference: the reference's algorithm on the CPU (the oracle
    port, oracle/hqr_oracle.py -- the reference package itself is Python and
    does not travel to the GPU box) on all host threads, same metric."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    from paper_1809_10585_b200.gen import CONFIGS
    n = args.n or CONFIGS[args.config]["n"]
    steps = max(1, min(args.steps, 2))
    v, procs, cnt = cpu_throughput(args.config, n, rounds=steps)
    line = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": steps,
            "warmup": 1, "ms_per_step": 1e3 * procs / v, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded generator of BASELINE config)",
            "config": config_dict(args.config, n, {"matrices_per_step": procs}), "impl": "reference",
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": procs, "kind": "port",
                             "sample": f"{cnt} full factorizations of workload matrices, {procs} single-threaded "
                                       "worker processes at once (oracle/hqr_oracle.py, numpy + OpenBLAS)"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "note": f"one step = one matrix per host thread; steps capped at {steps}"}
    print(json.dumps(line), flush=True)


def instrument(eng, torch):
    """One non-graph pass with CUDA events around every launch: device time
    per kernel class (plan.kind_key) for the rooflines."""
    from paper_1809_10585_b200.plan import kind_key
    plan = eng.plan
    lib = __import__("paper_1809_10585_b200._abi", fromlist=["load"]).load()
    s = eng.stream
    per = {}
    eng.upload()
    eng.stage_to_live()
    s.synchronize()
    evs = []
    orig = plan.launch
    bld = eng.builder
    converged = False
    skipped = set()     # gated launches that were no-ops (power iteration converged)
    with torch.cuda.stream(s):
        for i, rec in enumerate(orig):
            if converged and rec[4].get("skip") is not None:
                skipped.add(i)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            plan.launch = [rec]
            plan.run(s.cuda_stream)
            e1.record(s)
            evs.append((i, kind_key(rec[0], rec[4]), e0, e1))
            if rec[0] == "power" and not converged:
                s.synchronize()
                converged = bool(plan.rank[bld.all_done].item())
    plan.launch = orig
    s.synchronize()
    for i, kind, e0, e1 in evs:
        if i in skipped:
            continue
        d = per.setdefault(kind, [0.0, 0])
        d[0] += e0.elapsed_time(e1)
        d[1] += 1
    del lib
    return per, skipped


BATCH_CAP = int(os.environ.get("HQ_BENCH_BATCH_CAP", "74"))   # 74 two-CTA clusters fill the 148 SMs


def kcap_profile(cfg, tree, top=192):
    """Rank capacity per tree level for a rank-k input (root = 0): 2 k (l + 1),
    at most `top` -- the factors' ranks grow with the depth (measured over the
    bench seeds, tools/level_ranks.py: at most 32/48/64/96/141/159 on levels
    0..5 for k = 16), so the large top-level blocks are stored at their small
    ranks and more matrices fit the HBM.  An overflow raises
    RankCapacityError and the run is redone at a uniform 512."""
    k = cfg.get("rank")
    if not k:
        return top
    return tuple(min(top, 2 * k * (l + 1)) for l in range(max(tree.level, 1)))


def auto_batch(torch, ci, n, tol, local, cap=None, kcap=192, stream_out=True):
    """Matrices per step: as many as fit 85 % of the free HBM (the arena of a
    one-matrix plan scales linearly with the batch), at most `cap`."""
    from paper_1809_10585_b200.gen import gen_config
    from paper_1809_10585_b200.plan import LANE_STRIDE, R_OUT, R_WS, Builder
    bld = Builder(gen_config(ci, seed=0, n=n).tree(), 1, tol, False, kcap).build()
    # the output region aliases scratch unless the engine streams its output;
    # the K-split workspaces (R_WS lanes) are sized for a 1-matrix launch's
    # split factors -- a full batch splits little -- so they are counted once
    ws = sum(b.peak for r, b in bld.bumps.items() if r % LANE_STRIDE == R_WS)
    per_matrix = 8 * (sum(b.peak for r, b in bld.bumps.items() if stream_out or r != R_OUT) - ws)
    free, _ = torch.cuda.mem_get_info(local)
    return max(1, min(cap or BATCH_CAP, int((0.85 * free - 8 * ws) / per_matrix)))


def build_engine(torch, config, n, batch=None, kcap=None, local=0, ws=1, rank=0):
    """The timed engine, exactly as the bench runs it (the GPU parity test
    tests/test_gpu_bench_workload.py builds it through this function):
    config 2 -> seeds rank*B .. rank*B+B-1 with B = what fits 85 % of the free
    HBM (<= 64), rank capacity 192, streaming output; config 4 -> the fixed
    64-matrix batch sharded over the ranks.  The first run (capture + replay
    + download) has happened on return, so the Jacobi clusters are re-tuned
    and the next execute() captures the graph that gets timed.  Returns
    (engine, matrices, kcap, scaling)."""
    from paper_1809_10585_b200.gen import CONFIGS, gen_config
    from paper_1809_10585_b200.hqr import HQREngine, RankCapacityError
    from paper_1809_10585_b200.shard import shard_seeds
    cfg = CONFIGS[config]
    total_batch = cfg.get("batch", 1)
    if total_batch > 1:
        # config 4: a fixed batch of independent matrices sharded over the ranks
        seeds = shard_seeds(total_batch, ws, rank)
        scaling = "strong"
    else:
        tree0 = gen_config(config, seed=0, n=n).tree()
        kc0 = kcap or kcap_profile(cfg, tree0)
        per = batch or auto_batch(torch, config, n, cfg["tol"], local, kcap=kc0)
        seeds = list(range(rank * per, (rank + 1) * per))
        scaling = "weak"
    mats = [gen_config(config, seed=s, n=n) for s in seeds]
    a = mats[0]
    # rank capacity 192 (largest rank on this workload over 64 seeds: 159); an
    # overflow raises RankCapacityError -- it never truncates -- and the run
    # is redone at capacity 512 with the batch that fits
    kc = kcap or (kc0 if total_batch == 1 else 512)
    while True:
        eng = HQREngine(a.tree(), len(mats), cfg["tol"], kcap=kc, device=f"cuda:{local}", stream_out=True)
        eng.pack(mats)
        eng.upload()
        eng.snapshot_device_input()
        eng.execute()  # capture + first run
        try:
            eng.download()
            break
        except RankCapacityError:
            if kc == 512:
                raise
            del eng
            torch.cuda.empty_cache()
            kc = 512
            if total_batch == 1 and not batch:
                mats = mats[:auto_batch(torch, config, n, cfg["tol"], local, kcap=kc)]
                a = mats[0]
    return eng, mats, kc, scaling


def r_sketch_error(f, config):
    """Relative Frobenius error of matrix 0's R sketch (R @ G, G the fixed
    Gaussian of tests/golden/make_golden_full.py) against the reference's
    golden sketch, computed on the GPU (QROperator), or None without the
    golden file."""
    path = os.path.join(ROOT, "tests", "golden", f"golden_full_cfg{config}.npz")
    if not os.path.exists(path):
        return None
    from paper_1809_10585_b200.operators import QROperator
    g = np.load(path)["RG"]
    G = np.random.default_rng(0x5C37).standard_normal((g.shape[0], 8))
    rg = QROperator(f).apply_r(G)
    return float(np.linalg.norm(rg - g) / np.linalg.norm(g))


def run_partitioned(args, torch, ws, rank, local):
    """Config 3 under torchrun: ONE n = 65536 matrix partitioned over the
    ranks (distributed.py: the chain on rank 0, the off-spine subtree updates
    and T phase on the others, allocation instances exchanged with NCCL
    send / recv).  Strong scaling: the whole job is one factorization."""
    import torch.distributed as dist
    from paper_1809_10585_b200.distributed import DistEngine
    from paper_1809_10585_b200.gen import CONFIGS, gen_config
    from paper_1809_10585_b200.shard import max_over_ranks
    cfg = CONFIGS[args.config]
    n = args.n or cfg["n"]
    a = gen_config(args.config, seed=0, n=n)
    eng = DistEngine(a.tree(), cfg["tol"], kcap=args.kcap or 512, device=f"cuda:{local}")
    for _ in range(max(1, min(args.warmup, 1))):
        eng.factorize(a)
    clocks = ClockSampler(local)
    clocks.start()
    dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    steps = max(1, min(args.steps, 3))
    for _ in range(steps):
        f = eng.factorize(a)
    torch.cuda.synchronize()
    dist.barrier()
    clk = clocks.stop()
    ms = max_over_ranks((time.perf_counter() - t0) * 1e3, device=f"cuda:{local}") / steps
    sched = eng.sched
    line = {"metric": METRIC, "value": 1e3 / ms, "unit": UNIT, "n_gpus": ws, "steps": steps, "warmup": 1,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded generator of BASELINE config 3, seed 0)",
            "config": config_dict(args.config, n, {"parallelism": f"one matrix partitioned over {ws} ranks "
                                                                  "(DAG lanes, NCCL send/recv)"}),
            "e2e": {"value": 1e3 / ms, "unit": UNIT, "h2d_bytes_per_step": int(8 * eng.io.n_in),
                    "d2h_bytes_per_step": int(8 * eng.plan.totals[1].item()) if rank == 0 else 0,
                    "includes": "pack + H2D on every rank + partitioned factorization + D2H + assembly (rank 0)"},
            "gpu_launches": sum(1 for r in sched.rank_of_op if r == rank),
            "ops_by_rank": sched.ops_by_rank(), "exchanged_bytes": sched.bytes_total(),
            "exchanged_bytes_by_level": {str(k): v for k, v in sched.bytes_by_level().items()},
            "timing": "wall clock per factorization, max over ranks (host-driven launches and NCCL calls)",
            "clocks": clk}
    if rank == 0:
        line["r_sketch_rel_err_matrix0"] = r_sketch_error(f, args.config) if args.n is None else None
        print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    ws, rank, local = dist_env()
    if ws > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        if args.config == 3:
            run_partitioned(args, torch, ws, rank, local)
            dist.destroy_process_group()
            return
    from paper_1809_10585_b200.gen import CONFIGS
    from paper_1809_10585_b200.hqr import HQREngine
    from paper_1809_10585_b200.plan import plan_accounting
    cfg = CONFIGS[args.config]
    n = args.n or cfg["n"]
    total_batch = cfg.get("batch", 1)
    from paper_1809_10585_b200.shard import max_over_ranks
    eng, mats, kcap, scaling = build_engine(torch, args.config, n, args.batch, args.kcap, local, ws, rank)
    a = mats[0]
    s = eng.stream

    def barrier():
        if ws > 1:
            torch.distributed.barrier()

    for _ in range(max(args.warmup, 3)):
        eng.restore_device_input()
        eng.execute()
    s.synchronize()
    # ---- device-timed region: input resident in HBM
    clocks = ClockSampler(local)
    clocks.start()
    barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(s)
    for _ in range(args.steps):
        eng.restore_device_input()
        eng.execute()
    ev1.record(s)
    ev1.synchronize()
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    ms = max_over_ranks(ev0.elapsed_time(ev1), device=f"cuda:{local}")
    ms_step = ms / args.steps
    per_step = total_batch if total_batch > 1 else ws * len(mats)
    value = per_step * args.steps / (ms / 1e3)
    # ---- end-to-end through the public API with host buffers
    e2e_steps = max(4, min(2 * args.steps, 10))   # batches in the stream (fill and drain amortised)
    for f in eng.factorize_stream([mats] * 3):  # untimed warm-up: worker pools, pinned result blocks
        pass
    barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    # e2e_steps batches through the streaming API: every batch is packed from
    # the host matrices, uploaded, factored and its factors copied back and
    # assembled; batch i's copies overlap batch i+1's device work
    for f in eng.factorize_stream([mats] * e2e_steps):
        pass
    e2e_s = max_over_ranks((time.perf_counter() - t0) / e2e_steps, device=f"cuda:{local}")
    e2e = {"value": per_step / e2e_s, "unit": UNIT, "h2d_bytes_per_step": int(eng.h2d_bytes()),
           "d2h_bytes_per_step": int(eng.d2h_bytes()),
           "includes": "pack + H2D + graph replay + D2H + HodlrMatrix assembly, streamed: "
                       f"{e2e_steps} batches through HQREngine.factorize_stream"}
    rk = eng.h_rk_out.numpy()
    acc = plan_accounting(eng.builder, rk)
    flops = sum(v["flops"] for v in acc.values())
    from paper_1809_10585_b200.hodlr import stats
    ranks = {k: stats(getattr(f[0], k))["max_offdiag_rank"] for k in ("y", "t", "r")}
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded generator of BASELINE config; seeds " +
                    ("0..%d sharded over ranks)" % (total_batch - 1) if total_batch > 1 else "= rank)"),
            "config": config_dict(args.config, n, {"parallelism": f"independent matrices x{ws}",
                                                    "matrices_per_step_per_gpu": len(mats),
                                                    "kcap": kcap}),
            "e2e": e2e, "gpu_launches": eng.plan.n_launch * args.steps,
            "fp64_gflops_effective": flops / (ms_step / 1e3) / 1e9,
            "algorithmic_gflop_per_step": flops / 1e9,
            "norm_estimate": eng.norm_estimate(0), "max_ranks": ranks, "clocks": clk}
    if rank == 0 and args.n is None:
        # parity of what was timed: matrix 0 of the last e2e batch against the
        # reference's golden R sketch (tests/golden/make_golden_full.py)
        line["r_sketch_rel_err_matrix0"] = r_sketch_error(f[0], args.config)
    if rank == 0 and len(mats) > 1:
        # single-matrix latency (batch 1 plan, graph replay, input resident)
        e1 = HQREngine(a.tree(), 1, cfg["tol"], kcap=kcap, device=f"cuda:{local}")
        e1.pack([a])
        e1.upload()
        e1.snapshot_device_input()
        for _ in range(3):
            e1.restore_device_input()
            e1.execute()
        e1.stream.synchronize()
        l0, l1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        l0.record(e1.stream)
        for _ in range(3):
            e1.restore_device_input()
            e1.execute()
        l1.record(e1.stream)
        l1.synchronize()
        line["latency_ms_single_matrix"] = l0.elapsed_time(l1) / 3
        del e1
        torch.cuda.empty_cache()
        # the reference-facing single call, host matrix in, HodlrMatrix
        # factors out (pack, H2D, replay, D2H, assembly): hqr(a, eps)
        from paper_1809_10585_b200 import clear_engines, hqr
        for _ in range(2):   # plan build + capture, cluster re-tune + re-capture
            hqr(a, cfg["tol"], kcap=kcap)
        ts = []
        for _ in range(3):
            t0 = time.perf_counter()
            fa = hqr(a, cfg["tol"], kcap=kcap)
            ts.append((time.perf_counter() - t0) * 1e3)
            del fa
        line["latency_ms_single_matrix_api"] = min(ts)
        clear_engines()
    if not args.no_instrument and rank == 0:
        per, skipped = instrument(eng, torch)
        acc = plan_accounting(eng.builder, rk, skipped, rk_in=eng.rk)
        tot = sum(v[0] for v in per.values())
        kinds = {k: {"ms": v[0], "launches": v[1], "share": v[0] / tot,
                     "gflop": acc.get(k, {}).get("flops", 0.0) / 1e9,
                     "tflops": acc.get(k, {}).get("flops", 0.0) / max(v[0], 1e-9) / 1e9,
                     "gbytes": acc.get(k, {}).get("bytes", 0.0) / 1e9} for k, v in per.items()}
        top = max((k for k in per if acc.get(k, {}).get("flops", 0) > 0), key=lambda k: per[k][0])
        peak_fp64 = 37.16e12  # self-measured DMMA m8n8k4 FP64 (profiles/r01_fp64_peak.txt)
        ach = acc[top]["flops"] / (per[top][0] / 1e3)
        traffic, traffic_all = None, {}
        try:   # DRAM bytes per launch of this kernel from the committed ncu --set full capture
            with open(os.path.join(ROOT, "profiles", "r02_traffic.json")) as fh:
                traffic_all = json.load(fh)
            traffic = traffic_all.get(top, {}).get("dram_bytes_per_launch")
        except (OSError, ValueError):
            pass
        line["roofline"] = {"kernel": top, "bound": "tensor", "achieved": ach / 1e12, "peak": peak_fp64 / 1e12,
                            "unit": "TFLOP/s", "frac": ach / peak_fp64, "traffic": traffic,
                            "traffic_unit": "bytes/launch (dram__bytes_read+write, profiles/r02_traffic.json)",
                            "peak_source": "self-measured FP64 DMMA peak (profiles/r01_fp64_peak.txt); "
                                           "MEASURED_PEAKS.json has no FP64 entry",
                            "flops_per_launch": acc[top]["flops"] / max(acc[top]["launches"], 1),
                            "avg_launch_ms": per[top][0] / per[top][1], "share_of_step": kinds[top]["share"]}
        line["kernel_time_by_kind"] = kinds
        # every kernel class against its own roof: HBM bytes per launch for the
        # streaming / data-movement kernels, FP64 DMMA for the rest
        hbm = 6538.0
        try:
            with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
                hbm = float(json.load(fh).get("hbm_gbs", hbm))
        except (OSError, ValueError):
            pass
        rbk = {}
        for k, v in per.items():
            a = acc.get(k, {})
            sec = v[0] / 1e3
            if k in ("gemv", "concat", "pack_copy", "leaf_gather", "leaf_scatter"):
                gbs = a.get("bytes", 0.0) / max(sec, 1e-12) / 1e9
                rbk[k] = {"bound": "hbm", "achieved": gbs, "peak": hbm, "unit": "GB/s", "frac": gbs / hbm,
                          "bytes_per_launch": a.get("bytes", 0.0) / max(v[1], 1)}
            elif a.get("flops", 0.0) > 0:
                tf = a["flops"] / max(sec, 1e-12) / 1e12
                rbk[k] = {"bound": "tensor", "achieved": tf, "peak": peak_fp64 / 1e12, "unit": "TFLOP/s",
                          "frac": tf / (peak_fp64 / 1e12), "flops_per_launch": a["flops"] / max(v[1], 1)}
        for k in rbk:   # measured DRAM bytes of one captured launch of the class (ncu), where committed
            rbk[k]["traffic"] = traffic_all.get(k, {}).get("dram_bytes_per_launch")
        line["roofline_by_kind"] = rbk
    if rank == 0 and not args.no_cpu_baseline and ws == 1:
        v_cpu, procs, cnt = cpu_throughput(args.config, n, rounds=1)
        line["cpu_baseline"] = {"value": v_cpu, "unit": UNIT, "cores": procs, "kind": "port",
                                "sample": f"{cnt} full factorizations of workload matrices, one per host thread "
                                          "(single-threaded worker processes, oracle/hqr_oracle.py)"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
