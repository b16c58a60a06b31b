"""Device time of one graph replay for a config at a given batch size."""
import argparse, sys, time
sys.path.insert(0, ".")
import numpy as np, torch
from paper_1809_10585_b200 import gen
from paper_1809_10585_b200.hqr import HQREngine
from paper_1809_10585_b200.hodlr import stats
ap = argparse.ArgumentParser()
ap.add_argument("cfg", type=int); ap.add_argument("--n", type=int); ap.add_argument("--batch", type=int, default=1)
args = ap.parse_args()
c = gen.CONFIGS[args.cfg]
B = args.batch
t0 = time.time()
mats = [gen.gen_config(args.cfg, seed=s, n=args.n) for s in range(B)]
tg = time.time() - t0
t0 = time.time()
eng = HQREngine(mats[0].tree(), B, c["tol"])
tb = time.time() - t0
print(f"cfg{args.cfg} n={mats[0].n} B={B} gen {tg:.1f}s plan {tb:.1f}s launches {eng.plan.n_launch} arena {eng.plan.total_doubles*8/1e9:.2f} GB", flush=True)
eng.pack(mats); eng.upload(); eng.snapshot_device_input()
t0 = time.time(); eng.execute(); torch.cuda.synchronize(); print(f"  capture+first run {time.time()-t0:.2f}s", flush=True)
s = eng.stream
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for rep in range(3):
    eng.restore_device_input()
    ev0.record(s); eng.execute(); ev1.record(s); ev1.synchronize()
    ms = ev0.elapsed_time(ev1)
    print(f"  device time {ms:.2f} ms -> {B / ms * 1e3:.2f} factorizations/s", flush=True)
eng.download()
f = eng.factors(0)
print("  ranks Y T R", stats(f.y)["max_offdiag_rank"], stats(f.t)["max_offdiag_rank"], stats(f.r)["max_offdiag_rank"], flush=True)
