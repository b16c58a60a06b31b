import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
from paper_1809_10585_b200 import gen
from paper_1809_10585_b200.hqr import HQREngine
from paper_1809_10585_b200.hodlr import stats
cfgs = [int(c) for c in sys.argv[1:]] or [0, 2]
for ci in cfgs:
    c = gen.CONFIGS[ci]
    B = c.get("batch", 1) if len(sys.argv) > 1 else 1
    t0 = time.time()
    mats = [gen.gen_config(ci, seed=s) for s in range(B)]
    tg = time.time() - t0
    t0 = time.time()
    eng = HQREngine(mats[0].tree(), B, c["tol"])
    tb = time.time() - t0
    print(f"cfg{ci} {c['name']} B={B} gen {tg:.1f}s plan {tb:.1f}s launches {eng.plan.n_launch} arena {eng.plan.total_doubles*8/1e9:.2f} GB", flush=True)
    eng.pack(mats); eng.upload()
    t0 = time.time(); eng.execute(); torch.cuda.synchronize(); print(f"  capture+first run {time.time()-t0:.2f}s", flush=True)
    s = eng.stream
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for rep in range(3):
        eng.upload()
        ev0.record(s); eng.execute(); ev1.record(s); ev1.synchronize()
        print(f"  device time {ev0.elapsed_time(ev1):.2f} ms", flush=True)
    eng.download()
    f = eng.factors(0)
    print("  norm est", eng.norm_estimate(0), "ranks Y T R", stats(f.y)["max_offdiag_rank"], stats(f.t)["max_offdiag_rank"], stats(f.r)["max_offdiag_rank"], flush=True)
