"""e2e of one engine vs the pipelined engines for a batch (config 2)."""
import sys, time
sys.path.insert(0, ".")
import torch
from paper_1809_10585_b200 import gen
from paper_1809_10585_b200.hqr import HQREngine, HQRPipeline
B = int(sys.argv[1]); parts = [int(x) for x in sys.argv[2].split(",")]
mats = [gen.gen_config(2, seed=s) for s in range(B)]
for P in parts:
    eng = HQREngine(mats[0].tree(), B, 1e-10, kcap=256) if P == 1 else HQRPipeline(mats[0].tree(), B, 1e-10, kcap=256, parts=P)
    for _ in range(3):
        f = eng.factorize(mats)
    ts = []
    for i in range(4):
        t = time.perf_counter(); f = eng.factorize(mats); ts.append(time.perf_counter() - t)
    print(f"B={B} parts={P}: e2e {B / min(ts):.2f}/s  (ms {[round(x * 1e3) for x in ts]})", flush=True)
    del f, eng
    torch.cuda.empty_cache()
