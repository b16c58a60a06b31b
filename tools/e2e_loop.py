import sys, time
sys.path.insert(0, ".")
import torch
from paper_1809_10585_b200 import gen
from paper_1809_10585_b200.hqr import HQREngine
B = int(sys.argv[1])
mats = [gen.gen_config(2, seed=s) for s in range(B)]
eng = HQREngine(mats[0].tree(), B, 1e-10)
f = eng.factorize(mats)
for i in range(5):
    t = time.perf_counter(); f = eng.factorize(mats); print(i, round((time.perf_counter() - t) * 1e3, 1), "ms", flush=True)
