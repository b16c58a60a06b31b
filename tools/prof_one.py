"""Run one factorization of a config (for ncu launch lists)."""
import sys
sys.path.insert(0, ".")
import torch
from paper_1809_10585_b200 import gen
from paper_1809_10585_b200.hqr import HQREngine
ci = int(sys.argv[1]); n = int(sys.argv[2]) if len(sys.argv) > 2 else None
c = gen.CONFIGS[ci]
a = gen.gen_config(ci, seed=0, n=n)
eng = HQREngine(a.tree(), 1, c["tol"], use_graph=False)
eng.pack([a]); eng.upload(); eng.execute(); torch.cuda.synchronize()
print("ok launches", eng.plan.n_launch)
