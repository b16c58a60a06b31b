import sys
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np
from emu import emulate
from oracle import hqr_oracle as O
from paper_1809_10585_b200 import gen, hqr
from paper_1809_10585_b200.hodlr import to_dense
cases = {"ragged": (lambda: gen.gen_random_hodlr(200, 24, 3, 8.0, seed=2), 1e-12),
         "ragged2": (lambda: gen.gen_random_hodlr(100, 24, 3, 8.0, seed=2), 1e-12),
         "leaf25": (lambda: gen.gen_random_hodlr(25, 64, 3, 8.0, seed=2), 1e-12),
         "leaf40": (lambda: gen.gen_random_hodlr(40, 64, 3, 8.0, seed=2), 1e-12),
         "n50": (lambda: gen.gen_random_hodlr(50, 24, 3, 8.0, seed=2), 1e-12)}
for name, (b, eps) in cases.items():
    a = b()
    f = hqr(a, eps)
    (fe,), _, _ = emulate([a], eps)
    for k in ("y", "t", "r"):
        g, e = to_dense(getattr(f, k)), to_dense(getattr(fe, k))
        print(name, k, "max|gpu-emu|", np.abs(g - e).max(), flush=True)
    print(name, "metrics gpu", O.dense_metrics(to_dense(a), f.y, f.t, f.r), "emu", O.dense_metrics(to_dense(a), fe.y, fe.t, fe.r), flush=True)
