import sys, collections
sys.path.insert(0, ".")
import numpy as np, torch
from paper_1809_10585_b200 import gen
from paper_1809_10585_b200.hqr import HQREngine
from paper_1809_10585_b200.plan import _dv
ci = int(sys.argv[1]); n = int(sys.argv[2]) if len(sys.argv) > 2 else None
c = gen.CONFIGS[ci]
a = gen.gen_config(ci, seed=0, n=n)
eng = HQREngine(a.tree(), 1, c["tol"])
f = eng.factorize([a])
rk = eng.h_rk_out.numpy()
sizes = collections.Counter(); per_launch = []
for kind, probs, extra in eng.builder.ops:
    if kind == "svd":
        dims = [(_dv(p[5], rk), _dv(p[6], rk)) for p in probs]
        per_launch.append((len(probs), max(m * n for m, n in dims), max(max(d) for d in dims)))
        for m, nn in dims:
            sizes[(min(m, nn) // 32 * 32)] += 1
print("svd problems by min-dim bucket:", sorted(sizes.items()))
big = sum(v for k, v in sizes.items() if k >= 160)
print("problems with min dim >= 160:", big, "of", sum(sizes.values()))
print("launches (nprob, max m*n, max dim):", per_launch[:80])
