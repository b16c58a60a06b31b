"""Run-time dims of every Jacobi launch at one size (GPU): m, n, output rank, cluster."""
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
rows = []
for kind, probs, extra in eng.builder.ops:
    if kind == "svd":
        for p in probs:
            m, nn = _dv(p[5], rk), _dv(p[6], rk)
            rows.append((extra["cluster"], p[5].cap, p[6].cap, m, nn, int(rk[p[8]])))
print("cluster capM capN m n_eff rank -> count")
cnt = collections.Counter((r[0], r[1], r[2], r[3] // 16 * 16, min(r[3], r[4]) // 16 * 16, r[5] // 16 * 16) for r in rows)
for k, v in sorted(cnt.items()):
    if k[0] > 1 or k[3] >= 128:
        print(k, v)
