"""Largest rank per tree level (root = 0) over the bench batch: rA12 (R and Y
share it), rA21 (Y), rT12 (T)."""
import sys
sys.path.insert(0, ".")
import numpy as np, torch
import bench
B = int(sys.argv[1]) if len(sys.argv) > 1 else None
eng, mats, kc, _ = bench.build_engine(torch, 2, 16384, batch=B)
rk = eng.h_rk_out.numpy()
lay, t = eng.builder.lay, eng.builder.tree
out = {}
for b in range(len(mats)):
    d = lay.m[b]
    for name in ("rA12", "rA21", "rT12"):
        for u, ri in d[name].items():
            key = (u[0], name)
            out[key] = max(out.get(key, 0), int(rk[ri]))
for lv in range(t.L):
    print(lv, {n: out[(lv, n)] for n in ("rA12", "rA21", "rT12")})
