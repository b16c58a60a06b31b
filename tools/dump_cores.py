"""Dump the truncation cores of a config-2 factorization from the numpy
emulator (tests/emu.py): list of (C, thr), triu(C) = the core's R factor.
Input of tools/qrcp_ab.py and tools/jacobi_precond_ab.py.
    python tools/dump_cores.py n min_size out.pkl"""
import pickle
import sys
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import numpy as np
import emu
from paper_1809_10585_b200 import _abi
from paper_1809_10585_b200.gen import gen_config
import paper_1809_10585_b200.plan as plan

plan.PIVOT_CORE = False   # the unpivoted plan hands the Jacobi the full R_c
n, lo, out = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
cores = []
orig = emu.Emu.svd


def svd(self, o1, cnt, ex):
    for p in self.arr(o1, _abi.SVD_PROB, cnt):
        m, k = self.dim(p["m"], p["m_ri"]), self.dim(p["n"], p["n_ri"])
        if m > 0 and k > 0 and p["xform"] and min(m, k) >= lo:
            thr = p["eps_scale"] * (self.scal[p["eps_slot"]] if p["eps_slot"] >= 0 else 1.0)
            cores.append((np.array(self.mat(p["c"], p["ldc"], min(k, m), m)).copy(), thr))
    return orig(self, o1, cnt, ex)


emu.Emu.svd = svd
emu.emulate([gen_config(2, seed=0, n=n)], 1e-10, kcap=256)
print(len(cores), "cores", sorted({c[0].shape for c in cores}))
pickle.dump(cores, open(out, "wb"))
