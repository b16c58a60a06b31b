"""Sweeps and time of one graded core through the scalar and block Jacobi
kernels of a debug build (HQ_DEBUG_SWEEPS: sweep count in rank[flag + 1]).
Builds tools/libhq_dbg.so first.  python tools/jacobi_dbg.py 150,300"""
import os, subprocess, sys
sys.path.insert(0, ".")
os.environ["HQ_LIB_OUT"] = "tools/libhq_dbg.so"
os.environ["HQ_EXTRA_FLAGS"] = "-DHQ_DEBUG_SWEEPS"
from paper_1809_10585_b200 import build
build.build(force=True)
os.environ["HQ_LIB"] = "tools/libhq_dbg.so"
import importlib
import numpy as np, torch
from paper_1809_10585_b200 import _abi
from paper_1809_10585_b200.plan import svd_block_cluster
_abi.LIB_PATH = "tools/libhq_dbg.so"
lib = _abi.load(build_if_missing=False)
sizes = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [100, 150, 300]


def put(arr):
    return torch.tensor(np.frombuffer(arr.tobytes(), np.uint8), device="cuda")


for n in sizes:
    rng = np.random.default_rng(n)
    u = np.linalg.qr(rng.standard_normal((n, n)))[0]
    v = np.linalg.qr(rng.standard_normal((n, n)))[0]
    C = (u * np.logspace(0, -14, n)) @ v.T
    R = np.linalg.qr(C.T)[1]
    ld = (n + 1) // 2 * 2
    for name in ("scalar", "block"):
        dC = torch.tensor(R.T.copy().ravel(), device="cuda")
        dU = torch.zeros(n * n, dtype=torch.float64, device="cuda")
        dW = torch.zeros(ld * n, dtype=torch.float64, device="cuda")
        rank = torch.zeros(16, dtype=torch.int32, device="cuda")
        scal = torch.zeros(2, dtype=torch.float64, device="cuda")
        p = np.zeros(1, _abi.SVD_PROB)
        p[0] = (dC.data_ptr(), dU.data_ptr(), dW.data_ptr(), n, n, n, -1, n, -1, n, 0, 1, -1, 1e-10, 1, 0)
        dp = put(p)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        if name == "scalar":
            lib.hq_svd(None, dp.data_ptr(), 1, rank.data_ptr(), scal.data_ptr(), 1, n, 0)
        else:
            lib.hq_svd_block(None, dp.data_ptr(), 1, rank.data_ptr(), scal.data_ptr(), svd_block_cluster(1, n))
        e1.record(); torch.cuda.synchronize()
        print(n, name, "ms %.3f" % e0.elapsed_time(e1), "rank", int(rank[0]), "sweeps", int(rank[2]), flush=True)
