"""A/B of the truncation Jacobi kernels on batches of graded cores (the
LQ-preconditioned form the plan issues, xform=1): scalar kernel with the
plan's run-time cluster choice vs the block Jacobi (hq_svd_block).
    python tools/jacobi_ab.py [sizes] [batch]"""
import sys
sys.path.insert(0, ".")
import numpy as np, torch
from paper_1809_10585_b200 import _abi
from paper_1809_10585_b200.plan import svd_block_cluster, svd_cluster_runtime
lib = _abi.load()
sizes = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [64, 100, 150, 200, 300, 450, 560]
P = int(sys.argv[2]) if len(sys.argv) > 2 else 56


def put(arr):
    return torch.tensor(np.frombuffer(arr.tobytes(), np.uint8), device="cuda")


for n in sizes:
    rng = np.random.default_rng(n)
    u = np.linalg.qr(rng.standard_normal((n, n)))[0]
    v = np.linalg.qr(rng.standard_normal((n, n)))[0]
    s = np.logspace(0, -14, n)
    C = (u * s) @ v.T
    R = np.linalg.qr(C.T)[1]
    thr = 1e-10
    ld = (n + 1) // 2 * 2
    dC = torch.tensor(np.tile(R.T.copy().ravel(), P), device="cuda")
    dU = torch.zeros(P * n * n, dtype=torch.float64, device="cuda")
    dW = torch.zeros(P * ld * n, dtype=torch.float64, device="cuda")
    rank = torch.zeros(2 * P + 2, dtype=torch.int32, device="cuda")
    scal = torch.zeros(2, dtype=torch.float64, device="cuda")
    p = np.zeros(P, _abi.SVD_PROB)
    for i in range(P):
        p[i] = (dC.data_ptr() + 8 * i * n * n, dU.data_ptr() + 8 * i * n * n, dW.data_ptr() + 8 * i * ld * n, n, n,
                n, -1, n, -1, n, 2 + i, 1, -1, thr, 1, 0)
    dp = put(p)
    res = {}
    G = svd_cluster_runtime(P, n, n)
    for name, fn in (("scalar G=%d" % G, lambda: lib.hq_svd(None, dp.data_ptr(), P, rank.data_ptr(), scal.data_ptr(), G, n, 0)),
                     ("block", lambda: lib.hq_svd_block(None, dp.data_ptr(), P, rank.data_ptr(), scal.data_ptr(), svd_block_cluster(P, n)))):
        fn(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            assert fn() == 0
        e1.record(); torch.cuda.synchronize()
        k = int(rank[2].item())
        U = dU[:n * n].cpu().numpy().reshape(n, n).T[:, :k]
        err = np.linalg.norm(C - U @ (U.T @ C), 2)
        res[name] = "%.3f ms (rank %d, orth %.1e, proj %.1e)" % (e0.elapsed_time(e1) / 3, k, np.abs(U.T @ U - np.eye(k)).max(), err)
    print(n, "x", n, "batch", P, res, flush=True)
