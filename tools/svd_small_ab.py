"""Small-core Jacobi kernel (cluster = 0) against the cluster choice of the
plan on many small graded cores (m x n as after the pivoted QR).
    python tools/svd_small_ab.py [m,n;m,n;...] [problems]"""
import sys
sys.path.insert(0, ".")
import numpy as np, torch
from paper_1809_10585_b200 import _abi
from paper_1809_10585_b200.plan import svd_cluster_runtime
lib = _abi.load()
shapes = [tuple(int(x) for x in s.split(",")) for s in (sys.argv[1] if len(sys.argv) > 1 else "48,32;64,32;80,48;96,48;112,64;128,64").split(";")]
P = int(sys.argv[2]) if len(sys.argv) > 2 else 1482
for m, n in shapes:
    rng = np.random.default_rng(m * n)
    u = np.linalg.qr(rng.standard_normal((m, n)))[0]
    v = np.linalg.qr(rng.standard_normal((n, n)))[0]
    s = np.logspace(0, -10.5, n)
    X = (u * s) @ v.T
    thr = 1e-10
    ld = (m + 1) // 2 * 2
    src = torch.tensor(np.tile(np.asfortranarray(X).ravel(order="F"), P), device="cuda")
    dC = src.clone()
    dU = torch.zeros(P * m * n, dtype=torch.float64, device="cuda")
    dW = torch.zeros(P * ld * n, dtype=torch.float64, device="cuda")
    rank = torch.zeros(P + 2, dtype=torch.int32, device="cuda")
    scal = torch.zeros(2, dtype=torch.float64, device="cuda")
    p = np.zeros(P, _abi.SVD_PROB)
    for i in range(P):
        p[i] = (dC.data_ptr() + 8 * i * m * n, dU.data_ptr() + 8 * i * m * n, dW.data_ptr() + 8 * i * ld * n, m, m,
                m, -1, n, -1, n, 2 + i, 1, -1, thr, 0, 0)
    dp = torch.tensor(np.frombuffer(p.tobytes(), np.uint8), device="cuda")
    out = []
    for name, G, small in (("cl2", 2, 0), ("cl1", 1, 0), ("small", 0, ld * n), ("small-8k", 0, max(ld * n, 8192))):
        ts = []
        for _ in range(3):
            dC.copy_(src); torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            assert lib.hq_svd(None, dp.data_ptr(), P, rank.data_ptr(), scal.data_ptr(), G, m, small) == 0
            e1.record(); torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        k = int(rank[2].item())
        U = dU[:m * k].cpu().numpy().reshape(k, m).T
        out.append("%s %.3f ms (k %d orth %.0e)" % (name, min(ts), k, np.abs(U.T @ U - np.eye(k)).max()))
    print(m, n, "x", P, " | ".join(out), flush=True)
