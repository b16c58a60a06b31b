import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
from paper_1809_10585_b200 import _abi
lib = _abi.load()
def put(arr): return torch.tensor(np.frombuffer(arr.tobytes(), np.uint8), device="cuda")
cases = [(int(x), "decay") for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [(96, "decay"), (128, "decay"), (144, "decay"), (200, "decay"), (128, "flat"), (128, "lowrank")]
for n, kind in cases:
    rng = np.random.default_rng(n)
    u = np.linalg.qr(rng.standard_normal((n, n)))[0]; v = np.linalg.qr(rng.standard_normal((n, n)))[0]
    s = {"decay": np.logspace(0, -16, n), "flat": np.ones(n), "lowrank": np.r_[np.logspace(0, -3, n // 2), np.zeros(n - n // 2)]}[kind]
    C = (u * s) @ v.T
    for xf, CL in ((1, 1), (1, 2), (1, 4), (1, 8)):
        MM = n
        ld, bs = (n + 1) // 2 * 2, -(-n // (2 * CL))
        if CL > 1 and 4 * bs * ld > 26880: continue
        M = np.linalg.qr(C.T)[1] if xf else C
        for rep in range(2):
            dC = torch.tensor(M.T.copy(), device="cuda")
            dU = torch.zeros(n * n, dtype=torch.float64, device="cuda")
            dW = torch.zeros(n * n, dtype=torch.float64, device="cuda")
            rank = torch.zeros(10, dtype=torch.int32, device="cuda")
            scal = torch.zeros(2, dtype=torch.float64, device="cuda")
            p = np.zeros(1, _abi.SVD_PROB); p[0] = (dC.data_ptr(), dU.data_ptr(), dW.data_ptr(), n, n, n, -1, n, -1, n, 0, 1, -1, 1e-10, xf, 0)
            dp = put(p); torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); lib.hq_svd(None, dp.data_ptr(), 1, rank.data_ptr(), scal.data_ptr(), CL, MM, 0); e1.record(); torch.cuda.synchronize()
        k = int(rank[0]); U = dU.cpu().numpy().reshape(n, n).T[:, :k]
        err = np.linalg.norm(C - U @ (U.T @ C), 2)
        print(n, kind, "xform", xf, "cluster", CL, "ms %.3f" % e0.elapsed_time(e1), "rank", k, "sweeps(dbg)", int(rank[2]), "cyc/16 norm,intra,inter,xchg", rank[3:7].tolist(), "round work/bar", rank[7:9].tolist(), "proj err %.2e" % err, "orth %.1e" % np.abs(U.T @ U - np.eye(k)).max())
