"""Jacobi SVD launch time for a batch of nprob same-size cores at each cluster size.
usage: python tools/svd_batch.py n1,n2,.. nprob1,nprob2,.."""
import sys
sys.path.insert(0, ".")
import numpy as np, torch
from paper_1809_10585_b200 import _abi
lib = _abi.load()
ns = [int(x) for x in sys.argv[1].split(",")]
nps = [int(x) for x in sys.argv[2].split(",")]
for n in ns:
    rng = np.random.default_rng(n)
    u = np.linalg.qr(rng.standard_normal((n, n)))[0]; v = np.linalg.qr(rng.standard_normal((n, n)))[0]
    C = (u * np.logspace(0, -16, n)) @ v.T
    M = np.linalg.qr(C.T)[1]
    for P in nps:
        dC = [torch.tensor(M.T.copy(), device="cuda") for _ in range(P)]
        dU = torch.zeros(P, n * n, dtype=torch.float64, device="cuda")
        dW = torch.zeros(P, n * n, dtype=torch.float64, device="cuda")
        rank = torch.zeros(4 * P + 4, dtype=torch.int32, device="cuda")
        scal = torch.zeros(2, dtype=torch.float64, device="cuda")
        p = np.zeros(P, _abi.SVD_PROB)
        for i in range(P):
            p[i] = (dC[i].data_ptr(), dU[i].data_ptr(), dW[i].data_ptr(), n, n, n, -1, n, -1, n, 4 * i, -1, -1, 1e-10, 1, 0)
        dp = torch.tensor(np.frombuffer(p.tobytes(), np.uint8), device="cuda")
        res = []
        for CL in (1, 2, 4, 8, 16):
            best = 1e9
            for rep in range(3):
                for i in range(P):
                    dC[i].copy_(torch.tensor(M.T.copy(), device="cuda"))
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(); rc = lib.hq_svd(None, dp.data_ptr(), P, rank.data_ptr(), scal.data_ptr(), CL, n, 0); e1.record()
                torch.cuda.synchronize()
                best = min(best, e0.elapsed_time(e1))
            res.append(f"CL{CL} {best:7.3f} ms (rc {rc}, rank {int(rank[0])})")
        print(f"n={n} nprob={P}: " + " | ".join(res), flush=True)
