"""One Jacobi launch (nprob cores of size n, cluster CL) -- for ncu captures.
usage: python tools/svd_one.py n CL [nprob]"""
import sys
sys.path.insert(0, ".")
import numpy as np, torch
from paper_1809_10585_b200 import _abi
lib = _abi.load()
n, CL = int(sys.argv[1]), int(sys.argv[2])
P = int(sys.argv[3]) if len(sys.argv) > 3 else 1
rng = np.random.default_rng(n)
u = np.linalg.qr(rng.standard_normal((n, n)))[0]; v = np.linalg.qr(rng.standard_normal((n, n)))[0]
M = np.linalg.qr(((u * np.logspace(0, -16, n)) @ v.T).T)[1]
dC = [torch.tensor(M.T.copy(), device="cuda") for _ in range(P)]
dU = torch.zeros(P, n * n, dtype=torch.float64, device="cuda")
dW = torch.zeros(P, n * n, dtype=torch.float64, device="cuda")
rank = torch.zeros(4 * P + 4, dtype=torch.int32, device="cuda")
scal = torch.zeros(2, dtype=torch.float64, device="cuda")
p = np.zeros(P, _abi.SVD_PROB)
for i in range(P):
    p[i] = (dC[i].data_ptr(), dU[i].data_ptr(), dW[i].data_ptr(), n, n, n, -1, n, -1, n, 4 * i, -1, -1, 1e-10, 1, 0)
dp = torch.tensor(np.frombuffer(p.tobytes(), np.uint8), device="cuda")
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
rc = lib.hq_svd(None, dp.data_ptr(), P, rank.data_ptr(), scal.data_ptr(), CL, n, 0)
e1.record(); torch.cuda.synchronize()
print(f"n={n} CL={CL} nprob={P}: {e0.elapsed_time(e1):.3f} ms rc={rc} rank={int(rank[0])}")
