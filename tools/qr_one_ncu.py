import sys
sys.path.insert(0, ".")
import numpy as np, torch
from paper_1809_10585_b200 import _abi
lib = _abi.load()
import os
P, m, k = 148, int(os.environ.get("QM", "1024")), int(os.environ.get("QK", "48"))
def put(arr): return torch.tensor(np.frombuffer(arr.tobytes(), np.uint8), device="cuda")
rng = np.random.default_rng(1)
A = rng.standard_normal((m, k)); r = k; npan = (k + 15) // 16
dW = torch.tensor(np.tile(A.T.copy().ravel(), P), device="cuda")
tau = torch.zeros(P * r, dtype=torch.float64, device="cuda")
tp = torch.zeros(P * (npan * 256 + 2 * r * 16), dtype=torch.float64, device="cuda")
rank = torch.zeros(4, dtype=torch.int32, device="cuda")
q = np.zeros(P, _abi.QR_PROB)
for i in range(P):
    q[i] = (dW.data_ptr() + 8 * i * m * k, tau.data_ptr() + 8 * i * r, tp.data_ptr() + 8 * i * (npan * 256 + 2 * r * 16), 0, m, r, m, -1, k, -1)
dq = put(q)
for _ in range(2):
    assert lib.hq_qr(None, dq.data_ptr(), P, rank.data_ptr(), 1) == 0
torch.cuda.synchronize()
