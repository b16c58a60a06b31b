"""Time one hq_qr launch (leaf-like problem with full T) and apply-Q."""
import sys
sys.path.insert(0, ".")
import numpy as np, torch
from paper_1809_10585_b200 import _abi
lib = _abi.load()
def put(arr): return torch.tensor(np.frombuffer(arr.tobytes(), np.uint8), device="cuda")
for m, k, full, cl in [(352, 256, 1, 1), (352, 256, 1, 8), (352, 256, 0, 8), (256, 200, 0, 1), (256, 200, 0, 8), (2048, 112, 0, 8), (8192, 48, 0, 8)]:
    rng = np.random.default_rng(m + k)
    A = rng.standard_normal((m, k))
    for rep in range(3):
        dW = torch.tensor(A.T.copy(), device="cuda")
        r = min(m, k)
        tau = torch.zeros(r, dtype=torch.float64, device="cuda")
        tp = torch.zeros(((r + 15) // 16) * 256 + 2 * r * 16, dtype=torch.float64, device="cuda")
        tf = torch.zeros(r * r, dtype=torch.float64, device="cuda")
        rank = torch.zeros(4, dtype=torch.int32, device="cuda")
        q = np.zeros(1, _abi.QR_PROB)
        q[0] = (dW.data_ptr(), tau.data_ptr(), tp.data_ptr(), tf.data_ptr() if full else 0, m, r, m, -1, k, -1)
        dq = put(q); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); lib.hq_qr(None, dq.data_ptr(), 1, rank.data_ptr(), cl); e1.record(); torch.cuda.synchronize()
    fl = 2 * m * k * k - 2 * k ** 3 / 3
    print(f"qr {m}x{k} fullT={full} cluster={cl}: {e0.elapsed_time(e1):.3f} ms  ({fl / e0.elapsed_time(e1) / 1e6:.1f} GFLOP/s)")
