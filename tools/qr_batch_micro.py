"""hq_qr time for a batch of equal problems (one CTA each, or clusters):
cycles per column step at 1.965 GHz.  python tools/qr_batch_micro.py [P]"""
import sys
sys.path.insert(0, ".")
import numpy as np, torch
from paper_1809_10585_b200 import _abi
lib = _abi.load()
P = int(sys.argv[1]) if len(sys.argv) > 1 else 148
def put(arr): return torch.tensor(np.frombuffer(arr.tobytes(), np.uint8), device="cuda")
for m, k, cl in [(256, 48, 1), (512, 48, 1), (1024, 48, 1), (1024, 112, 1), (256, 16, 1), (1024, 16, 1), (448, 256, 1), (448, 256, 2), (700, 256, 1), (700, 256, 2)]:
    rng = np.random.default_rng(m + k)
    A = rng.standard_normal((m, k))
    r = min(m, k)
    npan = (r + 15) // 16
    src = torch.tensor(np.tile(A.T.copy().ravel(), P), device="cuda")
    dW = src.clone()
    tau = torch.zeros(P * r, dtype=torch.float64, device="cuda")
    tp = torch.zeros(P * (npan * 256 + 2 * r * 16), dtype=torch.float64, device="cuda")
    rank = torch.zeros(4, dtype=torch.int32, device="cuda")
    q = np.zeros(P, _abi.QR_PROB)
    for i in range(P):
        q[i] = (dW.data_ptr() + 8 * i * m * k, tau.data_ptr() + 8 * i * r, tp.data_ptr() + 8 * i * (npan * 256 + 2 * r * 16), 0, m, r, m, -1, k, -1)
    dq = put(q)
    n = P // cl if cl > 1 else P
    ts = []
    for rep in range(3):
        dW.copy_(src); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); rc = lib.hq_qr(None, dq.data_ptr(), n, rank.data_ptr(), cl); e1.record(); torch.cuda.synchronize()
        assert rc == 0
        ts.append(e0.elapsed_time(e1))
    t = min(ts)
    fl = n * (2 * m * k * k - 2 * k ** 3 / 3)
    print(f"qr {m}x{k} x{n} cluster={cl}: {t:.3f} ms  {fl / t / 1e9:.2f} TFLOP/s  {t * 1.965e6 / k:.0f} cycles/column", flush=True)
