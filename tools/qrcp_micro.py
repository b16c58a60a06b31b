"""hq_qrcp time over (cluster, threads) on graded synthetic cores.
    python tools/qrcp_micro.py [sizes] [batch]"""
import sys
sys.path.insert(0, ".")
import numpy as np, torch
from paper_1809_10585_b200 import _abi
from paper_1809_10585_b200.plan import qrcp_smem, QRCP_SMEM_MAX
lib = _abi.load()
sizes = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [48, 96, 144, 208]
P = int(sys.argv[2]) if len(sys.argv) > 2 else 57
for n in sizes:
    rng = np.random.default_rng(n)
    u = np.linalg.qr(rng.standard_normal((n, n)))[0]
    v = np.linalg.qr(rng.standard_normal((n, n)))[0]
    s = np.logspace(0, -14, n)
    C = (u * s) @ v.T
    thr = 1e-10
    src = torch.tensor(np.tile(np.asfortranarray(C).ravel(order="F"), P), device="cuda")
    dC = src.clone()
    rank = torch.zeros(P + 2, dtype=torch.int32, device="cuda")
    scal = torch.ones(2, dtype=torch.float64, device="cuda")
    qp = np.zeros(P, _abi.QRCP_PROB)
    for i in range(P):
        qp[i] = (dC.data_ptr() + 8 * i * n * n, n, n, -1, n, -1, 2 + i, -1, 0, 1e-3 * thr)
    dqp = torch.tensor(np.frombuffer(qp.tobytes(), np.uint8), device="cuda")
    out = []
    for G in (1, 2, 4, 8):
        for nt in (256, 512):
            smem = qrcp_smem(G, n, n, nt)
            if smem is None:
                continue
            ts = []
            for _ in range(3):
                dC.copy_(src); torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                assert lib.hq_qrcp(None, dqp.data_ptr(), P, rank.data_ptr(), scal.data_ptr(), G, smem, nt) == 0
                e1.record(); torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            r = int(rank[2].item())
            out.append("G%d/%d: %.3f ms (%.2f us/step)" % (G, nt, min(ts), 1e3 * min(ts) / max(r, 1)))
    print(n, "batch", P, "r", r, " | ".join(out), flush=True)
