"""hq_qrcp + xform-2 Jacobi against the unpivoted LQ path on real truncation
cores (pickle of (C, thr) from the numpy emulator; triu(C) = R_c).
    python tools/qrcp_ab.py cores.pkl [batch]"""
import sys, pickle
sys.path.insert(0, ".")
import numpy as np, torch
from paper_1809_10585_b200 import _abi
from paper_1809_10585_b200.plan import svd_cluster_runtime, qrcp_launch
lib = _abi.load()
cores = pickle.load(open(sys.argv[1], "rb"))
P = int(sys.argv[2]) if len(sys.argv) > 2 else 57


def put(arr):
    return torch.tensor(np.frombuffer(arr.tobytes(), np.uint8), device="cuda")


def timed(fn, reset):
    ts = []
    for _ in range(3):
        reset()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        assert fn() == 0
        e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return min(ts)


tot = np.zeros(3)
for C, thr in cores:
    Cu = np.triu(C)          # n2 x m: the core as the pivoted QR sees it (any matrix with these singular values)
    k2, k1 = Cu.shape
    ld = (k1 + 1) // 2 * 2
    src = torch.tensor(np.tile(np.asfortranarray(Cu).ravel(order="F"), P), device="cuda")
    dC = src.clone()
    dU = torch.zeros(P * k1 * k1, dtype=torch.float64, device="cuda")
    dW = torch.zeros(P * ld * k1, dtype=torch.float64, device="cuda")
    rank = torch.zeros(3 * P + 2, dtype=torch.int32, device="cuda")
    scal = torch.ones(2, dtype=torch.float64, device="cuda")
    res = {}
    for mode in ("lq", "piv"):
        sp = np.zeros(P, _abi.SVD_PROB)
        qp = np.zeros(P, _abi.QRCP_PROB)
        for i in range(P):
            c = dC.data_ptr() + 8 * i * k2 * k1
            if mode == "lq":
                sp[i] = (c, dU.data_ptr() + 8 * i * k1 * k1, dW.data_ptr() + 8 * i * ld * k1, k2, k1,
                         k1, -1, k2, -1, k1, 2 + i, 1, -1, thr, 1, 0)
            else:
                qp[i] = (c, k2, k2, -1, k1, -1, 2 + P + i, -1, 0, 1e-3 * thr)
                sp[i] = (c, dU.data_ptr() + 8 * i * k1 * k1, dW.data_ptr() + 8 * i * ld * k1, k2, k1,
                         k1, -1, min(k1, k2), 2 + P + i, k1, 2 + i, 1, -1, thr, 2, 0)
        dsp, dqp = put(sp), put(qp)
        tq = 0.0
        if mode == "piv":
            G, smem, nth = qrcp_launch(P, k2, k1)
            tq = timed(lambda: lib.hq_qrcp(None, dqp.data_ptr(), P, rank.data_ptr(), scal.data_ptr(), G, smem, nth),
                       lambda: dC.copy_(src))
            r = int(rank[2 + P].item())
            nn = r
        else:
            nn = min(k1, k2)
        Gs = svd_cluster_runtime(P, k1, nn)
        ts = timed(lambda: lib.hq_svd(None, dsp.data_ptr(), P, rank.data_ptr(), scal.data_ptr(), Gs, k1, 0),
                   (lambda: None) if mode == "piv" else (lambda: dC.copy_(src)))
        k = int(rank[2].item())
        kall = rank[2:2 + P].cpu().numpy()
        U = dU[:k1 * k].cpu().numpy().reshape(k, k1).T
        res[mode] = (tq, ts, k, U, Gs, nn, bool((kall == k).all()))
    (tq0, ts0, ka, Ua, Ga, _, _), (tq, ts, kb, Ub, Gb, r, same) = res["lq"], res["piv"]
    M = Cu.T     # k1 x k2: left singular vectors wanted
    sv = np.linalg.svd(M, compute_uv=False)
    ea = np.linalg.norm(M - Ua @ (Ua.T @ M), 2) / thr
    eb = np.linalg.norm(M - Ub @ (Ub.T @ M), 2) / thr
    G, smem, nth = qrcp_launch(P, k2, k1)
    tot += (ts0, tq, ts)
    print("%s rank %d | LQ svd %.3f ms G=%d k=%d err/thr %.3f | qrcp G=%d %.3f ms r=%d, svd %.3f ms G=%d k=%d err/thr %.3f orth %.1e batch-same %s" %
          (M.shape, int((sv > thr).sum()), ts0, Ga, ka, ea, G, tq, r, ts, Gb, kb, eb,
           np.abs(Ub.T @ Ub - np.eye(kb)).max(), same), flush=True)
print("total: LQ svd %.2f ms | qrcp %.2f + svd %.2f ms" % tuple(tot))
