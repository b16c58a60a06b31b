"""Jacobi time on real truncation cores: the plan's LQ-preconditioned X = R_c^T
against X = (first r rows of a column-pivoted R)^T (r: pivoted diagonal above
delta * thr).  Cores: pickle of (C, thr) dumped from the numpy emulator.
    python tools/jacobi_precond_ab.py cores.pkl [batch] [delta]"""
import sys, pickle
sys.path.insert(0, ".")
import numpy as np, scipy.linalg as sl, torch
from paper_1809_10585_b200 import _abi
from paper_1809_10585_b200.plan import svd_cluster_runtime
lib = _abi.load()
cores = pickle.load(open(sys.argv[1], "rb"))
P = int(sys.argv[2]) if len(sys.argv) > 2 else 57
delta = float(sys.argv[3]) if len(sys.argv) > 3 else 1e-3


def put(arr):
    return torch.tensor(np.frombuffer(arr.tobytes(), np.uint8), device="cuda")


def run(X, thr):
    m, n = X.shape
    ld = (m + 1) // 2 * 2
    dC = torch.tensor(np.tile(np.asfortranarray(X).ravel(order="F"), P), device="cuda")
    dU = torch.zeros(P * m * n, dtype=torch.float64, device="cuda")
    dW = torch.zeros(P * ld * n, dtype=torch.float64, device="cuda")
    rank = torch.zeros(2 * P + 2, dtype=torch.int32, device="cuda")
    scal = torch.zeros(2, dtype=torch.float64, device="cuda")
    p = np.zeros(P, _abi.SVD_PROB)
    for i in range(P):
        p[i] = (dC.data_ptr() + 8 * i * m * n, dU.data_ptr() + 8 * i * m * n, dW.data_ptr() + 8 * i * ld * n, m, m,
                m, -1, n, -1, n, 2 + i, 1, -1, thr, 0, 0)
    dp = put(p)
    G = svd_cluster_runtime(P, m, n)
    src = dC.clone()
    ts = []
    for _ in range(3):
        dC.copy_(src)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        assert lib.hq_svd(None, dp.data_ptr(), P, rank.data_ptr(), scal.data_ptr(), G, m, 0) == 0
        e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    k = int(rank[2].item())
    U = dU[:m * k].cpu().numpy().reshape(k, m).T
    return min(ts), k, U, G


tot = [0.0, 0.0]
for C, thr in cores:
    Cu = np.triu(C)
    Xa = Cu.T.copy()
    ta, ka, Ua, Ga = run(Xa, thr)
    Q, Rp, perm = sl.qr(Cu, pivoting=True)
    dg = np.abs(np.diag(Rp))
    r = max(1, int((dg > delta * thr).sum()))
    Xb = np.zeros((Cu.shape[1], r))
    Xb[perm, :] = Rp[:r].T
    tb, kb, Ub, Gb = run(Xb, thr)
    # both bases span (nearly) the same subspace; projection error of X on U
    ea = np.linalg.norm(Xa - Ua @ (Ua.T @ Xa), 2) / thr
    eb = np.linalg.norm(Xa @ Xa.T - Ub @ (Ub.T @ Xa @ Xa.T), 2)
    sv = np.linalg.svd(Xa, compute_uv=False)
    tot[0] += ta; tot[1] += tb
    print("%s rank %d | LQ: %.3f ms G=%d k=%d projerr/thr %.2f | piv r=%d: %.3f ms G=%d k=%d orth %.1e" %
          (Xa.shape, int((sv > thr).sum()), ta, Ga, ka, ea, r, tb, Gb, kb, np.abs(Ub.T @ Ub - np.eye(kb)).max()), flush=True)
print("total LQ %.2f ms  pivoted %.2f ms" % tuple(tot))
