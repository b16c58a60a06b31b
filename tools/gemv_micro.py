"""Skinny-product microbenchmark: P problems shaped like the power
iteration's leaf phase (256 rows, leaf term 256 k (ta) + 6 low-rank terms of
rank 16) and like its V^T X phase (rank rows, one A^T term of length K)."""
import sys
sys.path.insert(0, ".")
import numpy as np, torch
from paper_1809_10585_b200 import _abi
lib = _abi.load()
def put(arr):
    return torch.tensor(np.frombuffer(arr.tobytes(), np.uint8), device="cuda")
def timeit(fn, reps=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3
rank = torch.zeros(4, dtype=torch.int32, device="cuda")
P = int(sys.argv[1]) if len(sys.argv) > 1 else 512
# leaf phase
for ta in (0, 1):
    L = torch.randn(P, 256 * 256, dtype=torch.float64, device="cuda")
    U = torch.randn(P, 6, 256 * 16, dtype=torch.float64, device="cuda")
    X = torch.randn(P, 512, dtype=torch.float64, device="cuda")
    T = torch.randn(P, 6, 32, dtype=torch.float64, device="cuda")
    C = torch.zeros(P, 512, dtype=torch.float64, device="cuda")
    terms = np.zeros(P * 7, _abi.GEMM_TERM); probs = np.zeros(P, _abi.GEMM_PROB)
    for p in range(P):
        terms[7 * p] = (L[p].data_ptr(), X[p].data_ptr(), 256, 256, ta, 0, 256, -1, 0, 0, 1.0)
        for q in range(6):
            terms[7 * p + 1 + q] = (U[p, q].data_ptr(), T[p, q].data_ptr(), 256, 16, 0, 0, 16, -1, 0, 0, 1.0)
        probs[p] = (C[p].data_ptr(), 256, 256, -1, 2, -1, 7 * p, 7, 0, 0.0, 0, 0)
    dt, dp = put(terms), put(probs)
    nbytes = (L.numel() + U.numel()) * 8
    for mode in ((0, 1, 2, 3) if ta == 0 else (0, 1, 2, 4)):
        us = timeit(lambda: lib.hq_gemm_skinny(None, dp.data_ptr(), P, dt.data_ptr(), rank.data_ptr(), 1, 2, mode, 256, None))
        print(f"leaf phase P={P} ta={ta} mode {mode}: {us:8.1f} us  {nbytes / us / 1e3:7.1f} GB/s", flush=True)
# split of the mixed A^T leaf phase: leaf term alone (mode 4) + low-rank terms alone (mode 3)
L = torch.randn(P, 256 * 256, dtype=torch.float64, device="cuda")
U = torch.randn(P, 6, 256 * 16, dtype=torch.float64, device="cuda")
X = torch.randn(P, 512, dtype=torch.float64, device="cuda")
T = torch.randn(P, 6, 32, dtype=torch.float64, device="cuda")
C = torch.zeros(P, 512, dtype=torch.float64, device="cuda")
t1 = np.zeros(P, _abi.GEMM_TERM); p1 = np.zeros(P, _abi.GEMM_PROB)
t2 = np.zeros(P * 6, _abi.GEMM_TERM); p2 = np.zeros(P, _abi.GEMM_PROB)
for p in range(P):
    t1[p] = (L[p].data_ptr(), X[p].data_ptr(), 256, 256, 1, 0, 256, -1, 0, 0, 1.0)
    p1[p] = (C[p].data_ptr(), 256, 256, -1, 2, -1, p, 1, 0, 0.0, 0, 0)
    for q in range(6):
        t2[6 * p + q] = (U[p, q].data_ptr(), T[p, q].data_ptr(), 256, 16, 0, 0, 16, -1, 0, 0, 1.0)
    p2[p] = (C[p].data_ptr(), 256, 256, -1, 2, -1, 6 * p, 6, 0, 1.0, 0, 0)
d1, q1, d2, q2 = put(t1), put(p1), put(t2), put(p2)
us1 = timeit(lambda: lib.hq_gemm_skinny(None, q1.data_ptr(), P, d1.data_ptr(), rank.data_ptr(), 1, 2, 4, 256, None))
us2 = timeit(lambda: lib.hq_gemm_skinny(None, q2.data_ptr(), P, d2.data_ptr(), rank.data_ptr(), 1, 2, 3, 256, None))
print(f"split A^T leaf phase P={P}: leaf-only mode 4 {us1:8.1f} us ({L.numel() * 8 / us1 / 1e3:.0f} GB/s) + lowrank mode 3 {us2:8.1f} us ({U.numel() * 8 / us2 / 1e3:.0f} GB/s) = {us1 + us2:8.1f} us", flush=True)
# V^T X phase: rank 16 rows, K = 8192 .. 256 (2 blocks per node, 2**l nodes)
for K, cnt in ((8192, 2), (4096, 4), (1024, 16), (256, 64)):
    Pp = cnt * 8
    V = torch.randn(Pp, K * 16, dtype=torch.float64, device="cuda")
    X = torch.randn(Pp, 2 * K, dtype=torch.float64, device="cuda")
    C = torch.zeros(Pp, 32, dtype=torch.float64, device="cuda")
    terms = np.zeros(Pp, _abi.GEMM_TERM); probs = np.zeros(Pp, _abi.GEMM_PROB)
    for p in range(Pp):
        terms[p] = (V[p].data_ptr(), X[p].data_ptr(), K, K, 1, 0, K, -1, 0, 0, 1.0)
        probs[p] = (C[p].data_ptr(), 16, 16, -1, 2, -1, p, 1, 0, 0.0, 0, 0)
    dt, dp = put(terms), put(probs)
    for mode, ks, mr in ((0, min(32, K // 256), 16), (2, min(32, K // 256), 16), (2, min(32, K // 256), 512)):
        us = timeit(lambda: (C.zero_(), lib.hq_gemm_skinny(None, dp.data_ptr(), Pp, dt.data_ptr(), rank.data_ptr(), ks, 2, mode, mr, None)))
        print(f"VtX K={K} P={Pp} mode {mode} ks {ks} max_rows {mr}: {us:8.1f} us  {V.numel() * 8 / us / 1e3:7.1f} GB/s", flush=True)
