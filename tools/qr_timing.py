import sys, ctypes
sys.path.insert(0, ".")
import numpy as np, torch
from paper_1809_10585_b200 import _abi
lib = _abi.load()
dbg = torch.zeros(4096, dtype=torch.int64, device="cuda")
if hasattr(lib, "hq_debug_set"):
    lib.hq_debug_set.argtypes = [ctypes.c_void_p]
    lib.hq_debug_set(dbg.data_ptr())
def put(arr): return torch.tensor(np.frombuffer(arr.tobytes(), np.uint8), device="cuda")
m = int(sys.argv[1]) if len(sys.argv) > 1 else 400
k = int(sys.argv[2]) if len(sys.argv) > 2 else 256
cl = int(sys.argv[3]) if len(sys.argv) > 3 else 8
full = 1
A = np.random.default_rng(1).standard_normal((m, k))
for rep in range(2):
    dW = torch.tensor(A.T.copy(), device="cuda"); r = min(m, k)
    tau = torch.zeros(r, dtype=torch.float64, device="cuda"); tp = torch.zeros(((r + 15) // 16) * 256 + 2 * r * 16, dtype=torch.float64, device="cuda")
    tf = torch.zeros(r * r, dtype=torch.float64, device="cuda"); rank = torch.zeros(4, dtype=torch.int32, device="cuda")
    q = np.zeros(1, _abi.QR_PROB); q[0] = (dW.data_ptr(), tau.data_ptr(), tp.data_ptr(), tf.data_ptr() if full else 0, m, r, m, -1, k, -1)
    dq = put(q); torch.cuda.synchronize()
    lib.hq_qr(None, dq.data_ptr(), 1, rank.data_ptr(), cl); torch.cuda.synchronize()
dd = dbg.cpu().numpy(); d = dd[:2048].reshape(8, 64, 4)
acc, cnt = dd[2048:2064], dd[2064:2080]
names = {0: "apply W", 1: "apply T", 2: "apply X", 4: "f stage", 5: "f factor", 6: "f wb", 8: "reg cols", 9: "reg T"}
print({names[k]: (int(acc[k] // max(cnt[k], 1)), int(cnt[k])) for k in names})
np.set_printoptions(linewidth=200)
print("per phase (cycles): [applyfirst, factor, rest(pass1), barrier] for CTA 0..7")
for ph in range(17):
    print(ph, [tuple(int(x) for x in d[c, ph]) for c in range(8)][:8])
