"""Per-op differential test: GPU kernel vs numpy emulator on identical state."""
import sys
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np, torch
from emu import Emu
from paper_1809_10585_b200 import gen
from paper_1809_10585_b200.hqr import HQREngine
from paper_1809_10585_b200.plan import CompiledPlan
n = int(sys.argv[1]) if len(sys.argv) > 1 else 50
leaf = int(sys.argv[2]) if len(sys.argv) > 2 else 24
a = gen.gen_random_hodlr(n, leaf, 3, 8.0, seed=2)
eng = HQREngine(a.tree(), 1, 1e-12, use_graph=False)
eng.pack([a]); eng.upload(); torch.cuda.synchronize()
gp = eng.plan
cp = CompiledPlan(eng.builder, torch.device("cpu"))
em = Emu(cp)
# map GPU pointers in descriptors -> CPU arena: emulator uses cpu plan descriptors (same layout)
for i, rec in enumerate(gp.launch):
    # sync state gpu -> cpu
    cp.arena.copy_(gp.arena.cpu()); cp.rank.copy_(gp.rank.cpu()); cp.scal.copy_(gp.scal.cpu()); cp.totals.copy_(gp.totals.cpu())
    # run op on GPU
    saved = gp.launch; gp.launch = [rec]; gp.run(torch.cuda.current_stream().cuda_stream); gp.launch = saved
    torch.cuda.synchronize()
    # run op on emulator
    saved = cp.launch; cp.launch = [cp.launch[i]]; em.run(); cp.launch = saved
    ga, ea = gp.arena.cpu().numpy(), cp.arena.numpy()
    gr, er = gp.rank.cpu().numpy(), cp.rank.numpy()
    d = np.abs(ga - ea)
    kind = rec[0]
    if kind in ("svd", "power"):
        rdiff = np.abs(gr - er).max()
        if rdiff: print(i, kind, "RANK DIFF", np.nonzero(gr != er), gr[gr != er], er[gr != er]); break
        continue
    if d.max() > 1e-9 * max(1, np.abs(ea).max()) or (gr != er).any():
        j = int(d.argmax())
        print(f"op {i} {kind}: max diff {d.max():.3e} at {j} gpu {ga[j]:.6e} emu {ea[j]:.6e}; rank diff {np.nonzero(gr != er)[0][:10]}", flush=True)
        print("  region bases", gp.bases, "desc", rec[1:4], rec[4])
        break
else:
    print("no divergence")
# detail for the diverging op
from paper_1809_10585_b200 import _abi
if kind == "qr":
    arr = np.frombuffer(gp.desc.cpu().numpy()[rec[1]:rec[1] + 56 * rec[3]].tobytes(), _abi.QR_PROB)
    base = gp.arena.data_ptr()
    for p in arr:
        print({k: ((int(p[k]) - base) // 8 if k in ("w", "tau", "tpanel", "tfull") and p[k] else p[k]) for k in arr.dtype.names})
bad = np.nonzero(d > 1e-9)[0]
print("n differing", bad.size, "first", bad[:20], "last", bad[-5:])
print("gpu vals", ga[bad[:10]], "emu vals", ea[bad[:10]])
print("rank table", gr[:40])
