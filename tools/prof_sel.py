"""One factorization pass of the bench workload in which only SELECTED ops are
bracketed by cudaProfilerStart/Stop, so that one `ncu --profile-from-start off
--set full` run captures one launch per kernel class (instead of one
application run per class).
usage: python tools/prof_sel.py config [n|0] batch kcap|bench name:occurrence[,name:occurrence...]
names: gemm64 gemm32 gemv applyq concat qr qrcl qrcp qrcpcl svdcl<G> svdsmall svdblock ...
(the classes present and their launch counts are printed first)"""
import sys
sys.path.insert(0, ".")
import torch
from paper_1809_10585_b200 import gen
from paper_1809_10585_b200.hqr import HQREngine
ci = int(sys.argv[1]); n = int(sys.argv[2]) if sys.argv[2] != "0" else None
B = int(sys.argv[3]); kcap = sys.argv[4]
sel = [(a.split(":")[0], int(a.split(":")[1])) for a in sys.argv[5].split(",")]
c = gen.CONFIGS[ci]
mats = [gen.gen_config(ci, seed=s, n=n) for s in range(B)]
if kcap == "bench":
    import bench
    kcap = bench.kcap_profile(c, mats[0].tree())
else:
    kcap = int(kcap)
eng = HQREngine(mats[0].tree(), B, c["tol"], kcap=kcap, use_graph=False, stream_out=B > 1)
eng.factorize(mats)
plan = eng.plan


def cls(rec):
    kind, ex = rec[0], rec[-1]
    if kind == "gemm":
        if ex.get("skinny"):
            return "gemv"
        return "gemm%d" % ex.get("tile", 64)
    if kind == "svd":
        if ex.get("block"):
            return "svdblock"
        if ex.get("small"):
            return "svdsmall"
        return "svdcl%d" % ex.get("cluster", 1)
    if kind in ("qr", "qrcp") and ex.get("cluster", 1) > 1:
        return kind + "cl"
    return kind


seen, chosen = {}, {}
for i, rec in enumerate(plan.launch):
    k = cls(rec)
    seen[k] = seen.get(k, 0) + 1
    for name, occ in sel:
        if name == k and seen[k] == occ + 1:
            chosen[i] = "%s:%d" % (name, occ)
print("classes:", seen, flush=True)
print("chosen:", chosen, flush=True)
eng.pack(mats); eng.upload(); eng.stage_to_live(); torch.cuda.synchronize()
s = eng.stream
orig = plan.launch
with torch.cuda.stream(s):
    for i, rec in enumerate(orig):
        plan.launch = [rec]
        if i in chosen:
            torch.cuda.synchronize(); torch.cuda.profiler.start()
        plan.run(s.cuda_stream)
        if i in chosen:
            torch.cuda.synchronize(); torch.cuda.profiler.stop()
plan.launch = orig
torch.cuda.synchronize()
print("ok")
