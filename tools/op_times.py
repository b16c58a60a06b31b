"""Per-op device times (CUDA events, non-graph pass, after the cluster
re-tune) of one factorization pass, written as TSV for offline analysis:
index, ms, kind, role/key, lane, level, nprob, max shape.
usage: python tools/op_times.py config [n|0] [batch] [kcap] [out.tsv]"""
import sys
sys.path.insert(0, ".")
import numpy as np, torch
from paper_1809_10585_b200 import gen
from paper_1809_10585_b200.hqr import HQREngine
from paper_1809_10585_b200.plan import _dv
ci = int(sys.argv[1]); n = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2] != "0" else None
B = int(sys.argv[3]) if len(sys.argv) > 3 else 1
kcap = (192 if B > 1 else 512) if len(sys.argv) <= 4 else (sys.argv[4] if sys.argv[4] == "profile" else int(sys.argv[4]))
out = sys.argv[5] if len(sys.argv) > 5 else "gpurun_out/op_times.tsv"
c = gen.CONFIGS[ci]
mats = [gen.gen_config(ci, seed=s, n=n) for s in range(B)]
if kcap == "profile":
    import bench
    kcap = bench.kcap_profile(c, mats[0].tree())
eng = HQREngine(mats[0].tree(), B, c["tol"], kcap=kcap, use_graph=False, stream_out=B > 1)
eng.factorize(mats)
eng.factorize(mats)
rk = eng.h_rk_out.numpy()
plan = eng.plan
eng.pack(mats); eng.upload(); eng.stage_to_live(); torch.cuda.synchronize()
s = eng.stream
evs = []
orig = plan.launch
with torch.cuda.stream(s):
    for rec in orig:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s); plan.launch = [rec]; plan.run(s.cuda_stream); e1.record(s)
        evs.append((e0, e1))
plan.launch = orig
torch.cuda.synchronize()
times = [e0.elapsed_time(e1) for e0, e1 in evs]


def shape(kind, probs):
    if not probs:
        return ""
    if kind == "qr":
        return "m%d k%d" % (max(_dv(p[6], rk) for p in probs), max(_dv(p[7], rk) for p in probs))
    if kind == "qrcp":
        return "m%d n%d r%d" % (max(_dv(p[2], rk) for p in probs), max(_dv(p[3], rk) for p in probs),
                                max(int(rk[p[4]]) for p in probs))
    if kind == "svd":
        return "m%d n%d" % (max(_dv(p[5], rk) for p in probs), max(_dv(p[6], rk) for p in probs))
    if kind == "applyq":
        return "m%d k%d c%d" % tuple(max(_dv(p[i], rk) for p in probs) for i in (8, 9, 10))
    if kind == "gemm":
        return "m%d n%d k%d t%d" % (max(_dv(p[2], rk) for p in probs), max(_dv(p[3], rk) for p in probs),
                                   max(max((_dv(t[8], rk) for t in p[5]), default=0) for p in probs),
                                   max(len(p[5]) for p in probs))
    return ""


with open(out, "w") as fh:
    for i, (kind, probs, ex) in enumerate(eng.builder.ops):
        try:
            sh = shape(kind, probs if isinstance(probs, (list, tuple)) else None)
        except Exception as e:   # noqa: BLE001
            sh = "?"
        key = ex.get("role", "") if isinstance(ex, dict) else ""
        if kind == "svd":
            key = "cl%s%s" % (ex.get("cluster", 1), "b%d" % ex.get("bcluster", 1) if ex.get("block") else "")
        if kind == "qrcp":
            key = "cl%s" % ex.get("cluster", 1)
        if kind == "gemm":
            key = "split%s" % ex.get("ksplit", 1)
        npb = len(probs) if isinstance(probs, (list, tuple)) else 0
        fh.write(f"{i}\t{times[i]:.4f}\t{kind}\t{key}\t{ex.get('lane', -1)}\t{ex.get('level', -1)}\t{npb}\t{sh}\n")
print("total %.1f ms over %d launches" % (sum(times), len(times)))
