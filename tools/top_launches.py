"""Per-launch device times (CUDA events, non-graph pass) with problem shapes."""
import sys
sys.path.insert(0, ".")
import numpy as np, torch
from paper_1809_10585_b200 import gen
from paper_1809_10585_b200.hqr import HQREngine
from paper_1809_10585_b200.plan import _dv
ci = int(sys.argv[1]); n = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2] != "0" else None
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
B = int(sys.argv[4]) if len(sys.argv) > 4 else 1
c = gen.CONFIGS[ci]
mats = [gen.gen_config(ci, seed=s, n=n) for s in range(B)]
a = mats[0]
eng = HQREngine(a.tree(), B, c["tol"], kcap=192 if B > 1 else 512, use_graph=False)
eng.factorize(mats)
rk = eng.h_rk_out.numpy()
plan = eng.plan
eng.upload(); torch.cuda.synchronize()
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
ops = eng.builder.ops
def shape(kind, probs):
    if probs is None: return ""
    if kind == "qr": return [( _dv(p[6], rk), _dv(p[7], rk), p[3] is not None) for p in probs][:4]
    if kind == "svd": return [(_dv(p[5], rk), _dv(p[6], rk)) for p in probs][:4]
    if kind == "applyq": return [(_dv(p[8], rk), _dv(p[9], rk), _dv(p[10], rk)) for p in probs][:4]
    if kind == "gemm": return [(_dv(p[2], rk), _dv(p[3], rk), [_dv(t[8], rk) for t in p[5]][:3]) for p in probs][:3]
    return len(probs)
order = np.argsort(times)[::-1][:top]
tot = sum(times)
print(f"total {tot:.1f} ms over {len(times)} launches")
for i in order:
    kind, probs, ex = ops[i]
    print(f"{times[i]:8.3f} ms  {kind:8s} nprob={0 if probs is None else len(probs):4d} {shape(kind, probs)}")
# breakdown by kind / size class
import collections
agg = collections.defaultdict(lambda: [0.0, 0])
for i, (kind, probs, ex) in enumerate(ops):
    key = kind
    if kind == "qr" and probs:
        mm = max(_dv(p[6], rk) for p in probs)
        leaf = probs[0][3] is not None
        key = f"qr {'leaf' if leaf else 'trunc'} m{'<=512' if mm <= 512 else ('<=1024' if mm <= 1024 else '>1024')}"
    elif kind == "svd" and probs:
        key = f"svd cl{ex.get('cluster',1)}"
    elif kind == "gemm" and probs:
        kk = max(max((_dv(t[8], rk) for t in p[5]), default=0) for p in probs)
        key = f"gemm k{'<=256' if kk <= 256 else ('<=2048' if kk <= 2048 else '>2048')} split{ex['ksplit']}"
    agg[key][0] += times[i]; agg[key][1] += 1
for k, (tm, c) in sorted(agg.items(), key=lambda x: -x[1][0]):
    print(f"{k:32s} {c:5d} launches {tm:9.1f} ms")
# critical path through the DAG (per-op times from this serialized pass)
from paper_1809_10585_b200.plan import op_resources
lanes = plan.lanes
finish = [0.0] * len(ops)
pred = [-1] * len(ops)
last_in_lane = {}
last_w, readers = {}, {}
for i, (kind, probs, ex) in enumerate(ops):
    Rs, Ws = op_resources(eng.builder, kind, probs, ex)
    deps = set()
    for r in Rs | Ws:
        if r in last_w: deps.add(last_w[r])
    for r in Ws: deps.update(readers.get(r, ()))
    ln = lanes[i]
    if ln in last_in_lane: deps.add(last_in_lane[ln])
    best = max(deps, key=lambda d: finish[d], default=-1)
    finish[i] = (finish[best] if best >= 0 else 0.0) + times[i]
    pred[i] = best
    last_in_lane[ln] = i
    for r in Rs: readers.setdefault(r, []).append(i)
    for r in Ws: last_w[r] = i; readers[r] = []
end = max(range(len(ops)), key=lambda i: finish[i])
print(f"critical path {finish[end]:.1f} ms (serialized sum {sum(times):.1f} ms)")
cp = collections.defaultdict(lambda: [0.0, 0])
i = end
while i >= 0:
    kind, probs, ex = ops[i]
    key = kind
    if kind == "qr" and probs:
        mm = max(_dv(p[6], rk) for p in probs)
        key = f"qr {'leaf' if probs[0][3] is not None else 'trunc'} m{'<=512' if mm <= 512 else ('<=1024' if mm <= 1024 else '>1024')}"
    elif kind == "svd":
        key = f"svd cl{ex.get('cluster',1)}"
    cp[key][0] += times[i]; cp[key][1] += 1
    i = pred[i]
for k, (tm, c) in sorted(cp.items(), key=lambda x: -x[1][0]):
    print(f"  on path: {k:28s} {c:5d} ops {tm:9.1f} ms")
# on-path detail for one kind: shape buckets
detail = sys.argv[5] if len(sys.argv) > 5 else None
if detail:
    dd = collections.defaultdict(lambda: [0.0, 0])
    i = end
    while i >= 0:
        kind, probs, ex = ops[i]
        if kind == detail and probs:
            if kind == "qr":
                sh = max((_dv(p[6], rk), _dv(p[7], rk)) for p in probs)
                key = (len(probs), (sh[0] + 63) // 64 * 64, (sh[1] + 15) // 16 * 16, ex.get("cluster", 1) if isinstance(ex, dict) else ex)
            elif kind == "gemm":
                mm = max(_dv(p[2], rk) for p in probs); nn = max(_dv(p[3], rk) for p in probs)
                kk = max(max((_dv(t[8], rk) for t in p[5]), default=0) for p in probs)
                nterm = max(len(p[5]) for p in probs)
                key = (len(probs), ex.get("ksplit"), "m%d" % ((mm + 63) // 64 * 64), "n%d" % ((nn + 15) // 16 * 16), "k%d" % ((kk + 63) // 64 * 64), "t%d" % nterm)
            else:
                key = (len(probs),)
            dd[key][0] += times[i]; dd[key][1] += 1
        i = pred[i]
    print(f"on-path {detail} by (nprob, m64, k16, extra):")
    for k, (tm, c) in sorted(dd.items(), key=lambda x: -x[1][0])[:30]:
        print(f"    {str(k):40s} {c:4d} ops {tm:8.2f} ms  avg {1000 * tm / c:7.1f} us")
if detail == "gemm":
    from paper_1809_10585_b200.plan import op_flops
    allc = collections.defaultdict(lambda: [0.0, 0, 0.0])
    for i, (kind, probs, ex) in enumerate(ops):
        if kind != "gemm" or not probs:
            continue
        mm = max(_dv(p[2], rk) for p in probs); nn = max(_dv(p[3], rk) for p in probs)
        kk = max(sum(_dv(t[8], rk) for t in p[5]) for p in probs)
        key = (len(probs), ex.get("ksplit"), ex.get("tile"), "m%d" % (1 << max(0, (mm - 1)).bit_length()),
               "n%d" % (1 << max(0, (nn - 1)).bit_length()), "k%d" % (1 << max(0, (kk - 1)).bit_length()))
        allc[key][0] += times[i]; allc[key][1] += 1; allc[key][2] += op_flops(kind, probs, rk)
    print("all gemm ops by (nprob, ksplit, tile, m, n, sum k) pow2 classes:")
    for k, (tm, c, fl) in sorted(allc.items(), key=lambda x: -x[1][0])[:30]:
        print(f"    {str(k):56s} {c:4d} ops {tm:8.2f} ms  avg {1000 * tm / c:7.1f} us  {fl / max(tm, 1e-9) / 1e9:6.2f} TF/s")
if detail == "qr":
    allc = collections.defaultdict(lambda: [0.0, 0, 0])
    for i, (kind, probs, ex) in enumerate(ops):
        if kind != "qr" or not probs:
            continue
        mm = max(_dv(p[6], rk) for p in probs); kk = max(_dv(p[7], rk) for p in probs)
        key = (ex.get("role"), ex.get("cluster"), len(probs), "m%d" % (1 << max(0, mm - 1).bit_length()), "k%d" % (1 << max(0, kk - 1).bit_length()))
        allc[key][0] += times[i]; allc[key][1] += 1
    print("all qr ops by (role, cluster, nprob, m, k) pow2 classes:")
    for k, (tm, c, _) in sorted(allc.items(), key=lambda x: -x[1][0])[:30]:
        print(f"    {str(k):56s} {c:4d} ops {tm:8.2f} ms  avg {1000 * tm / c:7.1f} us")
