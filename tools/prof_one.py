"""One factorization pass of a config (for ncu launch lists / captures).
usage: python tools/prof_one.py config [n|0] [batch] [kcap|bench]
The first (untimed) factorization re-tunes the cluster sizes; the second pass,
bracketed by cudaProfilerStart/Stop, is what `ncu --profile-from-start off`
sees (non-graph launches, so every kernel is listed)."""
import sys
sys.path.insert(0, ".")
import torch
from paper_1809_10585_b200 import gen
from paper_1809_10585_b200.hqr import HQREngine
ci = int(sys.argv[1]); n = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2] != "0" else None
B = int(sys.argv[3]) if len(sys.argv) > 3 else 1
kcap = sys.argv[4] if len(sys.argv) > 4 else "512"
c = gen.CONFIGS[ci]
mats = [gen.gen_config(ci, seed=s, n=n) for s in range(B)]
if kcap == "bench":   # the per-level capacity profile bench.py times
    import bench
    kcap = bench.kcap_profile(c, mats[0].tree())
else:
    kcap = int(kcap)
eng = HQREngine(mats[0].tree(), B, c["tol"], kcap=kcap, use_graph=False, stream_out=B > 1)
eng.factorize(mats)
eng.pack(mats); eng.upload(); torch.cuda.synchronize()
torch.cuda.profiler.start()
eng.execute(); torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("ok launches", eng.plan.n_launch)
