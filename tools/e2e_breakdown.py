"""Phase breakdown of HQREngine.factorize (host pack / H2D / replay / D2H+assembly)."""
import sys, time
sys.path.insert(0, ".")
import torch
from paper_1809_10585_b200 import gen
from paper_1809_10585_b200.hqr import HQREngine
ci = int(sys.argv[1]) if len(sys.argv) > 1 else 2
B = int(sys.argv[2]) if len(sys.argv) > 2 else 8
c = gen.CONFIGS[ci]
mats = [gen.gen_config(ci, seed=s) for s in range(B)]
eng = HQREngine(mats[0].tree(), B, c["tol"])
for _ in range(2):
    f = eng.factorize(mats)
del f
T = {}
def tick(k, t0, sync=True):
    if sync: torch.cuda.synchronize()
    T[k] = T.get(k, 0) + time.perf_counter() - t0; return time.perf_counter()
R = 3
for _ in range(R):
    t = time.perf_counter()
    eng.pack(mats); t = tick("pack", t)
    eng.upload(); t = tick("h2d", t)
    eng.execute(); t = tick("replay_enqueue", t, False)
    torch.cuda.synchronize(); t = tick("replay_wait", t)
    eng.download(); t = tick("d2h_staging", t)
    fs = [eng.factors(b) for b in range(B)]; t = tick("assemble_serial", t)
    del fs
    f = eng.factorize(mats); t = tick("factorize_total", t); print({k: round(v, 1) for k, v in eng.last_trace.items()}, "pin_allocs", getattr(eng, "pin_allocs", 0))
    del f
print(f"B={B}", {k: round(v / R * 1e3, 1) for k, v in T.items()}, "ms; bytes in %.0f MB out %.0f MB" %
      (eng.h2d_bytes() / 1e6, eng.d2h_bytes() / 1e6))
