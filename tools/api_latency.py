"""Single-call latency of the reference-facing entry point hqr(a, eps) per
config (host matrices in, HodlrMatrix factors out), against the device-only
graph replay of the same engine; per-phase trace of the last call."""
import sys, time
sys.path.insert(0, ".")
import torch
from paper_1809_10585_b200 import gen, hqr
from paper_1809_10585_b200.hqr import engine_for
cfgs = [int(x) for x in sys.argv[1:]] or [0, 1, 2, 4]
for ci in cfgs:
    c = gen.CONFIGS[ci]
    a = gen.gen_config(ci, seed=0)
    for _ in range(2):
        f = hqr(a, c["tol"]); del f
    ts = []
    for _ in range(5):
        t = time.perf_counter(); f = hqr(a, c["tol"]); ts.append((time.perf_counter() - t) * 1e3); del f
    eng = engine_for(a.tree(), 1, c["tol"], False, 512)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    eng.pack([a]); eng.upload()
    eng.snapshot_device_input()   # the run state as uploaded (not a finished run's)
    e0.record(eng.stream)
    for _ in range(3):
        eng.restore_device_input(); eng.execute()
    e1.record(eng.stream); e1.synchronize()
    print(f"config {ci}: hqr() {min(ts):.1f} ms (min of 5; all {[round(x, 1) for x in ts]}), replay "
          f"{e0.elapsed_time(e1) / 3:.1f} ms, trace {eng.last_trace}, pin_allocs {getattr(eng, 'pin_allocs', 0)}", flush=True)
