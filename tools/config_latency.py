"""Single-matrix latency (graph replay, input resident) of every BASELINE config,
plus the CPU oracle's single-threaded time for the small ones."""
import sys, time
sys.path.insert(0, ".")
import torch
from paper_1809_10585_b200 import gen
from paper_1809_10585_b200.hqr import HQREngine
for ci in range(5):
    c = gen.CONFIGS[ci]
    a = gen.gen_config(ci, seed=0)
    eng = HQREngine(a.tree(), 1, c["tol"], kcap=512)
    eng.pack([a]); eng.upload(); eng.snapshot_device_input()
    eng.execute(); eng.download()          # capture, first run, cluster re-tune
    for _ in range(2):
        eng.restore_device_input(); eng.execute()
    eng.stream.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(eng.stream)
    for _ in range(3):
        eng.restore_device_input(); eng.execute()
    e1.record(eng.stream); e1.synchronize()
    ms = e0.elapsed_time(e1) / 3
    t = time.perf_counter(); eng.factorize([a]); e2e = (time.perf_counter() - t) * 1e3
    print(f"config {ci}: n={a.n} latency {ms:.1f} ms (device, graph replay), {e2e:.1f} ms through hqr/factorize", flush=True)
    del eng
    torch.cuda.empty_cache()
