"""Per-batch host timeline of HQREngine.factorize_stream on the bench engine
(ms since the batch's launch_main began): packed, replay_enqueued,
device_done, d2h_enqueued, assembled.
    python tools/stream_trace.py [batches] [batch size]"""
import sys, time
sys.path.insert(0, ".")
import torch
import bench
nb = int(sys.argv[1]) if len(sys.argv) > 1 else 6
B = int(sys.argv[2]) if len(sys.argv) > 2 else None
eng, mats, kc, _ = bench.build_engine(torch, 2, 16384, batch=B)
for f in eng.factorize_stream([mats] * 2):
    del f
import gc
t0 = time.perf_counter(); n_unreach = gc.collect(); print("gc.collect: %.0f ms, %d objects tracked" % ((time.perf_counter() - t0) * 1e3, len(gc.get_objects())))
if len(sys.argv) > 3:
    gc.freeze(); print("gc.freeze()")
torch.cuda.synchronize()
t0 = time.perf_counter()
tl = t0
for i, f in enumerate(eng.factorize_stream([mats] * nb)):
    now = time.perf_counter()
    print(i, "yield after %.0f ms" % ((now - tl) * 1e3), {k: round(v) for k, v in eng.last_trace.items()}, flush=True)
    tl = now
    del f
tot = time.perf_counter() - t0
print("batch %d: %.1f ms per batch, %.2f factorizations/s" % (len(mats), tot / nb * 1e3, len(mats) * nb / tot))
print("pin_allocs", getattr(eng, "pin_allocs", 0), "pool", len(eng._pins))
for _ in range(2):
    t0 = time.perf_counter()
    f = eng.factorize(mats)
    print("factorize: %.0f ms" % ((time.perf_counter() - t0) * 1e3), {k: round(v) for k, v in eng.last_trace.items()},
          "pin_allocs", getattr(eng, "pin_allocs", 0), flush=True)
    del f
# raw D2H of the output region into one pinned block, device idle
n = eng.n_out
hb = torch.empty(n, dtype=torch.float64, pin_memory=True)
for _ in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    hb.copy_(eng.d_out[:n], non_blocking=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print("raw D2H %.1f GB in %.0f ms = %.1f GB/s" % (8 * n / 1e9, dt * 1e3, 8 * n / 1e9 / dt))
