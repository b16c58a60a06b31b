import sys, time, traceback
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np, torch
from oracle import hqr_oracle as O
from paper_1809_10585_b200 import gen, hqr
from paper_1809_10585_b200.hodlr import to_dense, stats
print("device", torch.cuda.get_device_name(0), flush=True)
for name, a, eps in [("leaf", gen.gen_random_hodlr(48, 64, 1, 8.0, seed=3), 1e-14),
                     ("r64", gen.gen_random_hodlr(64, 16, 2, 8.0, seed=1), 1e-12),
                     ("r256", gen.gen_random_hodlr(256, 32, 4, 8.0, seed=0), 1e-10),
                     ("cfg0", gen.gen_config(0), 1e-10)]:
    try:
        t = time.time()
        f = hqr(a, eps)
        t1 = time.time() - t
        ad = to_dense(a)
        e = O.dense_metrics(ad, f.y, f.t, f.r)
        y, tt, r = O.hqr(a, eps)
        rel = np.linalg.norm(to_dense(f.r) - to_dense(r)) / np.linalg.norm(to_dense(r))
        print(name, "first call %.2fs" % t1, "metrics", e, "R rel", rel, "ranks",
              stats(f.y)["max_offdiag_rank"], stats(f.t)["max_offdiag_rank"], stats(f.r)["max_offdiag_rank"],
              "oracle", stats(y)["max_offdiag_rank"], stats(tt)["max_offdiag_rank"], stats(r)["max_offdiag_rank"], flush=True)
        t = time.time(); f = hqr(a, eps); torch.cuda.synchronize(); print("  second call %.4fs" % (time.time() - t), flush=True)
    except Exception:
        traceback.print_exc()
