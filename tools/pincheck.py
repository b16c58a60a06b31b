import sys, gc
sys.path.insert(0, ".")
import torch
from paper_1809_10585_b200 import gen
from paper_1809_10585_b200.hqr import HQREngine
B = 4
mats = [gen.gen_config(2, seed=s, n=4096) for s in range(B)]
eng = HQREngine(mats[0].tree(), B, 1e-10)
use = torch._C._storage_Use_Count
def counts(): return [(b.numel() >> 20, use(b.untyped_storage()._cdata)) for b in eng._pins]
for i in range(4):
    f = eng.factorize(mats)
    print(i, "alive", counts(), eng.pin_allocs)
    del f
    print(i, "freed", counts())
    gc.collect()
    print(i, "gc", counts())
