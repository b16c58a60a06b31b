"""Bytes exchanged between GPUs when one matrix is partitioned over ranks
(distributed.py): per tree level, for world sizes 2, 4, 8 (host-side plan
analysis, no GPU).  python tools/dist_bytes.py [config]"""
import sys, time
sys.path.insert(0, ".")
from paper_1809_10585_b200 import gen
from paper_1809_10585_b200.distributed import DistSchedule
from paper_1809_10585_b200.plan import Builder
ci = int(sys.argv[1]) if len(sys.argv) > 1 else 3
c = gen.CONFIGS[ci]
t0 = time.time()
tree = gen.gen_config(ci, seed=0).tree() if ci != 3 else __import__("paper_1809_10585_b200.hodlr", fromlist=["x"]).build_partition(c["n"], c["leaf"])
bld = Builder(tree, 1, c["tol"], False, 512, track=True).build()
print(f"config {ci}: n={tree.n}, {len(bld.ops)} ops, plan built in {time.time() - t0:.1f} s")
for world in (2, 4, 8):
    s = DistSchedule(bld, world)
    lv = s.bytes_by_level()
    print(f"world {world}: ops per rank {s.ops_by_rank()}, transfers {len(s.transfers())}, "
          f"{s.bytes_total() / 1e6:.1f} MB total; by level (MB): " +
          ", ".join(f"{k}: {v / 1e6:.1f}" for k, v in lv.items()), flush=True)
