"""N>1 path on CPU: world_size-2 gloo ranks factor their shards of a batch of
independent matrices (the kernel sequence interpreted by the emulator) and
agree on the max time; results equal the single-process batch."""

import os
import socket

import numpy as np
import torch.multiprocessing as mp

from paper_1809_10585_b200.shard import shard_seeds


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    import sys
    import torch
    import torch.distributed as dist
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, here)
    sys.path.insert(0, os.path.dirname(here))
    from emu import emulate
    from paper_1809_10585_b200 import gen
    from paper_1809_10585_b200.hodlr import to_dense
    from paper_1809_10585_b200.shard import max_over_ranks
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    seeds = shard_seeds(4, world, rank)
    mats = [gen.gen_random_hodlr(96, 24, 2, 8.0, seed=s) for s in seeds]
    fs, _, _ = emulate(mats, 1e-10)
    t = max_over_ranks(float(rank + 1))
    out[rank] = (seeds, [to_dense(f.r) for f in fs], t)
    dist.barrier()
    dist.destroy_process_group()


def test_shard_seeds_cover_batch():
    for total in (1, 5, 64):
        for world in (1, 2, 4, 8):
            got = sum((shard_seeds(total, world, r) for r in range(world)), [])
            assert got == list(range(total))


def test_two_rank_gloo_sharded_batch():
    from emu import emulate
    from paper_1809_10585_b200 import gen
    from paper_1809_10585_b200.hodlr import to_dense
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    ref_mats = [gen.gen_random_hodlr(96, 24, 2, 8.0, seed=s) for s in range(4)]
    ref, _, _ = emulate(ref_mats, 1e-10)
    seen = []
    for rank in (0, 1):
        seeds, rs, t = out[rank]
        assert t == 2.0            # max over ranks
        for s, r in zip(seeds, rs):
            seen.append(s)
            assert np.abs(r - to_dense(ref[s].r)).max() <= 1e-12 * np.abs(r).max()
    assert sorted(seen) == [0, 1, 2, 3]
