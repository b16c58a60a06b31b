"""Config-3 style partitioning of ONE matrix over ranks (distributed.py) on
CPU: world_size-2 gloo ranks run their lanes' ops through the kernel
emulator and exchange allocation instances point to point; rank 0's factors
equal the single-process run bit for bit."""

import os
import socket

import numpy as np
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _case():
    from paper_1809_10585_b200 import gen
    return gen.gen_random_hodlr(512, 32, 4, 8.0, seed=3), 1e-10


def _emulate_rank(rank, world, send, recv, flush):
    """Every rank: the tracked plan on a CPU arena, its ops through the
    emulator, transfers through the given callbacks."""
    import torch
    from emu import Emu
    from paper_1809_10585_b200.distributed import DistSchedule, key_view
    from paper_1809_10585_b200.hqr import PlanIO
    from paper_1809_10585_b200.plan import R_IN, R_OUT, R_PERSIST, Builder, CompiledPlan
    a, eps = _case()
    bld = Builder(a.tree(), 1, eps, False, 512, track=True).build()
    io = PlanIO(a.tree(), 1, eps, False, 512, builder=bld)
    sched = DistSchedule(bld, world)
    plan = CompiledPlan(bld, torch.device("cpu"), alias_out=False)
    io.pack([a])
    A = plan.arena.numpy()
    ib = plan.bases[R_IN]
    A[ib:ib + io.n_in] = io.inbuf[:io.n_in]
    pxo = plan.bases[R_PERSIST] + bld.PX.off
    A[pxo:pxo + io.px.size] = io.px
    plan.rank.numpy()[:] = io.rk
    plan.scal.numpy()[:] = io.sc
    emu = Emu(plan)
    sched.run(rank, lambda i: emu.run_ops([plan.launch[i]]), lambda k, d: send(key_view(plan, k), d),
              lambda k, s: recv(key_view(plan, k), s), flush)
    out = None
    if rank == 0:
        n_out = int(plan.totals.numpy()[1])
        ob = plan.bases[R_OUT]
        out = (A[ob:ob + n_out].copy(), plan.rank.numpy().copy())
    return out, sched


def _worker(rank, world, port, res):
    import sys
    import torch.distributed as dist
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, here)
    sys.path.insert(0, os.path.dirname(here))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    reqs = []

    def flush():
        for w in reqs:
            w.wait()
        reqs.clear()
    out, sched = _emulate_rank(rank, world, lambda t, d: reqs.append(dist.isend(t, d)),
                               lambda t, s: reqs.append(dist.irecv(t, s)), flush)
    res[rank] = (out, sched.ops_by_rank(), sched.bytes_total(), sched.bytes_by_level())
    dist.barrier()
    dist.destroy_process_group()


def test_schedule_partitions_side_lanes():
    from paper_1809_10585_b200.distributed import DistSchedule
    from paper_1809_10585_b200.plan import Builder
    a, eps = _case()
    bld = Builder(a.tree(), 1, eps, False, 512, track=True).build()
    for world in (2, 4):
        s = DistSchedule(bld, world)
        byr = s.ops_by_rank()
        assert set(byr) == set(range(world)) and all(v > 0 for v in byr.values())
        assert s.bytes_total() > 0
        assert sum(s.bytes_by_level().values()) == s.bytes_total()
    one = DistSchedule(bld, 1)
    assert not one.transfers()


def test_two_rank_gloo_matches_single_process():
    mgr = mp.Manager()
    res = mgr.dict()
    mp.spawn(_worker, args=(2, _free_port(), res), nprocs=2, join=True)
    (out, rk), byr, tot, lvl = res[0]
    (ref, rk_ref), _ = _emulate_rank(0, 1, None, None, None)
    # the factor stream and the ranks it is laid out by (rank 0 need not hold
    # scratch slots that only the side lanes used)
    from paper_1809_10585_b200.plan import Builder
    a, eps = _case()
    bld = Builder(a.tree(), 1, eps, False, 512).build()
    slots = sorted({c.ri for _, _, c, _ in bld.out_items if c.ri >= 0})
    assert np.array_equal(rk[slots], rk_ref[slots])
    assert out.shape == ref.shape and np.array_equal(out, ref)
    assert byr[1] > 0 and tot > 0
