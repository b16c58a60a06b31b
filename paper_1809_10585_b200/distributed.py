"""One HODLR matrix factored by several GPUs: the plan's DAG lanes on
different ranks (BASELINE config 3, "partitioned by top-level subtrees").

Algorithm 2 is a chain along the leftmost spine of the tree: factor the
first block column, update the second, factor it.  The planner already
separates the work nothing on that chain waits for -- the truncation of R's
coupling block (hqr.py:153-155), the recompression of every off-spine block
of the updated subtree (the low-rank update of arith.py:126-145 applied to
the independent subtrees of A22) and the whole T phase (hqr.py:169-181) --
into side lanes (plan.Builder.side_lane).  Here lane 0 (the chain, incl. the
power iteration) runs on rank 0 and side lane l on rank 1 + (l - 1) mod
(world - 1), so those subtree updates run on other GPUs while the chain goes
on.

Every rank holds the same arena layout.  The builder records, for every op,
the live allocation instances (region, start, size, generation) and rank
table slots it reads and writes (Builder(track=True)).  Walking the ops in
program order, a rank that is about to touch an instance whose latest version
another rank wrote first receives it (a write counts as read-modify-write:
an op may update part of an allocation).  Every rank follows the same global
order of transfers, so point-to-point sends and receives never deadlock.
The data moved is exactly what the DAG's cross-lane edges carry: factors of
the updated blocks and T / R coupling blocks (bytes per tree level:
DistSchedule.bytes_by_level()).

The executor is transport-agnostic: run(rank, run_op, send, recv) is driven
by NCCL point-to-point calls on GPUs (DistEngine) and by gloo on CPU tensors
with the kernel emulator in the test suite (tests/test_distributed_gloo.py).
"""

from __future__ import annotations

from collections import defaultdict

import numpy as np

from .plan import R_IN, R_OUT, R_PERSIST, Builder, CompiledPlan


def rank_of_lane(lane: int, world: int) -> int:
    if world <= 1 or lane == 0:
        return 0
    return 1 + (lane - 1) % (world - 1)


class DistSchedule:
    """Global sequence of ("op", i, rank) and ("xfer", key, src, dst, i)
    steps for a builder built with track=True."""

    def __init__(self, builder: Builder, world: int):
        if world < 1:
            raise ValueError("world must be >= 1")
        self.builder, self.world = builder, world
        ops = builder.ops
        self.rank_of_op = [rank_of_lane(ex.get("lane", 0), world) for _, _, ex in ops]
        # the input restore (first op) runs on every rank: each rank uploads
        # the packed input itself
        replicated = {0} if ops and ops[0][0] == "pack_copy" and ops[0][2].get("which") == 1 else set()
        everyone = frozenset(range(world))
        holders = defaultdict(lambda: set(everyone))   # key -> ranks holding its latest version
        steps = []
        for i, (kind, probs, ex) in enumerate(ops):
            if "_inst" not in ex:
                raise ValueError("the builder must be built with track=True")
            R, W = ex["_inst"]
            if i in replicated:
                steps.append(("op", i, -1))
                for x in W:
                    holders[x] = set(everyone)
                continue
            r = self.rank_of_op[i]
            for x in sorted(R | W, key=repr):
                h = holders[x]
                if r not in h:
                    steps.append(("xfer", x, min(h), r, i))
                    h.add(r)
            steps.append(("op", i, r))
            for x in W:
                holders[x] = {r}
        self.steps = steps
        self.holders = holders

    # ---------------------------------------------------------------- sizes
    def key_bytes(self, key) -> int:
        if key[0] == "i":
            return 8 * key[3]
        if key[0] == "r":
            return 4
        if key[0] == "scal":
            return 8 * max(2 * self.builder.B, 2)
        if key[0] == "totals":
            return 16
        raise ValueError(key)

    def transfers(self):
        return [s for s in self.steps if s[0] == "xfer"]

    def bytes_total(self) -> int:
        return sum(self.key_bytes(s[1]) for s in self.transfers())

    def bytes_by_level(self) -> dict:
        """Bytes moved between GPUs, by the tree level of the op that needs them."""
        out = defaultdict(int)
        for s in self.transfers():
            out[self.builder.ops[s[4]][2].get("level", -1)] += self.key_bytes(s[1])
        return dict(sorted(out.items()))

    def ops_by_rank(self) -> dict:
        c = defaultdict(int)
        for r in self.rank_of_op:
            c[r] += 1
        return dict(c)

    # ------------------------------------------------------------- executor
    def run(self, rank: int, run_op, send, recv, flush=None):
        """Drive one rank: run_op(i) for its ops (and replicated ones),
        send(key, dst) / recv(key, src) for its transfers in global order.
        flush() (optional) is called before every op that follows a group of
        transfers (batched point-to-point calls complete there)."""
        pending = False
        for st in self.steps:
            if st[0] == "op":
                if st[2] == rank or st[2] == -1:
                    if pending and flush is not None:
                        flush()
                    pending = False
                    run_op(st[1])
            else:
                _, key, src, dst, _ = st
                if src == rank:
                    send(key, dst)
                    pending = True
                elif dst == rank:
                    recv(key, src)
                    pending = True
        if pending and flush is not None:
            flush()


def key_view(plan: CompiledPlan, key):
    """The tensor (a view of the plan's device / host buffers) behind a key."""
    if key[0] == "i":
        _, reg, s, n, _ = key
        o = plan.bases[reg] + s
        return plan.arena[o:o + n]
    if key[0] == "r":
        return plan.rank[key[1]:key[1] + 1]
    if key[0] == "scal":
        return plan.scal
    if key[0] == "totals":
        return plan.totals
    raise ValueError(key)


class DistEngine:
    """hQR of one matrix over the torch.distributed world (NCCL, one GPU per
    rank): every rank builds the same tracked plan, uploads the input, runs
    its lanes' ops on its stream and exchanges allocation instances with
    batched NCCL send / recv; rank 0 ends with the compact factor stream and
    returns the factors (other ranks return None)."""

    def __init__(self, tree, eps, absolute=False, kcap=512, device=None):
        import torch
        import torch.distributed as dist
        from .hqr import PlanIO, _require_cuda
        _require_cuda()
        self.torch, self.dist = torch, dist
        self.world = dist.get_world_size() if dist.is_initialized() else 1
        self.rank = dist.get_rank() if dist.is_initialized() else 0
        self.device = torch.device(device if device is not None else f"cuda:{torch.cuda.current_device()}")
        bld = Builder(tree, 1, eps, absolute, kcap, track=True).build()
        self.io = PlanIO(tree, 1, eps, absolute, kcap, builder=bld)
        self.sched = DistSchedule(bld, self.world)
        self.plan = CompiledPlan(bld, self.device, alias_out=False)
        self.stream = torch.cuda.Stream(device=self.device)

    def factorize(self, a):
        torch, dist, p, io = self.torch, self.dist, self.plan, self.io
        io.pack([a])
        ib = p.bases[R_IN]
        pxo = p.bases[R_PERSIST] + io.builder.PX.off
        lib = __import__("paper_1809_10585_b200._abi", fromlist=["load"]).load()
        s = self.stream
        with torch.cuda.stream(s):
            p.arena[ib:ib + io.n_in].copy_(torch.from_numpy(io.inbuf[:io.n_in]), non_blocking=False)
            p.arena[pxo:pxo + io.px.size].copy_(torch.from_numpy(io.px))
            p.rank.copy_(torch.from_numpy(io.rk))
            p.scal.copy_(torch.from_numpy(io.sc))
        s.synchronize()
        reqs = []

        def run_op(i):
            p._launch_list([p.launch[i]], s.cuda_stream, lib)

        def send(key, dst):
            reqs.append(dist.P2POp(dist.isend, key_view(p, key), dst))

        def recv(key, src):
            reqs.append(dist.P2POp(dist.irecv, key_view(p, key), src))

        def flush():
            if reqs:
                with torch.cuda.stream(s):
                    for w in dist.batch_isend_irecv(reqs):
                        w.wait()
                reqs.clear()
        with torch.cuda.stream(s):
            self.sched.run(self.rank, run_op, send, recv, flush)
            flush()
            # the capacity flag may have been set on any rank
            flag = p.rank[io.builder.flag_slot:io.builder.flag_slot + 1].clone()
            if self.world > 1:
                dist.all_reduce(flag, op=dist.ReduceOp.MAX)
        s.synchronize()
        if int(flag.item()):
            from .hqr import RankCapacityError
            raise RankCapacityError(f"a truncated rank exceeded the capacity kcap={io.kcap}")
        if self.rank != 0:
            return None
        rk = p.rank.cpu().numpy()
        n_out = int(p.totals[1].item())
        ob = p.bases[R_OUT]
        out = p.arena[ob:ob + n_out].cpu().numpy()
        return io.factors(0, out, rk)
