"""numpy emulator of libhqb200.so's kernels -- TEST INFRASTRUCTURE ONLY.

Interprets a CompiledPlan built on the CPU (host pointers in the packed
descriptors) with the exact semantics documented in include/hodlrqr_b200.h.
It lets the non-GPU test tier check the host-side planner (layout, descriptor
packing, the unrolled recursion) against the oracle without a B200.  It is
never used by the product path.
"""

import numpy as np

from paper_1809_10585_b200 import _abi

NB = 16


class Emu:
    def __init__(self, plan):
        self.plan = plan
        self.A = plan.arena.numpy()
        self.base = plan.arena.data_ptr()
        self.rank = plan.rank.numpy()
        self.scal = plan.scal.numpy()
        self.desc = plan.desc.numpy()

    # ---------------------------------------------------------------- helpers
    def idx(self, ptr):
        d = int(ptr) - self.base
        assert d % 8 == 0 and 0 <= d < 8 * self.A.size, "pointer outside arena"
        return d // 8

    def mat(self, ptr, ld, rows, cols):
        if rows <= 0 or cols <= 0:
            return np.zeros((max(rows, 0), max(cols, 0)))
        i = self.idx(ptr)
        assert i + (cols - 1) * ld + rows <= self.A.size
        return np.lib.stride_tricks.as_strided(self.A[i:], shape=(rows, cols), strides=(8, 8 * ld))

    def dim(self, d, ri):
        if ri < 0:
            return int(d)
        return int(min(max(self.rank[ri], 0), d))

    def arr(self, off, dtype, count):
        return np.frombuffer(self.desc[off:off + dtype.itemsize * count].tobytes(), dtype=dtype)

    @staticmethod
    def masked(s, mask):
        if mask == 1:
            return np.triu(s)
        if mask == 2:
            out = np.tril(s, -1)
            k = min(s.shape)
            out[np.arange(k), np.arange(k)] = 1.0
            return out
        return np.array(s)

    # ---------------------------------------------------------------- kernels
    def gemm(self, o1, o2, cnt, ex):
        if ex["skip"] is not None and self.rank[ex["skip"]] != 0:
            return
        probs = self.arr(o1, _abi.GEMM_PROB, cnt)
        nt = int(max((p["term0"] + p["nterm"] for p in probs), default=0))
        terms = self.arr(o2, _abi.GEMM_TERM, nt)
        for p in probs:
            m, n = self.dim(p["m"], p["m_ri"]), self.dim(p["n"], p["n_ri"])
            if m <= 0 or n <= 0:
                continue
            acc = np.zeros((m, n))
            for t in terms[p["term0"]:p["term0"] + p["nterm"]]:
                k = self.dim(t["k"], t["k_ri"])
                if k <= 0:
                    continue
                a = self.masked(self.mat(t["a"], t["lda"], m, k), t["mask_a"]) if t["ta"] == 0 else \
                    self.masked(self.mat(t["a"], t["lda"], k, m), t["mask_a"]).T
                b = self.masked(self.mat(t["b"], t["ldb"], k, n), t["mask_b"]) if t["tb"] == 0 else \
                    self.masked(self.mat(t["b"], t["ldb"], n, k), t["mask_b"]).T
                acc += t["alpha"] * (a @ b)
            c = self.mat(p["c"], p["ldc"], m, n)
            # K-split launches sum their slices deterministically: same
            # contract as an unsplit product (C = beta C + sum of terms)
            if p["beta"] == 0.0:
                c[:] = acc
            else:
                c[:] = p["beta"] * c + acc

    def zero(self, o1, cnt, ex):
        r = self.arr(o1, np.dtype(np.int64), 2 * cnt)
        for i in range(cnt):
            j = self.idx(r[2 * i])
            self.A[j:j + r[2 * i + 1]] = 0.0

    def concat(self, o1, o2, cnt, ex):
        probs = self.arr(o1, _abi.CONCAT_PROB, cnt)
        npc = int(max((p["piece0"] + p["npiece"] for p in probs), default=0))
        pieces = self.arr(o2, _abi.PIECE, max(npc, 1))
        for p in probs:
            col = 0
            for q in pieces[p["piece0"]:p["piece0"] + p["npiece"]]:
                nc = self.dim(q["cols"], q["cols_ri"])
                src = q["alpha"] * self.mat(q["p"], q["ld"], p["rows"], nc)
                self.mat(p["dst"], p["ldd"], p["rows"], col + nc)[:, col:] = src
                if p["dst2"]:
                    self.mat(p["dst2"], p["ldd2"], p["rows"], col + nc)[:, col:] = src
                col += nc
            if p["ktot_ri"] >= 0:
                self.rank[p["ktot_ri"]] = col

    @staticmethod
    def house(x):
        x0, ss = x[0], float(x[1:] @ x[1:])
        nrm = np.sqrt(x0 * x0 + ss)
        if nrm == 0.0:
            return 0.0, 0.0, 0.0
        sg = -1.0 if x0 < 0 else 1.0
        u1 = x0 + sg * nrm
        return 2.0 / (1.0 + ss / (u1 * u1)), -sg * nrm, 1.0 / u1

    def qr(self, o1, cnt, ex):
        for p in self.arr(o1, _abi.QR_PROB, cnt):
            m, k = self.dim(p["m"], p["m_ri"]), self.dim(p["k"], p["k_ri"])
            r = min(m, k)
            if r <= 0:
                continue
            W = self.mat(p["w"], p["ldw"], m, k)
            tau = self.mat(p["tau"], 1, r, 1)[:, 0]
            Y = np.zeros((m, r))
            for j in range(r):
                g, rho, inv = self.house(W[j:, j].copy())
                y = np.zeros(m - j)
                y[0] = 1.0
                y[1:] = W[j + 1:, j] * inv
                W[j, j] = rho
                W[j + 1:, j] = y[1:]
                tau[j] = g
                Y[j:, j] = y
                if g != 0.0 and j + 1 < k:
                    W[j:, j + 1:] -= g * np.outer(y, y @ W[j:, j + 1:])
            T = np.zeros((r, r))
            for j in range(r):
                T[:j, j] = -tau[j] * (T[:j, :j] @ (Y[:, :j].T @ Y[:, j]))
                T[j, j] = tau[j]
            if p["tpanel"]:
                for q, p0 in enumerate(range(0, r, NB)):
                    pw = min(NB, r - p0)
                    tp = self.mat(p["tpanel"] + 8 * q * NB * NB, NB, NB, NB)
                    tp[:] = 0.0
                    tp[:pw, :pw] = T[p0:p0 + pw, p0:p0 + pw]
            if p["tfull"]:
                self.mat(p["tfull"], p["ldt"], r, r)[:] = T

    def qrcp(self, o1, cnt, ex):
        """hq_qrcp: Businger-Golub pivoted Householder QR without column
        swaps, stopped when (n - j) max ||remaining column||^2 <= stop^2; rows
        0..r-1 keep [R11 R12] P^T, r goes to the rank table."""
        for p in self.arr(o1, _abi.QRCP_PROB, cnt):
            m, n = self.dim(p["m"], p["m_ri"]), self.dim(p["n"], p["n_ri"])
            if m <= 0 or n <= 0:
                self.rank[p["r_ri"]] = 0
                continue
            stop = p["stop_scale"] * (self.scal[p["eps_slot"]] if p["eps_slot"] >= 0 else 1.0)
            C = self.mat(p["c"], p["ldc"], m, n)
            done = np.zeros(n, bool)
            r = min(m, n)
            for j in range(min(m, n)):
                nr = np.sqrt((C[j:] * C[j:]).sum(0))
                nr[done] = -1.0
                c = int(np.argmax(nr))
                if nr[c] <= 0.0 or (n - j) * nr[c] ** 2 <= stop * stop:
                    r = j
                    break
                g, rho, inv = self.house(C[j:, c].copy())
                y = np.concatenate([[1.0], C[j + 1:, c] * inv])
                rest = ~done
                rest[c] = False
                C[j:, rest] -= g * np.outer(y, y @ C[j:, rest])
                C[j, c] = rho
                C[j + 1:, c] = 0.0
                done[c] = True
            self.rank[p["r_ri"]] = r

    def applyq(self, o1, cnt, ex):
        for p in self.arr(o1, _abi.APPLYQ_PROB, cnt):
            m, k = self.dim(p["m"], p["m_ri"]), self.dim(p["k"], p["k_ri"])
            c = self.dim(p["c"], p["c_ri"])
            r = min(m, k)
            if m <= 0 or c <= 0:
                continue
            X = self.mat(p["x"], p["ldx"], m, c)
            if p["x0"]:
                r0 = self.dim(p["r0"], p["r0_ri"])
                new = np.zeros((m, c))
                new[:r0] = self.mat(p["x0"], p["ldx0"], r0, c)
                X[:] = new
            W = self.mat(p["w"], p["ldw"], m, max(r, 1))
            tau = self.mat(p["tau"], 1, max(r, 1), 1)[:, 0]
            order = range(r) if p["trans"] else range(r - 1, -1, -1)
            for j in order:
                y = np.concatenate([[1.0], W[j + 1:, j]])
                X[j:] -= tau[j] * np.outer(y, y @ X[j:])

    def svd(self, o1, cnt, ex):
        for p in self.arr(o1, _abi.SVD_PROB, cnt):
            m, n = self.dim(p["m"], p["m_ri"]), self.dim(p["n"], p["n_ri"])
            thr = p["eps_scale"] * (self.scal[p["eps_slot"]] if p["eps_slot"] >= 0 else 1.0)
            if m <= 0 or n <= 0:
                self.rank[p["rank_ri"]] = 0
                continue
            if p["xform"]:
                n = min(n, m)
                R = self.mat(p["c"], p["ldc"], n, m)
                X = (R if p["xform"] == 2 else np.triu(R)).T
            else:
                X = self.mat(p["c"], p["ldc"], m, n)
            u, s, _ = np.linalg.svd(X, full_matrices=False)
            k = int(np.sum(s > thr))
            if k > p["cap"]:
                if p["flag_ri"] >= 0:
                    self.rank[p["flag_ri"]] = 1
                k = int(p["cap"])
            self.mat(p["u"], p["ldu"], m, k)[:] = u[:, :k]
            self.rank[p["rank_ri"]] = k

    def leaf(self, o1, o2, cnt, scatter):
        probs = self.arr(o1, _abi.LEAF_PROB, cnt)
        ns = int(max((p["slab0"] + p["nslab"] for p in probs), default=0))
        slabs = self.arr(o2, _abi.SLAB, max(ns, 1))
        for p in probs:
            nl = p["nl"]
            leaf = self.mat(p["leaf"], nl, nl, nl)
            row = nl
            rows_total = nl + sum(int(self.rank[s["k_ri"]]) for s in slabs[p["slab0"]:p["slab0"] + p["nslab"]])
            panel = self.mat(p["panel"], p["ldp"], rows_total, nl)
            if scatter:
                leaf[:] = panel[:nl]
            else:
                panel[:nl] = leaf
            for s in slabs[p["slab0"]:p["slab0"] + p["nslab"]]:
                kk = int(self.rank[s["k_ri"]])
                if kk:
                    if scatter:
                        self.mat(s["yv"], s["ldy"], nl, kk)[:] = panel[row:row + kk].T
                    else:
                        panel[row:row + kk] = self.mat(s["v"], s["ld"], nl, kk).T
                row += kk
            if not scatter and p["m_ri"] >= 0:
                self.rank[p["m_ri"]] = row

    def power(self, ex):
        b = self.plan.b
        n, B = b.tree.n, b.B
        for i in range(B):
            done = b.power_done + i
            if self.rank[done]:
                continue
            x = self.mat(self.plan.addr(b.PX) + 8 * 2 * n * i, n, n, 2)
            w = self.mat(self.plan.addr(b.PW) + 8 * 2 * n * i, n, n, 2)
            g = self.mat(self.plan.addr(b.PG) + 8 * 4 * i, 2, 2, 2)
            lam, vec = np.linalg.eigh(0.5 * (g + g.T))
            theta = float(lam[-1])
            est = np.sqrt(max(theta, 0.0))
            v = vec[:, -1]
            fin = est == 0.0 or np.linalg.norm(w @ v - theta * (x @ v)) <= 2 * b.tol * theta \
                or ex["final"]
            if fin:
                self.scal[2 * i], self.scal[2 * i + 1] = est, b.eps * est
                self.rank[done] = 1
                self.rank[b.all_done + 1] += 1
                if self.rank[b.all_done + 1] == B:
                    self.rank[b.all_done] = 1
                continue
            x[:] = np.linalg.qr(np.array(w))[0]
            self.scal[2 * i] = est

    def rowblk(self, o1, cnt, ex):
        for B in self.arr(o1, _abi.ROWBLK_PROB, cnt):
            K = self.dim(B["k"], B["k_ri"])
            ch, rt = int(B["ch"]), int(B["rows_total"])
            nch = -(-rt // ch)
            krf = min(ch, K)
            for c in range(nch):
                off = c * krf
                rows_c = min(ch, rt - c * ch)
                kr = min(rows_c, K)
                if B["mode"] == 0:
                    if kr and K:
                        src = np.triu(np.array(self.mat(B["w"] + 8 * c * ch, B["ldw"], kr, K)))
                        self.mat(B["s"] + 8 * off, B["lds"], kr, K)[:] = src
                    if c == nch - 1:
                        self.rank[B["ms_ri"]] = off + kr
                else:
                    nc = self.dim(B["ncol"], B["ncol_ri"])
                    if nc:
                        blk = np.zeros((rows_c, nc))
                        if kr:
                            blk[:kr] = self.mat(B["s"] + 8 * off, B["lds"], kr, nc)
                        self.mat(B["w"] + 8 * c * ch, B["ldw"], rows_c, nc)[:] = blk

    def pack_copy(self, o1, cnt, ex):
        items = self.arr(o1, _abi.COPY_ITEM, cnt)
        base = ex["base_ptr"]
        off = 0
        for it in items:
            cols = self.dim(it["cols"], it["cols_ri"])
            rows = int(it["rows"])
            if ex["which"] == 1:
                src = self.mat(base + 8 * off, rows, rows, cols)
                dst = self.mat(it["dst"], it["ldd"], rows, cols)
            else:
                src = self.mat(it["src"], it["lds"], rows, cols)
                dst = self.mat(base + 8 * off, rows, rows, cols)
            if rows and cols:
                v = np.array(src)
                if it["mode"] == 1:
                    v = np.triu(v)
                elif it["mode"] == 2:
                    v = np.tril(v, -1)
                    np.fill_diagonal(v, 1.0)
                dst[:] = v
            off += rows * cols
        self.plan.totals.numpy()[ex["total"]] = off

    def copy(self, o1, cnt, ex):
        for it in self.arr(o1, _abi.COPY_ITEM, cnt):
            cols = self.dim(it["cols"], it["cols_ri"])
            rows = int(it["rows"])
            if not rows or not cols:
                continue
            v = np.array(self.mat(it["src"], it["lds"], rows, cols))
            if it["mode"] == 1:
                v = np.triu(v)
            elif it["mode"] == 2:
                v = np.tril(v, -1)
                k = min(rows, cols)
                v[np.arange(k), np.arange(k)] = 1.0
            self.mat(it["dst"], it["ldd"], rows, cols)[:] = v

    def run_interleaved(self, seed):
        """Execute the ops in a random order that respects only the plan's
        lanes (program order within a lane) and cross-lane waits -- what the
        multi-stream graph guarantees.  A missed hazard changes the result."""
        import random
        rnd = random.Random(seed)
        plan = self.plan
        queues = {}
        for i, ln in enumerate(plan.lanes):
            queues.setdefault(ln, []).append(i)
        pos = {ln: 0 for ln in queues}
        done = set()
        launch = plan.launch
        while any(pos[ln] < len(q) for ln, q in queues.items()):
            ready = [ln for ln, q in queues.items()
                     if pos[ln] < len(q) and all(w in done for w in plan.waits[q[pos[ln]]])]
            assert ready, "deadlock in the lane schedule"
            ln = rnd.choice(ready)
            i = queues[ln][pos[ln]]
            pos[ln] += 1
            self.run_ops([launch[i]])
            done.add(i)

    def run(self):
        self.run_ops(self.plan.launch)

    def run_ops(self, ops):
        for kind, o1, o2, cnt, ex in ops:
            if kind == "gemm":
                self.gemm(o1, o2, cnt, ex)
            elif kind == "zero":
                self.zero(o1, cnt, ex)
            elif kind == "concat":
                self.concat(o1, o2, cnt, ex)
            elif kind == "qr":
                self.qr(o1, cnt, ex)
            elif kind == "qrcp":
                self.qrcp(o1, cnt, ex)
            elif kind == "applyq":
                self.applyq(o1, cnt, ex)
            elif kind == "svd":
                self.svd(o1, cnt, ex)
            elif kind == "leaf_gather":
                self.leaf(o1, o2, cnt, False)
            elif kind == "leaf_scatter":
                self.leaf(o1, o2, cnt, True)
            elif kind == "power":
                self.power(ex)
            elif kind == "pack_copy":
                self.pack_copy(o1, cnt, ex)
            elif kind == "copy":
                self.copy(o1, cnt, ex)
            elif kind == "rowblk":
                self.rowblk(o1, cnt, ex)
            else:
                raise ValueError(kind)


def emulate(mats, eps, absolute=False, kcap=512, interleave_seed=None):
    """Run a plan for `mats` through the emulator; return (factors, io, plan)."""
    import torch
    from paper_1809_10585_b200.hqr import PlanIO
    from paper_1809_10585_b200.plan import CompiledPlan
    io = PlanIO(mats[0].tree(), len(mats), eps, absolute, kcap)
    plan = CompiledPlan(io.builder, torch.device("cpu"))
    from paper_1809_10585_b200.plan import R_IN, R_OUT, R_PERSIST
    io.pack(mats)
    A = plan.arena.numpy()
    ib, ob = plan.bases[R_IN], plan.bases[R_OUT]
    A[ib:ib + io.n_in] = io.inbuf[:io.n_in]
    pxo = plan.bases[R_PERSIST] + io.builder.PX.off
    A[pxo:pxo + io.px.size] = io.px
    plan.rank.numpy()[:] = io.rk
    plan.scal.numpy()[:] = io.sc
    if interleave_seed is None:
        Emu(plan).run()
    else:
        Emu(plan).run_interleaved(interleave_seed)
    rk = plan.rank.numpy().copy()
    if rk[io.builder.flag_slot]:
        raise RuntimeError("rank capacity overflow")
    n_out = int(plan.totals.numpy()[1])
    out = A[ob:ob + n_out].copy()
    return [io.factors(b, out, rk) for b in range(len(mats))], io, plan
