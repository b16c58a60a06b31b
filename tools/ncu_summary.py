"""Summarise an ncu --set full report: key SOL / occupancy / stall metrics,
per-launch DRAM traffic, and the stall mix of the SASS source page."""
import csv, subprocess, sys


SEL = ()   # import filter: one result of a multi-kernel report
SEL_INDEX = 0


def page(rep, name, extra=()):
    out = subprocess.run(["ncu", "-i", rep, "--page", name, "--csv", *SEL, *extra], capture_output=True, text=True).stdout
    return list(csv.reader(out.splitlines()))


def count(rep):
    rows = page(rep, "details")
    if not rows or "ID" not in rows[0]:
        return 0
    return len({r[rows[0].index("ID")] for r in rows[1:] if r})


def summary(rep):
    rows = page(rep, "details")
    h = rows[0]
    si, mi, vi, ui = (h.index(k) for k in ("Section Name", "Metric Name", "Metric Value", "Metric Unit"))
    want = ["Duration", "Elapsed Cycles", "SM Active Cycles", "Executed Ipc Active", "Issue Slots Busy",
            "DRAM Throughput", "L1/TEX Hit Rate", "L2 Hit Rate", "Warp Cycles Per Issued Instruction",
            "Registers Per Thread", "Grid Size", "Block Size", "Cluster Size", "Achieved Occupancy",
            "Dynamic Shared Memory Per Block", "Compute (SM) Throughput", "Memory Throughput"]
    out = ["kernel: " + rows[1][h.index("Kernel Name")]]
    seen = set()
    for r in rows[1:]:
        if r[mi] in want and (r[si], r[mi]) not in seen:
            seen.add((r[si], r[mi]))
            out.append(f"  {r[si][:30]:30s} {r[mi]:38s} {r[vi]:>14s} {r[ui]}")
    raw = page(rep, "raw")
    rh = raw[0]
    row = raw[2] if len(raw) > 2 else raw[1]
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
              "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
              "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
              "sm__pipe_tensor_op_dmma_cycles_active.avg.pct_of_peak_sustained_active"):
        if k in rh:
            out.append(f"  {k:70s} {row[rh.index(k)]} {raw[1][rh.index(k)]}")
    src = page(rep, "source", ("--print-source", "sass"))
    # a multi-kernel report prints one section per kernel, each with its own
    # header row: take the section of the selected result
    heads = [i for i, r in enumerate(src) if "Source" in r and len(r) > 5]
    if not heads:
        return "\n".join(out)
    which = min(SEL_INDEX, len(heads) - 1) if len(heads) > 1 else 0
    hi = heads[which]
    sh = src[hi]
    data = [r for r in src[hi + 1:(heads[which + 1] if which + 1 < len(heads) else len(src))] if len(r) == len(sh)]
    if "Warp Stall Sampling (All Samples)" in sh:
        si2 = sh.index("Warp Stall Sampling (All Samples)")
        cols = [c for c in sh if c.startswith("stall_") and "Not Issued" not in c]
        def num(x):
            try:
                return float(x or 0)
            except ValueError:
                return 0.0
        tot = sum(num(r[si2]) for r in data) or 1.0
        agg = {c: sum(num(r[sh.index(c)]) for r in data) for c in cols}
        out.append("  stall mix (% of samples): " + ", ".join(
            f"{k[6:]} {100 * v / tot:.1f}" for k, v in sorted(agg.items(), key=lambda x: -x[1])[:8]))
    return "\n".join(out)


if __name__ == "__main__":
    for rep in sys.argv[1:]:
        n = count(rep)
        for i in range(max(n, 1)):
            SEL = ("--launch-skip", str(i), "--launch-count", "1") if n > 1 else ()
            SEL_INDEX = i
            try:
                print(summary(rep))
            except Exception as e:   # noqa: BLE001
                print("summary failed for result", i, repr(e))
            print()
