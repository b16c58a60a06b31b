"""Summarise an ncu report's SASS source page: stall mix + hottest lines."""
import csv, subprocess, sys
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
for hi, r in enumerate(rows):
    if "Source" in r and len(r) > 5: break
h = rows[hi]; data = rows[hi + 1:]
si = h.index("Warp Stall Sampling (All Samples)"); src = h.index("Source")
cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
tot = sum(float(r[si] or 0) for r in data)
agg = {c: sum(float(r[h.index(c)] or 0) for r in data) for c in cols}
print("samples", tot, {k[6:]: round(100 * v / tot, 1) for k, v in sorted(agg.items(), key=lambda x: -x[1])[:9]})
for i, r in enumerate(data):
    v = float(r[si] or 0)
    if v >= tot / top / 2:
        tops = sorted(((float(r[h.index(c)] or 0), c[6:]) for c in cols), reverse=True)[:2]
        print("%5d %5.1f%% %-60s %s" % (i, 100 * v / tot, r[src][:60], tops))
