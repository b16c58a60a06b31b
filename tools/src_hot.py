"""Per-CUDA-source-line stall samples from an ncu report (needs -lineinfo + --import-source)."""
import csv, subprocess, sys, io
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
res = []; fname = None; hdr = None
for row in csv.reader(io.StringIO(out)):
    if not row: continue
    if row[0] == "File Path": fname = row[1].split("/")[-1]; continue
    if row[0] == "Line No": hdr = row; continue
    if hdr is None or len(row) < 5 or row[2] != "-": continue
    si = hdr.index("Warp Stall Sampling (All Samples)")
    v = float(row[si] or 0)
    if v > 0:
        stalls = sorted(((float(row[i] or 0), c[6:]) for i, c in enumerate(hdr) if c.startswith("stall_") and "Not Issued" not in c and i < len(row) and row[i] not in ("", "-")), reverse=True)[:2]
        res.append((v, fname, row[0], row[1].strip()[:72], stalls))
tot = sum(r[0] for r in res)
for v, f, ln, src, st in sorted(res, reverse=True)[:top]:
    print("%5.1f%% %s:%s %-72s %s" % (100 * v / tot, f, ln, src, [(int(a), b) for a, b in st]))
