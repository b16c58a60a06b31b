"""Fill the FINAL_* placeholders of DESIGN.md / profiles/README.md from a bench line.
usage: python tools/fill_docs.py profiles/r02_bench_config2_with_cpu.json"""
import json, re, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
k, r = d["kernel_time_by_kind"], d["roofline_by_kind"]
rep = {"FINAL_VALUE": "%.1f" % d["value"], "FINAL_MS": "%.0f" % d["ms_per_step"], "FINAL_E2E": "%.1f" % d["e2e"]["value"],
       "FINAL_LAT": "%.0f" % d["latency_ms_single_matrix"], "FINAL_API": "%.0f" % d["latency_ms_single_matrix_api"],
       "FINAL_RERR": "%.2e" % d["r_sketch_rel_err_matrix0"]}
for name in ("qr", "svd", "gemm", "qrcp", "gemv", "applyq", "concat", "pack_copy"):
    rep["FINAL_%s_ach" % name] = ("%.0f" if r[name]["unit"] == "GB/s" else "%.2f") % r[name]["achieved"]
    rep["FINAL_%s_frac" % name] = "%.1f %%" % (100 * r[name]["frac"])
    rep["FINAL_%s" % name] = "%.0f" % k[name]["ms"]
for path in ("DESIGN.md", "profiles/README.md"):
    s = open(path).read()
    for key in sorted(rep, key=len, reverse=True):
        s = re.sub(key + r"(?![A-Za-z_])", rep[key], s)
    open(path, "w").write(s)
print(rep)
