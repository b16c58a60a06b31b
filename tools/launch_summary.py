"""Summarise an ncu --csv launch list (gpu__time_duration.sum) by kernel."""
import collections
import csv
import sys


def summarise(path, top=20):
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.reader(lines))
    hdr = rows[0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot, cnt, mx = collections.defaultdict(float), collections.Counter(), collections.defaultdict(float)
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    for r in rows[1:]:
        name = r[ki].split("(")[0].replace("void ", "")
        v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
        tot[name] += v
        cnt[name] += 1
        mx[name] = max(mx[name], v)
    T = sum(tot.values())
    out = [f"{'kernel':44s} {'launches':>8s} {'total ms':>10s} {'share':>7s} {'max ms':>8s}"]
    for k in sorted(tot, key=lambda k: -tot[k])[:top]:
        out.append(f"{k[:44]:44s} {cnt[k]:8d} {tot[k]/1e3:10.3f} {100*tot[k]/T:6.1f}% {mx[k]/1e3:8.3f}")
    out.append(f"{'TOTAL':44s} {sum(cnt.values()):8d} {T/1e3:10.3f}")
    return "\n".join(out)


if __name__ == "__main__":
    print(summarise(sys.argv[1]))
