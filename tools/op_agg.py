"""Aggregate tools/op_times.py output: by (kind, role), by lane, by level."""
import collections, sys
rows = [l.rstrip('\n').split('\t') for l in open(sys.argv[1] if len(sys.argv) > 1 else 'gpurun_out/op_times_b57.tsv')]
agg = collections.defaultdict(lambda: [0.0, 0]); lk = collections.defaultdict(float); lev = collections.defaultdict(float)
for i, ms, kind, key, ln, lv, npb, sh in rows:
    ms = float(ms); agg[(kind, key)][0] += ms; agg[(kind, key)][1] += 1; lk[(ln, kind)] += ms; lev[(kind, lv)] += ms
print("total %.1f" % sum(v[0] for v in agg.values()))
for k, v in sorted(agg.items(), key=lambda x: -x[1][0])[:20]:
    print(k, "%.1f ms" % v[0], v[1], "avg %.3f" % (v[0] / v[1]))
lanes = collections.defaultdict(float)
for (ln, kind), v in lk.items(): lanes[ln] += v
print({k: round(v, 1) for k, v in sorted(lanes.items())})
for k, v in sorted(lk.items()):
    if v > 5: print(k, "%.1f" % v)
print("by level:", {k: round(v, 1) for k, v in sorted(lev.items()) if v > 8})
top = sorted(rows, key=lambda r: -float(r[1]))[:int(sys.argv[2]) if len(sys.argv) > 2 else 30]
for r in top: print(r)
