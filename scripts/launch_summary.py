#!/usr/bin/env python3
"""Per-kernel totals from an `ncu --metrics gpu__time_duration.sum --csv` launch list."""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[h]; ix = {k: j for j, k in enumerate(hdr)}
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[h + 1:]:
    if len(r) < len(hdr) or r[ix["Metric Name"]] != "gpu__time_duration.sum":
        continue
    v = float(r[ix["Metric Value"]].replace(",", ""))
    u = r[ix["Metric Unit"]]
    v = v / 1000 if u in ("nsecond", "ns") else v * 1000 if u in ("msecond", "ms") else v
    k = r[ix["Kernel Name"]].split("(")[0][:60]
    agg[k][0] += 1
    agg[k][1] += v
tot = sum(a[1] for a in agg.values())
print(f"{'kernel':60s} {'n':>5s} {'total_us':>10s} {'avg_us':>9s} share")
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:60s} {n:5d} {t:10.1f} {t / n:9.1f} {t / tot:.3f}")
