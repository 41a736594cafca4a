#!/bin/bash
mkdir -p gpurun_out
for w in single 1x1x1 2x2x2; do
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,smsp__inst_executed.sum --csv --log-file gpurun_out/dvs_$w.csv python scripts/domain_vs_single.py 64 $w > gpurun_out/dvs_$w.log 2>&1
echo "== $w"; cat gpurun_out/dvs_$w.log | tail -1
python3 - gpurun_out/dvs_$w.csv <<'PY'
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[0]; ix = {h: i for i, h in enumerate(hdr)}
agg = {}
for r in rows[1:]:
    if len(r) != len(hdr) or not r[ix["Metric Value"]].replace('.', '', 1).replace(',', '').isdigit():
        continue
    k = (r[ix["Kernel Name"]][:40], r[ix["Metric Name"]])
    agg.setdefault(k, []).append(float(r[ix["Metric Value"]].replace(',', '')))
for (k, m), v in sorted(agg.items()):
    if any(t in k for t in ("tile_build", "tile_order", "tile_force", "tile_rows")):
        print(f"{k:42s} {m:28s} n={len(v)} sum={sum(v):.4g}")
PY
done
