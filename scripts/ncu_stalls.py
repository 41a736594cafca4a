"""Per-instruction stall attribution from an ncu source-page CSV export:
  ncu -i REP --page source --csv --print-source sass > src.csv
  python scripts/ncu_stalls.py src.csv [top]
Prints the instructions with the most stall samples and, per opcode class,
the executed-instruction and sample shares."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
recs = []
for r in rows[2:]:
    if len(r) != len(hdr):
        continue
    samp = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    ex = int(r[ix["Instructions Executed"]] or 0)
    st = {h: int(r[ix[h]] or 0) for h in stall_cols}
    recs.append((r[ix["Address"]], r[ix["Source"]].strip(), samp, ex, st))
tot_s = sum(x[2] for x in recs) or 1
tot_e = sum(x[3] for x in recs) or 1
print(f"total samples {tot_s}, executed warp instructions {tot_e}")
agg = defaultdict(lambda: [0, 0])
for a, src, s, e, st in recs:
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    op = op.split(".")[0]
    agg[op][0] += s
    agg[op][1] += e
print("opcode      samples%  executed%")
for op, (s, e) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:25]:
    print(f"{op:10s} {100*s/tot_s:8.2f} {100*e/tot_e:9.2f}")
print("\ntop instructions by stall samples")
for a, src, s, e, st in sorted(recs, key=lambda x: -x[2])[:top]:
    why = sorted(st.items(), key=lambda kv: -kv[1])[:3]
    print(f"{a[-5:]} {100*s/tot_s:5.2f}% ex={e:10d}  {src[:60]:60s} " +
          " ".join(f"{k[6:]}={v}" for k, v in why if v))
