"""Per-CUDA-source-line executed instructions and stall samples from an ncu
mixed source export:
  ncu -i REP --page source --csv --print-source cuda,sass > src.csv
  python scripts/ncu_lines.py src.csv [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
fname, recs = "?", []
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) < 9 or not r[0] or not r[0].isdigit():
        continue
    try:
        samp, ex = int(r[4]), int(r[7])
    except ValueError:
        continue
    recs.append((fname, int(r[0]), r[1].strip(), samp, ex))
ts = sum(x[3] for x in recs) or 1
te = sum(x[4] for x in recs) or 1
print(f"executed warp instructions {te}, stall samples {ts}")
print(" exec%  samp%  file:line  source")
for f, ln, src, s, e in sorted(recs, key=lambda x: -x[4])[:top]:
    print(f"{100*e/te:6.2f} {100*s/ts:6.2f}  {f}:{ln}  {src[:90]}")
