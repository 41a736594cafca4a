#!/bin/bash
mkdir -p gpurun_out
for g in planar pos4; do
  timeout 300 python bench.py --steps 400 --warmup 20 --no-cpu-baseline --no-e2e --gather $g > gpurun_out/bench_$g.log 2>&1
  python - <<PY
import json
d=json.loads(open("gpurun_out/bench_$g.log").read().strip().splitlines()[-1])
print("$g", d["value"], d["ms_per_step"], d["roofline"]["avg_launch_us"], d["roofline"]["frac"])
PY
done
timeout 300 python -m pytest tests -m gpu -q -x -k "md_" > gpurun_out/pytest_md.log 2>&1; tail -2 gpurun_out/pytest_md.log
