#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "half or md_" > gpurun_out/pytest_half.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_half.log; tail -4 gpurun_out/pytest_half.log
for l in full half; do
timeout 300 python bench.py --steps 400 --warmup 20 --no-cpu-baseline --no-e2e --list $l > gpurun_out/bench_$l.log 2>&1
python - <<PY
import json
d=json.loads(open("gpurun_out/bench_$l.log").read().strip().splitlines()[-1])
print("$l", d["value"], d["ms_per_step"], d["roofline"]["avg_launch_us"], d["roofline"]["frac"], d["config"]["mean_neighbors"])
PY
done
