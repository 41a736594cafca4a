#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "md_ or neighbor" > gpurun_out/pytest_quick.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_quick.log; tail -3 gpurun_out/pytest_quick.log
timeout 300 python bench.py --steps 400 --warmup 20 --no-cpu-baseline --no-e2e > gpurun_out/bench_q.log 2>&1
python - <<PY
import json
d=json.loads(open("gpurun_out/bench_q.log").read().strip().splitlines()[-1])
print(d["value"], d["ms_per_step"], d["roofline"]["avg_launch_us"], d["roofline"]["frac"])
PY
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches_q.csv python bench.py --steps 25 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python3 scripts/launch_summary.py gpurun_out/launches_q.csv | head -12
