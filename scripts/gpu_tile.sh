#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "md_" > gpurun_out/pytest_tile.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_tile.log; tail -25 gpurun_out/pytest_tile.log
for p in tile sell; do
timeout 300 python bench.py --steps 400 --warmup 20 --no-cpu-baseline --no-e2e --path $p > gpurun_out/bench_$p.log 2>&1
python - <<PY
import json
d=json.loads(open("gpurun_out/bench_$p.log").read().strip().splitlines()[-1])
print("$p", d["value"], d["ms_per_step"], d["roofline"]["avg_launch_us"], d["roofline"]["frac"], d["check"])
PY
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tile_ -s 2 -c 2 -o gpurun_out/tile python bench.py --steps 25 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/ncu_tile.log 2>&1
ls gpurun_out | head -30
