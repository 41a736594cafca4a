#!/bin/bash
# tile path: parity subset + bench + launch list
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "md_" > gpurun_out/pytest_tile.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_tile.log; tail -25 gpurun_out/pytest_tile.log
timeout 300 python bench.py --steps 400 --warmup 20 --no-cpu-baseline --no-e2e > gpurun_out/bench_tile.log 2>&1
tail -3 gpurun_out/bench_tile.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches_tile.csv python bench.py --steps 25 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python3 scripts/launch_summary.py gpurun_out/launches_tile.csv | head -12
