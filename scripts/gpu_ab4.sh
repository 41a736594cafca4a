#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "md_ or tile" > gpurun_out/pytest_ab4.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_ab4.log
for cfg in "3 1" "3 2"; do
  set -- $cfg
  export PC_TILE_SCHED=$1 PC_TILE_ORDER=$2
  tag=s$1o$2
  timeout 300 python bench.py --steps 300 --warmup 20 --no-cpu-baseline --no-e2e > gpurun_out/bench_$tag.log 2>&1
  tail -1 gpurun_out/bench_$tag.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('$tag value',d['value'],'ms/step',d['ms_per_step'],'force_us',d['roofline']['avg_launch_us'])"
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_$tag.csv python bench.py --steps 25 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
  python3 scripts/launch_summary.py gpurun_out/launches_$tag.csv 2>/dev/null | grep -E "force|build|order"
done
