#!/bin/bash
mkdir -p gpurun_out
for v in sched nosched; do
  if [ $v == sched ]; then export PC_TILE_SCHED=1; else unset PC_TILE_SCHED; fi
  timeout 300 python bench.py --steps 300 --warmup 20 --no-cpu-baseline --no-e2e > gpurun_out/bench_$v.log 2>&1
  tail -1 gpurun_out/bench_$v.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v value',d['value'],'ms/step',d['ms_per_step'],'force_us',d['roofline']['avg_launch_us'])"
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_$v.csv python bench.py --steps 25 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
  python3 scripts/launch_summary.py gpurun_out/launches_$v.csv 2>/dev/null | head -4
done
