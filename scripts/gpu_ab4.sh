#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "md_" > gpurun_out/pytest_ab4.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_ab4.log
for v in 0 3; do
  export PC_TILE_SCHED=$v
  timeout 300 python bench.py --steps 300 --warmup 20 --no-cpu-baseline --no-e2e > gpurun_out/bench_s$v.log 2>&1
  tail -1 gpurun_out/bench_s$v.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('sched=$v value',d['value'],'ms/step',d['ms_per_step'],'force_us',d['roofline']['avg_launch_us'])"
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_s$v.csv python bench.py --steps 25 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
  python3 scripts/launch_summary.py gpurun_out/launches_s$v.csv 2>/dev/null | head -3 | tail -2
done
unset PC_TILE_SCHED
bash scripts/gpu_ncu2.sh rr > /dev/null 2>&1; ls gpurun_out/rr_*
