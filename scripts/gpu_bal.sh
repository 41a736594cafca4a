#!/bin/bash
mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -q -x -k "md_ or fabric or tile" > gpurun_out/pytest_bal.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_bal.log
for B in 1 0; do for c in 64 128; do
  PC_TILE_BALANCE=$B timeout 300 python bench.py --cells $c --steps 200 --warmup 10 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('balance=$B cells=$c value',d['value'],'ms/step',d['ms_per_step'],'force_us',d['roofline']['avg_launch_us'])"
done; done
