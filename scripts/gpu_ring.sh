#!/bin/bash
mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -q -x > gpurun_out/pytest_ring.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_ring.log
timeout 300 python bench.py --steps 300 --warmup 20 --no-cpu-baseline --no-e2e > gpurun_out/bench_ring.log 2>&1
tail -1 gpurun_out/bench_ring.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('value',d['value'],'ms/step',d['ms_per_step'],'force_us',d['roofline']['avg_launch_us'])"
