#!/bin/bash
# A/B of the force kernel's warps per CTA (rebuilds the library on the box)
mkdir -p gpurun_out
for W in 32 24 16; do
  make -C paper_2109_09056_b200/csrc -B EXTRA=-DPC_FORCE_WARPS=$W > gpurun_out/make_$W.log 2>&1
  timeout 300 python bench.py --steps 300 --warmup 20 --no-cpu-baseline --no-e2e > gpurun_out/bench_w$W.log 2>&1
  tail -1 gpurun_out/bench_w$W.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('W=$W value',d['value'],'ms/step',d['ms_per_step'],'force_us',d['roofline']['avg_launch_us'])"
done
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "md_ or tile" 2>&1 | tail -1
