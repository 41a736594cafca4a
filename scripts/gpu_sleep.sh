#!/bin/bash
# A/B of the force kernel's buffer-wait poll interval (rebuilds the library on the box)
mkdir -p gpurun_out
for S in 64 256 1024 4096; do
  make -C paper_2109_09056_b200/csrc -B EXTRA=-DPC_FORCE_SLEEP=$S > gpurun_out/make_s$S.log 2>&1
  timeout 300 python bench.py --steps 300 --warmup 20 --no-cpu-baseline --no-e2e > gpurun_out/bench_sl$S.log 2>&1
  tail -1 gpurun_out/bench_sl$S.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('sleep=$S value',d['value'],'ms/step',d['ms_per_step'],'force_us',d['roofline']['avg_launch_us'])"
done
