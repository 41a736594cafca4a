#!/bin/bash
# r02aw: round evidence at HEAD (smoke, GPU tests, default bench, reference arm, launch list,
# ncu captures) plus the C2 and hot-configuration bench lines and a driver-style 20-step run
mkdir -p gpurun_out
bash scripts/gpu_full.sh r02aw
timeout 600 python bench.py --cells 64 > gpurun_out/bench_c2_r02aw.log 2>&1
timeout 900 python bench.py --temperature 3.0 --rebuild 5 > gpurun_out/bench_hot_r02aw.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_drv_r02aw.log 2>&1
for f in gpurun_out/bench_c2_r02aw.log gpurun_out/bench_hot_r02aw.log gpurun_out/bench_drv_r02aw.log; do tail -1 $f | cut -c1-300; done
