#!/bin/bash
# r02x: force loader L2-prefetch of the staged tile's row-warp list heads (hp1: one group, hp2: two) vs none (hp0)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_tile_r02x.txt 2>&1; tail -2 gpurun_out/pytest_tile_r02x.txt
VARIANTS="hp0 hp1 hp2" bash scripts/gpu_ab_force.sh 2>&1 | grep -v "^  \|Traceback\|raise\|json.decoder" | tee gpurun_out/ab_force_r02x.txt
