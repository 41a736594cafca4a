#!/bin/bash
# r02p: force kernel -- packed f32x2 LJ terms (pk) and per-tile mbarrier waits (tb), A/B vs base;
# tile-path parity tests with the default build (both on)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_tile_r02p.txt 2>&1; tail -3 gpurun_out/pytest_tile_r02p.txt
VARIANTS="base pk tb pktb" bash scripts/gpu_ab_force.sh 2>&1 | grep -v "^  \|Traceback\|raise\|json.decoder" > gpurun_out/ab_force_r02p.txt
cat gpurun_out/ab_force_r02p.txt
