#!/bin/bash
# r02aa: round-robin order fused into the build (pc_tile_build_ordered) vs the separate pass
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py tests/test_gpu_dist.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_tile_r02aa.txt 2>&1; tail -2 gpurun_out/pytest_tile_r02aa.txt
ENVS="PC_TILE_FUSED=0 PC_TILE_FUSED=1" ARGS="--cells 128" bash scripts/gpu_ab_env.sh 2>&1 | grep -v "^  \|Traceback\|raise\|json.decoder" | tee gpurun_out/ab_fused_r02aa.txt
ENVS="PC_TILE_FUSED=0 PC_TILE_FUSED=1" ARGS="--cells 64" bash scripts/gpu_ab_env.sh 2>&1 | grep -v "^  \|Traceback\|raise\|json.decoder" | tee -a gpurun_out/ab_fused_r02aa.txt
ENVS="PC_TILE_ORDER=0 PC_TILE_ORDER=1" ARGS="--cells 128 --temperature 3.0 --rebuild 5" REPS=1 bash scripts/gpu_ab_env.sh 2>&1 | grep -v "^  \|Traceback\|raise\|json.decoder" | tee -a gpurun_out/ab_fused_r02aa.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tile_build -s 1 -c 1 -o gpurun_out/r02aa_build python bench.py --steps 25 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; ls gpurun_out/r02aa_*
