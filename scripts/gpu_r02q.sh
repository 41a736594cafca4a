#!/bin/bash
# r02q: tile build v2 (flattened spherical windows, packed tests): tile parity
# tests, A/B vs the r02 build at C3 and the hot config, ncu capture
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_tile_r02q.txt 2>&1; tail -3 gpurun_out/pytest_tile_r02q.txt
ENVS="PC_TILE_BUILD=1 PC_TILE_BUILD=2" ARGS="--cells 128" bash scripts/gpu_ab_env.sh 2>&1 | grep -v "^  \|Traceback\|raise\|json.decoder" | tee gpurun_out/ab_build_r02q.txt
ENVS="PC_TILE_BUILD=1 PC_TILE_BUILD=2" ARGS="--cells 128 --temperature 3.0 --rebuild 5" REPS=1 bash scripts/gpu_ab_env.sh 2>&1 | grep -v "^  \|Traceback\|raise\|json.decoder" | tee -a gpurun_out/ab_build_r02q.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tile_build2 -s 1 -c 1 -o gpurun_out/r02q_build2 python bench.py --steps 25 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_r02q_build2.log 2>&1; ls gpurun_out/r02q_build2*
