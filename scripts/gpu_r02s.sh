#!/bin/bash
# r02s: tile build variants (1: r02 build, 2: flat spherical windows, 3: column-lockstep
# spherical windows, planar FP32 + packed tests): tile parity with the default (3),
# A/B at C3 and the hot config, ncu of the variant-3 build
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_tile_r02s.txt 2>&1; tail -2 gpurun_out/pytest_tile_r02s.txt
ENVS="PC_TILE_BUILD=1 PC_TILE_BUILD=2 PC_TILE_BUILD=3" ARGS="--cells 128" bash scripts/gpu_ab_env.sh 2>&1 | grep -v "^  \|Traceback\|raise\|json.decoder" | tee gpurun_out/ab_build_r02s.txt
ENVS="PC_TILE_BUILD=1 PC_TILE_BUILD=2 PC_TILE_BUILD=3" ARGS="--cells 128 --temperature 3.0 --rebuild 5" REPS=1 bash scripts/gpu_ab_env.sh 2>&1 | grep -v "^  \|Traceback\|raise\|json.decoder" | tee -a gpurun_out/ab_build_r02s.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tile_build2 -s 1 -c 1 -o gpurun_out/r02s_build_s python bench.py --steps 25 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_r02s_build_s.log 2>&1; ls gpurun_out/r02s_build_s*
