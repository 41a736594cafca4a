#!/bin/bash
# r02ab: r02 round-robin order kernel (fast paths, doubled mask) vs r01; order kinds at the hot config
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "order" > gpurun_out/pytest_order_r02ab.txt 2>&1; tail -2 gpurun_out/pytest_order_r02ab.txt
ENVS="PC_TILE_ORDER_IMPL=1 PC_TILE_ORDER_IMPL=2" ARGS="--cells 128" bash scripts/gpu_ab_env.sh 2>&1 | grep -v "^  \|Traceback\|raise\|json.decoder" | tee gpurun_out/ab_order_r02ab.txt
ENVS="PC_TILE_ORDER=0 PC_TILE_ORDER=1" ARGS="--cells 128 --temperature 3.0 --rebuild 5" REPS=1 bash scripts/gpu_ab_env.sh 2>&1 | grep -v "^  \|Traceback\|raise\|json.decoder" | tee -a gpurun_out/ab_order_r02ab.txt
ENVS="PC_TILE_ORDER=0 PC_TILE_ORDER=1" ARGS="--cells 128 --temperature 1.44 --rebuild 5" REPS=1 bash scripts/gpu_ab_env.sh 2>&1 | grep -v "^  \|Traceback\|raise\|json.decoder" | tee -a gpurun_out/ab_order_r02ab.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tile_order -s 1 -c 1 -o gpurun_out/r02ab_order python bench.py --steps 25 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; ls gpurun_out/r02ab_*
