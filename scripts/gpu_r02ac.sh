#!/bin/bash
# r02ac: order pass with two list groups in flight in its count pass; order kind 1 from rebuild 5
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "order" > gpurun_out/pytest_order_r02ac.txt 2>&1; tail -2 gpurun_out/pytest_order_r02ac.txt
ENVS="PC_TILE_ORDER_IMPL=2" ARGS="--cells 128" bash scripts/gpu_ab_env.sh 2>&1 | grep -v "^  \|Traceback\|raise\|json.decoder" | tee gpurun_out/ab_order_r02ac.txt
ENVS="PC_TILE_ORDER_IMPL=2" ARGS="--cells 128 --temperature 3.0 --rebuild 5" REPS=1 bash scripts/gpu_ab_env.sh 2>&1 | grep -v "^  \|Traceback\|raise\|json.decoder" | tee -a gpurun_out/ab_order_r02ac.txt
