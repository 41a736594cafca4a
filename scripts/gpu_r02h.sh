#!/bin/bash
# r02h: Newton-3 accumulation micro-costs; two-rank bench line incl. the N-GPU e2e leg
mkdir -p gpurun_out
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/n3_cost scripts/micro/n3_cost.cu && timeout 120 /tmp/n3_cost > gpurun_out/n3_cost_r02h.txt 2>&1; cat gpurun_out/n3_cost_r02h.txt
timeout 900 python -m pytest tests/test_bench_contract.py -m gpu -q -k "two_rank or device_line" > gpurun_out/pytest_bench_r02h.txt 2>&1; tail -3 gpurun_out/pytest_bench_r02h.txt
PC_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --cells 64 --steps 20 --warmup 3 > gpurun_out/bench2_r02h.log 2>&1; grep '^{' gpurun_out/bench2_r02h.log | cut -c1-400; tail -3 gpurun_out/bench2_r02h.log | cut -c1-300
