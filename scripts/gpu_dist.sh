#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dist.py tests/test_gpu_distmd.py -q -x > gpurun_out/pytest_dist.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_dist.log
tail -30 gpurun_out/pytest_dist.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/bench_torchrun1.log 2>&1
tail -2 gpurun_out/bench_torchrun1.log | cut -c1-300
