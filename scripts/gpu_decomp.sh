#!/bin/bash
mkdir -p gpurun_out
./scripts/micro/pipes > gpurun_out/pipes.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_decomp.py -q > gpurun_out/pytest_decomp.log 2>&1
cat gpurun_out/pipes.txt; tail -15 gpurun_out/pytest_decomp.log
