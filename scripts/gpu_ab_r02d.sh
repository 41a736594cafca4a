#!/bin/bash
# r02d: force-kernel regression A/B (claim-ahead spills) + exact-sum fix check
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_dist.py -m gpu -q -k exact_sum > gpurun_out/pytest_exact_r02d.log 2>&1; tail -2 gpurun_out/pytest_exact_r02d.log
VARIANTS="old9a next1 next0" bash scripts/gpu_ab_force.sh > gpurun_out/ab_force_r02d.txt 2>&1
cat gpurun_out/ab_force_r02d.txt
