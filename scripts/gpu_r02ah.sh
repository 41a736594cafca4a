#!/bin/bash
# r02ah: warp-uniform minimum-image axis flags (miu) vs per-lane (fl1); parity with miu
mkdir -p gpurun_out
PARTICULA_B200_LIB=libparticula_b200_miu.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_miu_r02ah.txt 2>&1; tail -2 gpurun_out/pytest_miu_r02ah.txt
VARIANTS="fl1 miu" bash scripts/gpu_ab_force.sh 2>&1 | grep -v "^  \|Traceback\|raise\|json.decoder" | tee gpurun_out/ab_force_miu.txt
