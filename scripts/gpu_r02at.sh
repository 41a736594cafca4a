#!/bin/bash
# r02at: build -- candidate test as the sign of |d|^2 - hi2 with LEA.HI hit counts and a min-|r| band check (s1) vs FSETP/SEL + max band (s0)
mkdir -p gpurun_out
PARTICULA_B200_LIB=libparticula_b200_s0.so timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k search_radius 2>&1 | tail -1
PARTICULA_B200_LIB=libparticula_b200_s1.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_s1_r02at.txt 2>&1; tail -2 gpurun_out/pytest_s1_r02at.txt
for args in "--cells 128" "--cells 128 --temperature 3.0 --rebuild 5"; do for rep in 1 2; do for v in s0 s1; do
  PARTICULA_B200_LIB=libparticula_b200_$v.so timeout 300 python bench.py $args --steps 100 --warmup 10 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v $args value %.4g force_us %.1f build_us %.1f' % (d['value'],d['roofline']['avg_launch_us'],d['roofline_build']['avg_launch_us']))"
done; done; done 2>&1 | grep -v "^  \|Traceback\|raise\|json.decoder" | tee gpurun_out/ab_s_r02at.txt
