#!/bin/bash
# r02bf: force -- item -> tile by a forward scan from the warp's last tile (q1) vs bisection over the CTA's tiles (q0)
mkdir -p gpurun_out
for args in "--cells 128" "--cells 64" "--cells 128 --temperature 3.0 --rebuild 5"; do for rep in 1 2; do for v in q0 q1; do
  PARTICULA_B200_LIB=libparticula_b200_$v.so timeout 300 python bench.py $args --steps 100 --warmup 10 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v $args value %.4g force_us %.1f' % (d['value'],d['roofline']['avg_launch_us']))"
done; done; done 2>&1 | grep -v "^  \|Traceback\|raise\|json.decoder" | tee gpurun_out/ab_locate_r02bf.txt
PARTICULA_B200_LIB=libparticula_b200_q1.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -1 | tee gpurun_out/pytest_q1_r02bf.txt
