#!/bin/bash
# r02au: force -- next list group prefetched into L1 (distance 2 / 3, the group load allowed to hit L1) vs L2 prefetch only (l0)
mkdir -p gpurun_out
for args in "--cells 128" "--cells 64"; do for rep in 1 2; do for v in l0 l2 l3; do
  PARTICULA_B200_LIB=libparticula_b200_$v.so timeout 300 python bench.py $args --steps 100 --warmup 10 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v $args value %.4g force_us %.1f build_us %.1f' % (d['value'],d['roofline']['avg_launch_us'],d['roofline_build']['avg_launch_us']))"
done; done; done 2>&1 | grep -v "^  \|Traceback\|raise\|json.decoder" | tee gpurun_out/ab_l1pf_r02au.txt
PARTICULA_B200_LIB=libparticula_b200_l2.so timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "engine or tile" 2>&1 | tail -1
