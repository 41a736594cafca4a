#!/bin/bash
# r02az: force kernel warps per CTA (one CTA per SM): 24 / 28 / 32 (default) -- registers per thread 85 / 73 / 64
mkdir -p gpurun_out
for args in "--cells 128" "--cells 64"; do for rep in 1 2; do for v in w32 w24 w28; do
  PARTICULA_B200_LIB=libparticula_b200_$v.so timeout 300 python bench.py $args --steps 100 --warmup 10 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v $args value %.4g force_us %.1f' % (d['value'],d['roofline']['avg_launch_us']))"
done; done; done 2>&1 | grep -v "^  \|Traceback\|raise\|json.decoder" | tee gpurun_out/ab_force_warps_r02az.txt
