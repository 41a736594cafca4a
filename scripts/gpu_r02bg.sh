#!/bin/bash
# r02bg: round-robin order pass with u16 class state and 9 warps per CTA (o1) vs u32 state, 8 warps (o0)
mkdir -p gpurun_out
for args in "--cells 128" "--cells 128 --temperature 3.0 --rebuild 5"; do for rep in 1 2; do for v in o0 o1; do
  PARTICULA_B200_LIB=libparticula_b200_$v.so timeout 300 python bench.py $args --steps 100 --warmup 10 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v $args value %.4g force_us %.1f build+order_us %.1f' % (d['value'],d['roofline']['avg_launch_us'],d['roofline_build']['avg_launch_us']))"
done; done; done 2>&1 | grep -v "^  \|Traceback\|raise\|json.decoder" | tee gpurun_out/ab_order_u16_r02bg.txt
PARTICULA_B200_LIB=libparticula_b200_o1.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -1 | tee gpurun_out/pytest_o1_r02bg.txt
