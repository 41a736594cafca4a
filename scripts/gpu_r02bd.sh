#!/bin/bash
# r02bd: force -- rows accumulate u/2 and fm/2 (h1: one FADD2 with an immediate, no materialised 2.0; bit-identical) vs the r02 form (h0)
mkdir -p gpurun_out
for args in "--cells 128" "--cells 64" "--cells 128 --temperature 3.0 --rebuild 5"; do for rep in 1 2; do for v in h0 h1; do
  PARTICULA_B200_LIB=libparticula_b200_$v.so timeout 300 python bench.py $args --steps 100 --warmup 10 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v $args value %.4g force_us %.1f E %r' % (d['value'],d['roofline']['avg_launch_us'], d.get('check')))"
done; done; done 2>&1 | grep -v "^  \|Traceback\|raise\|json.decoder" | tee gpurun_out/ab_halfu_r02bd.txt
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2 | tee gpurun_out/pytest_h1_r02bd.txt
