#!/bin/bash
# r02av: force -- r^2 by DFMA with an exact redo of row-warps near the cutoff (f1) vs the reference's r^2 form (f0)
mkdir -p gpurun_out
for args in "--cells 128" "--cells 64" "--cells 128 --temperature 3.0 --rebuild 5"; do for rep in 1 2; do for v in f0 f1; do
  PARTICULA_B200_LIB=libparticula_b200_$v.so timeout 300 python bench.py $args --steps 100 --warmup 10 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v $args value %.4g force_us %.1f build_us %.1f' % (d['value'],d['roofline']['avg_launch_us'],d['roofline_build']['avg_launch_us']))"
done; done; done 2>&1 | grep -v "^  \|Traceback\|raise\|json.decoder" | tee gpurun_out/ab_fastr2_r02av.txt
PARTICULA_B200_LIB=libparticula_b200_f1.so timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -3 | tee gpurun_out/pytest_f1_r02av.txt
