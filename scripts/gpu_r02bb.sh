#!/bin/bash
# r02bb: longest rows vs the build's hit capacity; build warps per CTA 10 (cap 112, default) / 11 (cap 104) / 12 (cap 96)
mkdir -p gpurun_out
timeout 600 python scripts/rounds_probe.py 2>&1 | tee gpurun_out/rounds_probe_r02bb.txt
for args in "--cells 128" "--cells 128 --temperature 3.0 --rebuild 5"; do for rep in 1 2; do for v in b10 b11 b12; do
  PARTICULA_B200_LIB=libparticula_b200_$v.so timeout 300 python bench.py $args --steps 100 --warmup 10 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v $args value %.4g force_us %.1f build+order_us %.1f mode %s' % (d['value'],d['roofline']['avg_launch_us'],d['roofline_build']['avg_launch_us'], d['config'].get('path', d['config'].get('mode'))))"
done; done; done 2>&1 | grep -v "^  \|Traceback\|raise\|json.decoder" | tee gpurun_out/ab_build_warps_r02bb.txt
