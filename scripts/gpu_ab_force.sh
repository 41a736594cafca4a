#!/bin/bash
# same-box A/B of force-kernel variants at C3 (and C2), interleaved twice
mkdir -p gpurun_out
V=${VARIANTS:-"novir nopf pf"}
for cells in 128 64; do for rep in 1 2; do for v in $V; do
  PARTICULA_B200_LIB=libparticula_b200_$v.so timeout 300 python bench.py --cells $cells --steps 200 --warmup 20 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('cells $cells $v value %.4g ms/step %.4f force_us %.1f build_us %.1f' % (d['value'],d['ms_per_step'],d['roofline']['avg_launch_us'],d['roofline_build']['avg_launch_us']))"
done; done; done
