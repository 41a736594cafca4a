#!/bin/bash
# same-box A/B of library builds (PARTICULA_B200_LIB), interleaved twice
mkdir -p gpurun_out
for rep in 1 2; do for v in old nov; do
  PARTICULA_B200_LIB=libparticula_b200_$v.so timeout 300 python bench.py --steps 300 --warmup 20 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v value',d['value'],'ms/step',d['ms_per_step'],'force_us',d['roofline']['avg_launch_us'])"
done; done
