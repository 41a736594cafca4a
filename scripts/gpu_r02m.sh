#!/bin/bash
# r02m: round order kind in the hot configuration (rebuild 5) and at rebuild 10/20
mkdir -p gpurun_out
for rb in 5 10; do for k in 0 1 2; do
T=$([ $rb = 5 ] && echo 3.0 || echo 1.44)
PC_TILE_ORDER=$k timeout 600 python bench.py --temperature $T --rebuild $rb --steps 200 --warmup 10 --no-cpu-baseline --no-e2e 2>&1 | grep '^{' | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('rebuild $rb T $T order $k value %.4g ms/step %.4f force_us %.1f build+order_us %.1f' % (d['value'], d['ms_per_step'], d['roofline']['avg_launch_us'], d['roofline_build']['avg_launch_us']))"
done; done 2>&1 | tee gpurun_out/order_kinds_r02m.txt
