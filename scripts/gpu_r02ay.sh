#!/bin/bash
# r02ay: round order at rebuild 5 / 10 / 20: residue round-robin (kind 1, default) vs class-major lane-rotated (kind 2)
mkdir -p gpurun_out
for args in "--temperature 3.0 --rebuild 5" "--rebuild 10" "--rebuild 20"; do for rep in 1 2; do for k in 1 2; do
  PC_TILE_ORDER=$k timeout 300 python bench.py $args --steps 100 --warmup 10 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('kind $k $args value %.4g force_us %.1f build+order_us %.1f rebuild_us %.1f' % (d['value'],d['roofline']['avg_launch_us'],d['roofline_build']['avg_launch_us'],d['roofline_build']['rebuild_us']))"
done; done; done 2>&1 | grep -v "^  \|Traceback\|raise\|json.decoder" | tee gpurun_out/ab_order_kind_r02ay.txt
