#!/bin/bash
mkdir -p gpurun_out
PC_TILE_ORDER=3 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -q -x -k "md_ or tile or fabric" 2>&1 | tail -1
for rep in 1 2; do for o in 1 3; do
  PC_TILE_ORDER=$o timeout 300 python bench.py --steps 300 --warmup 20 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('order=$o value',d['value'],'ms/step',d['ms_per_step'],'force_us',d['roofline']['avg_launch_us'])"
done; done
for o in 1 3; do PC_TILE_ORDER=$o timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:tile_order -c 3 --csv python bench.py --steps 45 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | grep tile_order | awk -F'","' '{print "order='$o'", $NF}' | tr -d '"'; done
