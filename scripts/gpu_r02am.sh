#!/bin/bash
# r02am: persistent round-order kernel with an L2 prefetch of each warp's next row-warp list
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "order or md_engine" > gpurun_out/pytest_r02am.txt 2>&1; tail -2 gpurun_out/pytest_r02am.txt
for args in "--cells 128" "--cells 128 --temperature 3.0 --rebuild 5"; do for rep in 1 2; do
  timeout 300 python bench.py $args --steps 100 --warmup 10 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); rb=d['roofline_build']; print('$args value %.4g force_us %.1f build+order_us %.1f build_issue_frac %.3f' % (d['value'], d['roofline']['avg_launch_us'], rb['avg_launch_us'], rb.get('issue',{}).get('frac',0)))"
done; done | tee gpurun_out/bench_r02am.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:tile_order -c 3 --csv python bench.py --steps 25 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | grep tile_order | tail -3
