#!/bin/bash
# r02al: after stripping the measured-off A/B code paths -- tile/dist parity and a C3 bench
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py tests/test_gpu_dist.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_r02al.txt 2>&1; tail -2 gpurun_out/pytest_r02al.txt
for rep in 1 2; do timeout 300 python bench.py --steps 100 --warmup 10 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3 value %.4g force_us %.1f build_us %.1f' % (d['value'], d['roofline']['avg_launch_us'], d['roofline_build']['avg_launch_us']))"; done | tee gpurun_out/bench_r02al.txt
