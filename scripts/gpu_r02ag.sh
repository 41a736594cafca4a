#!/bin/bash
# r02ag: after removing the build variants -- tile/dist parity, C2 end-to-end repeat
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py tests/test_gpu_dist.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_r02ag.txt 2>&1; tail -2 gpurun_out/pytest_r02ag.txt
for rep in 1 2 3; do timeout 300 python bench.py --cells 64 --no-cpu-baseline 2>&1 | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('c2 value %.4g e2e %.4g' % (d['value'], d['e2e']['value']))"; done | tee gpurun_out/c2_e2e_r02ag.txt
