#!/bin/bash
# r02f: force-kernel item-ahead L2 prefetch (AHEAD 0/1/2) + order-kernel list prefetch (ahead0 has both off)
mkdir -p gpurun_out
VARIANTS="ahead0 ahead1 ahead2" bash scripts/gpu_ab_force.sh 2>&1 | grep -v "^  \|Traceback\|raise\|json.decoder" > gpurun_out/ab_force_r02f.txt
cat gpurun_out/ab_force_r02f.txt
