#!/bin/bash
mkdir -p gpurun_out
T=${1:-t}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tile_build -s 0 -c 1 -o gpurun_out/${T}_build python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_${T}_build.log 2>&1
