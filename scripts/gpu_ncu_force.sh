#!/bin/bash
mkdir -p gpurun_out
T=${1:-t}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tile_force -s 3 -c 1 -o gpurun_out/${T}_force python bench.py --steps 12 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_${T}_force.log 2>&1
