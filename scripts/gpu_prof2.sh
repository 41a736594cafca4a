#!/bin/bash
mkdir -p gpurun_out
for g in planar pos4; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:lj_force_sell \
   -s 10 -c 1 -o gpurun_out/force_$g python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --gather $g > gpurun_out/ncu_force_$g.log 2>&1
done
ls gpurun_out
