#!/bin/bash
# ncu: launch list of a short bench + full capture of the force and build kernels.
mkdir -p gpurun_out
B="python bench.py --steps 40 --warmup 5 --no-cpu-baseline --no-e2e"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
   --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_list.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:lj_force_sell \
   -s 10 -c 1 -o gpurun_out/force $B > gpurun_out/ncu_force.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:nbr_build_staged \
   -s 1 -c 1 -o gpurun_out/build $B > gpurun_out/ncu_build.log 2>&1
ls gpurun_out
