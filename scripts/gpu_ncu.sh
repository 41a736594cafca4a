#!/bin/bash
# usage: gpu_ncu.sh <kernel regex> <tag> [bench args...]: one full ncu capture of a kernel in a short bench
mkdir -p gpurun_out
K=$1; T=$2; shift 2
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 3 -c 1 -o gpurun_out/$T python bench.py --steps 12 --warmup 3 --no-cpu-baseline --no-e2e "$@" > gpurun_out/ncu_$T.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/ncu_$T.log
