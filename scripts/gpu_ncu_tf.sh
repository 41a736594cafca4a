#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tile_force -s 3 -c 1 -o gpurun_out/tforce python bench.py --steps 12 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/ncu_tf.log 2>&1
tail -3 gpurun_out/ncu_tf.log
