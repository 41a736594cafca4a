#!/bin/bash
# r02e: HEAD evidence after the claim-ahead revert -- default bench (C3),
# decomposed-engine tests, overlap split cost, 2x2x2 rebuild launch list,
# fresh ncu source capture of the force kernel (stall attribution)
T=r02e
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench_$T.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_$T.log
timeout 1500 python -m pytest tests/test_gpu_dist.py tests/test_gpu_distmd.py tests/test_gpu_decomp.py -m gpu -q > gpurun_out/pytest_dist_$T.txt 2>&1; tail -3 gpurun_out/pytest_dist_$T.txt
timeout 600 python scripts/overlap_timing.py 128 > gpurun_out/overlap_timing_$T.txt 2>&1; tail -6 gpurun_out/overlap_timing_$T.txt
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --csv --log-file gpurun_out/rebuild_launches_$T.csv python scripts/rebuild_launches.py 128 > /dev/null 2>&1
python3 scripts/launch_summary.py gpurun_out/rebuild_launches_$T.csv > gpurun_out/rebuild_launch_summary_$T.txt 2>&1; head -14 gpurun_out/rebuild_launch_summary_$T.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tile_force -s 3 -c 1 -o gpurun_out/${T}_force python bench.py --steps 12 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_${T}_force.log 2>&1
tail -1 gpurun_out/bench_$T.log | cut -c1-300
