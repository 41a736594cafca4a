#!/bin/bash
# r02n: owned-rows-only numbering of decomposed-domain tiles -- dist GPU tests,
# 2x2x2 fabric rebuild launch list and wall time, overlap split timing
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_dist.py tests/test_gpu_distmd.py tests/test_gpu_decomp.py tests/test_bench_contract.py -m gpu -q -x > gpurun_out/pytest_dist_r02n.txt 2>&1; tail -3 gpurun_out/pytest_dist_r02n.txt
timeout 600 ncu --profile-from-start off --clock-control none --metrics gpu__time_duration.sum --csv --log-file gpurun_out/rebuild_launches_r02n.csv python scripts/rebuild_launches.py 128 > /dev/null 2>&1
python3 scripts/launch_summary.py gpurun_out/rebuild_launches_r02n.csv > gpurun_out/rebuild_launch_summary_r02n.txt 2>&1; head -10 gpurun_out/rebuild_launch_summary_r02n.txt
timeout 600 python scripts/fabric_rebuild.py 128 > gpurun_out/fabric_rebuild_r02n.txt 2>&1; grep -v "^ " gpurun_out/fabric_rebuild_r02n.txt | head -4
timeout 600 python scripts/overlap_timing.py 128 > gpurun_out/overlap_timing_r02n.txt 2>&1; tail -6 gpurun_out/overlap_timing_r02n.txt
bash scripts/gpu_r02m.sh
