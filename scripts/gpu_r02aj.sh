#!/bin/bash
# r02aj: P2P transport tests after the plan refactor; 2x2x2 fabric rebuild cost and launch list at HEAD
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_distmd.py tests/test_bench_contract.py -m gpu -q -p no:cacheprovider > gpurun_out/pytest_distmd_r02aj.txt 2>&1; tail -2 gpurun_out/pytest_distmd_r02aj.txt
timeout 600 python scripts/fabric_rebuild.py 128 > gpurun_out/fabric_rebuild_r02aj.txt 2>&1; grep -v "^  " gpurun_out/fabric_rebuild_r02aj.txt | head -6
timeout 600 ncu --profile-from-start off --clock-control none --metrics gpu__time_duration.sum --csv --log-file gpurun_out/rebuild_launches_r02aj.csv python scripts/rebuild_launches.py 128 > /dev/null 2>&1
python3 scripts/launch_summary.py gpurun_out/rebuild_launches_r02aj.csv > gpurun_out/rebuild_launch_summary_r02aj.txt 2>&1; head -14 gpurun_out/rebuild_launch_summary_r02aj.txt
