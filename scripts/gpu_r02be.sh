#!/bin/bash
# r02be: HEAD after the u/2 force change: smoke, all GPU tests, default bench, C2, hot, driver-style 20 steps, launch list, force ncu
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r02be.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_r02be.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_r02be.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_r02be.log
timeout 900 python bench.py > gpurun_out/bench_r02be.log 2>&1
timeout 600 python bench.py --cells 64 > gpurun_out/bench_c2_r02be.log 2>&1
timeout 900 python bench.py --temperature 3.0 --rebuild 5 > gpurun_out/bench_hot_r02be.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_drv_r02be.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r02be.csv python bench.py --steps 40 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python3 scripts/launch_summary.py gpurun_out/launches_r02be.csv > gpurun_out/launch_summary_r02be.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tile_force -s 3 -c 1 -o gpurun_out/r02be_force python bench.py --steps 12 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
tail -1 gpurun_out/smoke_r02be.log; tail -2 gpurun_out/pytest_gpu_r02be.log
