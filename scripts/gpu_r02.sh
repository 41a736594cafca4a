#!/bin/bash
# Round-2 evidence run: smoke, GPU tests (incl. the reference suite and the
# benched-size parity tests), default bench (C3), driver-like bench, hot
# config, launch list, ncu full captures of the force / build kernels.
T=${1:-r02}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu_$T.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$T.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$T.log
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider -rs --durations=15 > gpurun_out/pytest_gpu_$T.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$T.log
timeout 600 python bench.py > gpurun_out/bench_$T.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_$T.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_drv_$T.log 2>&1
timeout 600 python bench.py --cells 64 --no-cpu-baseline > gpurun_out/bench_c2_$T.log 2>&1
timeout 600 python bench.py --temperature 3.0 --rebuild 5 --no-cpu-baseline > gpurun_out/bench_hot_$T.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$T.csv python bench.py --steps 40 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python3 scripts/launch_summary.py gpurun_out/launches_$T.csv > gpurun_out/launch_summary_$T.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tile_force -s 3 -c 1 -o gpurun_out/${T}_force python bench.py --steps 12 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_${T}_force.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tile_build -s 1 -c 1 -o gpurun_out/${T}_build python bench.py --steps 25 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_${T}_build.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tile_order -s 1 -c 1 -o gpurun_out/${T}_order python bench.py --steps 25 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_${T}_order.log 2>&1
tail -2 gpurun_out/smoke_$T.log; tail -5 gpurun_out/pytest_gpu_$T.log; tail -1 gpurun_out/bench_$T.log | cut -c1-400; head -8 gpurun_out/launch_summary_$T.txt; ls gpurun_out/${T}_*.ncu-rep
