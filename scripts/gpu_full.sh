#!/bin/bash
# Full round evidence: smoke, GPU tests, default bench, launch list, ncu full captures.
T=${1:-full}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu_$T.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$T.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$T.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_$T.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$T.log
timeout 900 python bench.py > gpurun_out/bench_$T.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_$T.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_$T.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$T.csv python bench.py --steps 40 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python3 scripts/launch_summary.py gpurun_out/launches_$T.csv > gpurun_out/launch_summary_$T.txt 2>&1
bash scripts/gpu_ncu2.sh $T > /dev/null 2>&1
tail -2 gpurun_out/smoke_$T.log; tail -3 gpurun_out/pytest_gpu_$T.log; tail -1 gpurun_out/bench_$T.log; tail -1 gpurun_out/bench_ref_$T.log | cut -c1-200; head -8 gpurun_out/launch_summary_$T.txt; ls gpurun_out/${T}_*.ncu-rep
