#!/bin/bash
# iteration loop: md parity subset, bench, launch list, ncu of force+build
mkdir -p gpurun_out
T=${1:-it}
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "md_" > gpurun_out/pytest_$T.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_$T.log; tail -4 gpurun_out/pytest_$T.log
timeout 300 python bench.py --steps 400 --warmup 20 --no-cpu-baseline --no-e2e > gpurun_out/bench_$T.log 2>&1
tail -1 gpurun_out/bench_$T.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('value',d['value'],'ms/step',d['ms_per_step'],'force_us',d['roofline']['avg_launch_us'],'frac',d['roofline']['frac'])" || tail -5 gpurun_out/bench_$T.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches_$T.csv python bench.py --steps 25 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python3 scripts/launch_summary.py gpurun_out/launches_$T.csv > gpurun_out/launch_summary_$T.txt 2>&1; head -8 gpurun_out/launch_summary_$T.txt
if [ "$2" == "ncu" ]; then bash scripts/gpu_ncu2.sh $T > /dev/null 2>&1; ls gpurun_out/${T}_*.ncu-rep; fi
