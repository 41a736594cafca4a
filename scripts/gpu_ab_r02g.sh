#!/bin/bash
# r02g: force-kernel tile-wait polling interval (nanosleep 64 / 256 / 1024 ns);
# decomposed rebuild launch list after the local-memory fixes (halo select, owner, bin count)
mkdir -p gpurun_out
VARIANTS="s64 s256 s1024" bash scripts/gpu_ab_force.sh 2>&1 | grep -v "^  \|Traceback\|raise\|json.decoder" > gpurun_out/ab_force_r02g.txt
cat gpurun_out/ab_force_r02g.txt
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --csv --log-file gpurun_out/rebuild_launches_r02g.csv python scripts/rebuild_launches.py 128 > /dev/null 2>&1
python3 scripts/launch_summary.py gpurun_out/rebuild_launches_r02g.csv > gpurun_out/rebuild_launch_summary_r02g.txt 2>&1; head -16 gpurun_out/rebuild_launch_summary_r02g.txt
timeout 600 python scripts/fabric_rebuild.py 128 > gpurun_out/fabric_rebuild_r02g.txt 2>&1; tail -5 gpurun_out/fabric_rebuild_r02g.txt
