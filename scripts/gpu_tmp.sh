VARIANTS="next0 next1" bash scripts/gpu_ab_force.sh > gpurun_out/ab_force2.txt 2>&1
cat gpurun_out/ab_force2.txt
timeout 1200 python -m pytest tests/test_gpu_dist.py tests/test_gpu_distmd.py tests/test_gpu_decomp.py -m gpu -q > gpurun_out/pytest_dist4.txt 2>&1
tail -5 gpurun_out/pytest_dist4.txt
timeout 600 python scripts/overlap_timing.py 128 > gpurun_out/overlap_timing.txt 2>&1
tail -4 gpurun_out/overlap_timing.txt
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --csv --log-file gpurun_out/rebuild_launches.csv python scripts/rebuild_launches.py 128 > /dev/null 2>&1
python3 scripts/launch_summary.py gpurun_out/rebuild_launches.csv > gpurun_out/rebuild_launch_summary.txt 2>&1
head -12 gpurun_out/rebuild_launch_summary.txt
