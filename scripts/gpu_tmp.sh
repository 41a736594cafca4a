timeout 1200 python -m pytest tests/test_gpu_dist.py tests/test_gpu_distmd.py tests/test_gpu_decomp.py tests/test_bench_contract.py -m gpu -q -x > gpurun_out/pytest_dist2.txt 2>&1
tail -15 gpurun_out/pytest_dist2.txt
timeout 600 python scripts/fabric_rebuild.py 128 > gpurun_out/fabric_rebuild2.txt 2>&1
head -4 gpurun_out/fabric_rebuild2.txt
timeout 600 python scripts/overlap_timing.py 128 > gpurun_out/overlap_timing.txt 2>&1
cat gpurun_out/overlap_timing.txt
