VARIANTS="novir base nosb nopf" bash scripts/gpu_ab_force.sh > gpurun_out/ab_force1.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_scale.py tests/test_gpu_parity.py -m gpu -q -x -k "md_ or c2 or c3 or hot" > gpurun_out/pytest_ab1.txt 2>&1
tail -3 gpurun_out/pytest_ab1.txt
cat gpurun_out/ab_force1.txt
