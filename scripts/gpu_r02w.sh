#!/bin/bash
# r02w: build sweep -- hit stores without a memory clobber (bnc) and the next
# step's candidates loaded one step ahead (bpf, default) vs the r02 build (bold)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_tile_r02w.txt 2>&1; tail -2 gpurun_out/pytest_tile_r02w.txt
for args in "--cells 128" "--cells 128 --temperature 3.0 --rebuild 5"; do for rep in 1 2; do for v in bold bnc bpf; do
  PARTICULA_B200_LIB=libparticula_b200_$v.so timeout 300 python bench.py $args --steps 200 --warmup 20 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v $args value %.4g ms/step %.4f force_us %.1f build_us %.1f rebuild_us %.1f' % (d['value'],d['ms_per_step'],d['roofline']['avg_launch_us'],d['roofline_build']['avg_launch_us'],d['roofline_build']['rebuild_us']))"
done; done; done 2>&1 | grep -v "^  \|Traceback\|raise\|json.decoder" | tee gpurun_out/ab_build_r02w.txt
