#!/bin/bash
# r02t: build v3 (column lockstep) with the per-column z index vs binary searches (noz), v1, v2
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_tile_r02t.txt 2>&1; tail -2 gpurun_out/pytest_tile_r02t.txt
for args in "--cells 128" "--cells 128 --temperature 3.0 --rebuild 5"; do for rep in 1 2; do
for v in "PC_TILE_BUILD=1" "PC_TILE_BUILD=2" "PC_TILE_BUILD=3" "PC_TILE_BUILD=3 PARTICULA_B200_LIB=libparticula_b200_noz.so"; do
  env $v timeout 300 python bench.py $args --steps 200 --warmup 20 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v $args value %.4g ms/step %.4f force_us %.1f build_us %.1f rebuild_us %.1f' % (d['value'],d['ms_per_step'],d['roofline']['avg_launch_us'],d['roofline_build']['avg_launch_us'],d['roofline_build']['rebuild_us']))"
done; done; done 2>&1 | grep -v "^  \|Traceback\|raise\|json.decoder" | tee gpurun_out/ab_build_r02t.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tile_build2 -s 1 -c 1 -o gpurun_out/r02t_build3 python bench.py --steps 25 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; ls gpurun_out/r02t_*
