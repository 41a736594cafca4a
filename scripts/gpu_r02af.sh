#!/bin/bash
# r02af: u8 hit rows in the build (MODE 2: 4.8 instead of 7.4 KB per warp) with 12/13/14 warps
# per CTA vs the u16 build with 10 warps (PC_TILE_HITS8=0)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py tests/test_gpu_dist.py tests/test_gpu_distmd.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_b8_r02af.txt 2>&1; tail -2 gpurun_out/pytest_b8_r02af.txt
cp paper_2109_09056_b200/libparticula_b200.so paper_2109_09056_b200/libparticula_b200_b8w13.so
for args in "--cells 128" "--cells 128 --temperature 3.0 --rebuild 5"; do for rep in 1 2; do
for v in "PC_TILE_HITS8=0 PARTICULA_B200_LIB=libparticula_b200_b8w13.so" "PARTICULA_B200_LIB=libparticula_b200_b8w12.so" "PARTICULA_B200_LIB=libparticula_b200_b8w13.so" "PARTICULA_B200_LIB=libparticula_b200_b8w14.so"; do
  env $v timeout 300 python bench.py $args --steps 100 --warmup 10 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v $args value %.4g ms/step %.4f force_us %.1f build_us %.1f' % (d['value'],d['ms_per_step'],d['roofline']['avg_launch_us'],d['roofline_build']['avg_launch_us']))"
done; done; done 2>&1 | grep -v "^  \|Traceback\|raise\|json.decoder" | tee gpurun_out/ab_b8_r02af.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tile_build -s 1 -c 1 -o gpurun_out/r02af_build python bench.py --steps 25 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; ls gpurun_out/r02af_*
