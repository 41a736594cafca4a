#!/bin/bash
# r02ae: build occupancy sensitivity -- 10 (default), 8, 6 build warps per CTA (2 CTAs per SM)
mkdir -p gpurun_out
cp paper_2109_09056_b200/libparticula_b200.so paper_2109_09056_b200/libparticula_b200_bw10.so
for args in "--cells 128" "--cells 128 --temperature 3.0 --rebuild 5"; do for v in bw10 bw8 bw6; do
  PARTICULA_B200_LIB=libparticula_b200_$v.so timeout 300 python bench.py $args --steps 100 --warmup 10 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v $args value %.4g ms/step %.4f force_us %.1f build_us %.1f' % (d['value'],d['ms_per_step'],d['roofline']['avg_launch_us'],d['roofline_build']['avg_launch_us']))"
done; done 2>&1 | grep -v "^  \|Traceback\|raise\|json.decoder" | tee gpurun_out/ab_buildwarps_r02ae.txt
