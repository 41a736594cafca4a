#!/bin/bash
# same-box A/B of environment variants of the default build:
#   ENVS="PC_TILE_BUILD=1 PC_TILE_BUILD=2" ARGS="--cells 128" REPS=2 bash scripts/gpu_ab_env.sh
mkdir -p gpurun_out
for rep in $(seq ${REPS:-2}); do for v in $ENVS; do
  env $v timeout 300 python bench.py ${ARGS:---cells 128} --steps ${STEPS:-200} --warmup 20 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v ${ARGS} value %.4g ms/step %.4f force_us %.1f build_us %.1f rebuild_us %.1f' % (d['value'],d['ms_per_step'],d['roofline']['avg_launch_us'],d['roofline_build']['avg_launch_us'],d['roofline_build']['rebuild_us']))"
done; done
