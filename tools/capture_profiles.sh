#!/bin/bash
# On the GPU box: bench line + per-step launch list + ncu --set full of the
# dominant kernels, all restricted to the timed steps (DOT_PROFILE_RANGE).
#   bash tools/capture_profiles.sh <tag>
TAG=${1:-r1}
OUT=gpurun_out/prof_$TAG
mkdir -p $OUT
CMD="python bench.py --steps 3 --warmup 3 --skip-cpu --skip-render --skip-refine"
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err
DOT_PROFILE_RANGE=1 timeout 300 $CMD > $OUT/plain.log 2>&1 && \
DOT_PROFILE_RANGE=1 timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \
    --csv --log-file $OUT/launches.csv $CMD > $OUT/ncu_list.log 2>&1
DOT_PROFILE_RANGE=1 timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k regex:"render_bwd_buffered|rmsprop_kernel" -c 2 -o $OUT/full -f $CMD > $OUT/ncu_full.log 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 --skip-cpu --skip-refine > $OUT/plain_render.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:render_camera_kernel -s 3 -c 1 \
    -o $OUT/render_full -f python bench.py --steps 3 --warmup 3 --skip-cpu --skip-refine > $OUT/ncu_render.log 2>&1
ls -la $OUT
