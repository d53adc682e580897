#!/bin/bash
# On the GPU box: bench line + per-step launch list + ncu --set full of the
# dominant kernels (restricted to the timed steps via DOT_PROFILE_RANGE), the
# 200-view render launch, and the launch list (time + DRAM bytes) of one
# configs[4] refine pass (DOT_PROFILE_REFINE).
#   bash tools/capture_profiles.sh <tag>        then here: python tools/summarise_profiles.py <tag>
TAG=${1:-r2}
OUT=gpurun_out/prof_$TAG
mkdir -p $OUT
CMD="python bench.py --steps 3 --warmup 3 --skip-cpu --skip-render --skip-refine"
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err
DOT_PROFILE_RANGE=1 timeout 300 $CMD > $OUT/plain.log 2>&1 && \
DOT_PROFILE_RANGE=1 timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \
    --csv --log-file $OUT/launches.csv $CMD > $OUT/ncu_list.log 2>&1
DOT_PROFILE_RANGE=1 timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k regex:"render_bwd_buffered|rmsprop|plan_coop" -c 3 -o $OUT/full -f $CMD > $OUT/ncu_full.log 2>&1
RCMD="python bench.py --steps 3 --warmup 3 --skip-cpu --skip-refine"
timeout 600 $RCMD > $OUT/plain_render.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:render_camera_kernel -s 3 -c 1 \
    -o $OUT/render_full -f $RCMD > $OUT/ncu_render.log 2>&1
FCMD="python bench.py --steps 3 --warmup 3 --skip-cpu --skip-render"
DOT_PROFILE_REFINE=1 timeout 600 $FCMD > $OUT/plain_refine.log 2>&1 && \
DOT_PROFILE_REFINE=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file $OUT/refine_launches.csv $FCMD > $OUT/ncu_refine.log 2>&1
ls -la $OUT
