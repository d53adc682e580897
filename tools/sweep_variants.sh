#!/bin/bash
# On the GPU box: bench (training step; + render with RENDER=1) with each
# experiment library, two rounds.
#   [RENDER=1] bash tools/sweep_variants.sh tag lib1 lib2 ...   (paths relative to the repo; "prod" = product lib)
TAG=$1; shift
mkdir -p gpurun_out/sweep_$TAG
SKIP="--skip-render"
[ -n "$RENDER" ] && SKIP=""
for rep in 1 2; do
for v in "$@"; do
  if [ "$v" = prod ]; then unset DOT_LIB_PATH; else export DOT_LIB_PATH=$PWD/$v; fi
  name=$(basename $v .so)
  timeout 300 python bench.py $SKIP --skip-refine --skip-cpu --steps 30 > gpurun_out/sweep_$TAG/${name}_$rep.json 2> gpurun_out/sweep_$TAG/${name}_$rep.err
  python -c "
import json; d=json.load(open('gpurun_out/sweep_$TAG/${name}_$rep.json'))
r=d.get('render') or {}
print('$name', 'step', round(d['ms_per_step'],4), 'bwd', round(d['roofline']['kernel_ms'],4), 'e2e', round(d['e2e']['ms_per_step'],4),
      'render', round(r.get('rays_per_s',0)/1e9,3), 'sig', round(d['signal_fwd']['ms_per_batch'],4))"
done; done
