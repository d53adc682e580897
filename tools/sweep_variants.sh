#!/bin/bash
# On the GPU box: bench (training step only) with each experiment library.
#   bash tools/sweep_variants.sh tag lib1 lib2 ...   (paths relative to the repo; "prod" = product lib)
TAG=$1; shift
mkdir -p gpurun_out/sweep_$TAG
for rep in 1 2; do
for v in "$@"; do
  if [ "$v" = prod ]; then unset DOT_LIB_PATH; else export DOT_LIB_PATH=$PWD/$v; fi
  name=$(basename $v .so)
  timeout 300 python bench.py --skip-render --skip-refine --skip-cpu --steps 30 > gpurun_out/sweep_$TAG/${name}_$rep.json 2> gpurun_out/sweep_$TAG/${name}_$rep.err
  python -c "import json,sys; d=json.load(open('gpurun_out/sweep_$TAG/${name}_$rep.json')); print('$name', round(d['ms_per_step'],4), round(d['roofline']['kernel_ms'],4), round(d['e2e']['ms_per_step'],4))"
done; done
