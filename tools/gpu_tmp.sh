mkdir -p gpurun_out
for L in 7 8 7 8; do echo "L=$L"; DOT_LOCATE_LEVEL=$L timeout 600 python bench.py --skip-cpu --skip-refine --steps 20 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['roofline']['kernel_ms'], d['render']['rays_per_s'])"; done > gpurun_out/bench_L.log 2>&1
