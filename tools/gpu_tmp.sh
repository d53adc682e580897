mkdir -p gpurun_out
for wo in 0 1; do echo "WO=$wo"; DOT_WARP_ORDER=$wo timeout 300 python tools/micro.py --order random --flags 0,0 --batch 20; done > gpurun_out/micro_wo.log 2>&1
DOT_WARP_ORDER=1 timeout 300 python -m pytest tests/test_gpu_render.py -q -x >> gpurun_out/micro_wo.log 2>&1
