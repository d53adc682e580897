mkdir -p gpurun_out
timeout 300 python tools/micro.py --order random --flags 0,32768,0,32768 > gpurun_out/micro_bm.log 2>&1
