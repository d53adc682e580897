mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_deterministic.py tests/test_gpu_render.py -q -s > gpurun_out/pytest_det.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_det.log
timeout 600 python -m pytest tests -m gpu -q > gpurun_out/pytest_all.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_all.log
timeout 300 python tools/micro.py --order random --flags 0,det,0 > gpurun_out/micro_det.log 2>&1
