mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_optim.py tests/test_gpu_render.py -q -x > gpurun_out/pytest_new.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_new.log
