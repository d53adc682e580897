mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_all.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_all.log
timeout 300 python tools/micro.py --order random --flags 0,0 > gpurun_out/micro.log 2>&1
