mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_all.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_all.log
timeout 300 python tools/micro.py --order random --flags 0,32768,0 > gpurun_out/micro.log 2>&1
timeout 600 python bench.py --skip-cpu > gpurun_out/bench.json 2> gpurun_out/bench.err
