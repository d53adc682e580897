mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_refine.py tests/test_gpu_optim.py tests/test_gpu_deterministic.py -q -x > gpurun_out/pytest_refine.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_refine.log
timeout 300 python tools/micro_refine.py > gpurun_out/refine.log 2>&1 && \
DOT_PROFILE_REFINE=1 timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/refine_launches.csv python tools/micro_refine.py > gpurun_out/refine_ncu.log 2>&1
