mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_deterministic.py tests/test_gpu_refine.py -q -x > gpurun_out/pytest_det.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_det.log
timeout 300 python tools/exp_det.py > gpurun_out/det.log 2>&1 && \
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/det_launches.csv python tools/exp_det.py >> gpurun_out/det.log 2>&1
