mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_all.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_all.log
timeout 600 python bench.py --skip-cpu --skip-render --skip-refine > gpurun_out/bench.json 2> gpurun_out/bench.err
DOT_PROFILE_RANGE=1 timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --skip-cpu --skip-render --skip-refine > gpurun_out/ncu_list.log 2>&1
