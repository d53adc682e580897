#!/bin/bash
# One GPU session: tests, bench arms, launch list, one ncu --set full capture.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 python bench.py --workload c4 --skip-cpu --steps 10 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
if [ "${NCU:-1}" = 1 ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
   python bench.py --steps 3 --warmup 3 --skip-cpu --skip-render --skip-refine > gpurun_out/ncu_list.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:render_bwd_buffered -s 2 -c 1 \
   -o gpurun_out/bwd_full -f python bench.py --steps 3 --warmup 3 --skip-cpu --skip-render --skip-refine > gpurun_out/ncu_full.log 2>&1
fi
ls -la gpurun_out
