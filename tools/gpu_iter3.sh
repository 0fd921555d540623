#!/bin/bash
# Iteration: GPU tests, bench A/B (one-launch vs three-kernel reduction), CTA-0 timeline of the
# contraction, launch list and full capture of the reduction kernel.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
for k in 1 2; do
  timeout 600 python bench.py --no-cpu > gpurun_out/bench_$k.json 2> gpurun_out/bench_$k.err
  EMBER_REDUCE_SPLIT=1 timeout 600 python bench.py --no-cpu > gpurun_out/bench_split_$k.json 2> gpurun_out/bench_split_$k.err
done
EMBER_TC_TRACE=gpurun_out/trace timeout 600 python bench.py --no-cpu --steps 5 --warmup 3 > gpurun_out/bench_trace.json 2>&1
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/ncu_launch.log 2>&1
timeout 1200 ncu --profile-from-start off --set full --import-source on --clock-control none \
  -k regex:"k_reduce_pipe|k_long_list" -c 2 -o gpurun_out/reduce_full -f python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu_full.log 2>&1
ls gpurun_out
