#!/bin/bash
# Slot-sort iteration: its tests + a launch list of the bench's timed steps.
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_sort.py tests/test_gpu_parity.py -x -q > gpurun_out/pytest_sort.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_sort.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/ncu_bench.log 2>&1
timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu > gpurun_out/bench_1.json 2> gpurun_out/bench_1.err
