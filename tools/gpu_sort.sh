#!/bin/bash
# Hand-written slot sort: its own tests, the GPU suite, the bench, and a launch list of the timed steps.
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_sort.py -x -q > gpurun_out/pytest_sort.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_sort.log
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for r in 1 2; do timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu > gpurun_out/bench_$r.json 2> gpurun_out/bench_$r.err; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/ncu_bench.log 2>&1
