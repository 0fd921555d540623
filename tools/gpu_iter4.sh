#!/bin/bash
# Iteration: GPU tests, default bench, the library multi-GPU driver at N=1 (--distributed).
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu > gpurun_out/bench_1.json 2> gpurun_out/bench_1.err
timeout 900 python bench.py --distributed --steps 100 --warmup 5 > gpurun_out/bench_dist1.json 2> gpurun_out/bench_dist1.err
tail -5 gpurun_out/bench_dist1.err
ls gpurun_out
