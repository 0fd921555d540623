#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_all.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_all.log
tail -5 gpurun_out/pytest_all.log
timeout 600 python bench.py --distributed --steps 60 --warmup 5 > gpurun_out/bench_dist1.json 2> gpurun_out/bench_dist1.err
tail -c 1500 gpurun_out/bench_dist1.json; tail -5 gpurun_out/bench_dist1.err
timeout 900 python bench.py --capacity 8 > gpurun_out/bench_buf8.json 2> gpurun_out/bench_buf8.err
tail -c 1500 gpurun_out/bench_buf8.json; tail -5 gpurun_out/bench_buf8.err
