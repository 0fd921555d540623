#!/bin/bash
# Round checkpoint on one B200: GPU tests, the default bench (with the CPU baseline), the reference
# arm, a launch list of the timed steps, one ncu --set full capture of every kernel of one step, and
# the rows/dN kernels' per-CTA spans.
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvidia-smi.txt 2>&1
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/ncu_launch.log 2>&1
timeout 1200 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:"^k_" -c 16 \
  -o gpurun_out/step_full -f python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu_full.log 2>&1
EMBER_TC_CTATIMES=gpurun_out/ct.bin timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/ct_bench.json 2>&1
