#!/bin/bash
# Iteration run: GPU tests, default bench twice, launch list, full capture of the memory-bound step kernels.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
for k in 1 2; do timeout 600 python bench.py --no-cpu > gpurun_out/bench_$k.json 2> gpurun_out/bench_$k.err; done
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/ncu_launch.log 2>&1
timeout 1200 ncu --profile-from-start off --set full --import-source on --clock-control none \
  -k regex:"${NCU_K:-k_gather_pack|k_chain_pipe|k_segments_pipe|k_long_partial|k_long_final}" -c ${NCU_C:-5} \
  -o gpurun_out/step_full -f python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu_full.log 2>&1
ls gpurun_out
