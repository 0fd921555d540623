#!/bin/bash
# Launch list of bench.py's timed region + one ncu --set full capture of kernels matching $TOPK.
mkdir -p gpurun_out
TAG=${TAG:-prof}
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_${TAG}.csv python bench.py --engine tc --steps 2 --warmup 3 --no-cpu ${BENCH_ARGS} > gpurun_out/ncu_launch_${TAG}.log 2>&1
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:"${TOPK:-k_tc}" -c ${TOPC:-2} \
  -o gpurun_out/full_${TAG} -f python bench.py --engine tc --steps 1 --warmup 3 --no-cpu ${BENCH_ARGS} > gpurun_out/ncu_full_${TAG}.log 2>&1
tail -3 gpurun_out/ncu_full_${TAG}.log
