#!/bin/bash
# One gpurun session: GPU parity tests, tcgen05 self-test, a short bench, the ncu launch list of
# the timed region and one full ncu capture of the top kernel. Everything lands in gpurun_out/.
set -x
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvidia-smi.txt 2>&1
ENGINE=${ENGINE:-simt}
CONFIG=${CONFIG:-fb86m}
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/tc_probe.py > gpurun_out/tc_probe.log 2>&1
timeout 900 python bench.py --config $CONFIG --engine $ENGINE --steps ${STEPS:-50} --warmup 5 > gpurun_out/bench_${CONFIG}_${ENGINE}.json 2> gpurun_out/bench_${CONFIG}_${ENGINE}.err
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_${CONFIG}_${ENGINE}.csv python bench.py --config $CONFIG --engine $ENGINE --steps 2 --warmup 3 --no-cpu > gpurun_out/ncu_launch.log 2>&1
if [ -n "$TOPK" ]; then
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:"$TOPK" -c ${TOPC:-1} \
  -o gpurun_out/top_${CONFIG}_${ENGINE} -f python bench.py --config $CONFIG --engine $ENGINE --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu_full.log 2>&1
fi
ls -la gpurun_out
