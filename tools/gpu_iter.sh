#!/bin/bash
# One iteration on the GPU box: GPU tests, bench, launch list of the timed region (+ a full capture of $TOPK).
mkdir -p gpurun_out
TAG=${TAG:-iter}
timeout 900 python -m pytest ${PYTEST:-tests -m gpu} -x -q > gpurun_out/pytest_${TAG}.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_${TAG}.log
tail -3 gpurun_out/pytest_${TAG}.log
grep -q "rc=0" gpurun_out/pytest_${TAG}.log || exit 1
timeout 600 python bench.py --steps 50 --warmup 5 ${BENCH_ARGS} > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
python -c "import json;d=json.load(open('gpurun_out/bench_${TAG}.json'));print(d['value'],d['ms_per_step'],d['phase_ms_per_step'],d.get('e2e'))"
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_${TAG}.csv python bench.py --steps 2 --warmup 3 --no-cpu ${BENCH_ARGS} > gpurun_out/ncu_launch_${TAG}.log 2>&1
python tools/ncu_summary.py launches gpurun_out/launches_${TAG}.csv gpurun_out/launches_${TAG}.md | head -30
if [ -n "$TOPK" ]; then
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:"${TOPK}" -c ${TOPC:-2} \
  -o gpurun_out/full_${TAG} -f python bench.py --steps 1 --warmup 3 --no-cpu ${BENCH_ARGS} > gpurun_out/ncu_full_${TAG}.log 2>&1
tail -2 gpurun_out/ncu_full_${TAG}.log
fi
