#!/bin/bash
# One iteration on the GPU box: TC parity tests, bench, launch list and a full capture of $TOPK.
mkdir -p gpurun_out
TAG=${TAG:-iter}
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu ${PYK:--k tc} > gpurun_out/pytest_${TAG}.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_${TAG}.log
tail -3 gpurun_out/pytest_${TAG}.log
grep -q "rc=0" gpurun_out/pytest_${TAG}.log || exit 1
timeout 600 python bench.py --engine tc --steps 50 --warmup 5 --no-cpu > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
python -c "import json;d=json.load(open('gpurun_out/bench_${TAG}.json'));print(d['value'],d['ms_per_step'],d['phase_ms_per_step'])"
if [ -n "$PROF" ]; then
  bash tools/gpu_prof.sh
fi
