#!/bin/bash
# GPU parity tests, then an A/B of library builds / env switches (VARIANTS), 3 reps each, alternating.
mkdir -p gpurun_out
if [ -z "$NOTEST" ]; then timeout 1200 python -m pytest tests -x -q -m gpu ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log; tail -3 gpurun_out/pytest_gpu.log; fi
for rep in 1 2 3; do
for v in ${VARIANTS:-base}; do
  if [ "$v" = base ]; then envs=""; else envs="$v"; fi
  env $envs timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu ${BENCH_ARGS} > gpurun_out/ab.json 2> gpurun_out/ab.err
  python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('$v', d['value'],d['ms_per_step'],d['e2e']['value'],d['phase_ms_per_step'])" || tail -3 gpurun_out/ab.err
done
done
