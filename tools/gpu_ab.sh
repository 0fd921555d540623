#!/bin/bash
# A/B of environment switches on the bench (no tests): VARIANTS="NAME=VAL ..." ; "base" = no switch;
# "A=1__B=2" sets both.
mkdir -p gpurun_out
for v in ${VARIANTS:-base}; do
  if [ "$v" = base ]; then envs=""; else envs="${v//__/ }"; fi
  for rep in 1 2; do
    env $envs timeout 150 python bench.py --steps 200 --warmup 10 --no-cpu ${BENCH_ARGS} > gpurun_out/ab.json 2> gpurun_out/ab.err
    python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('$v', d['value'],d['ms_per_step'],d['phase_ms_per_step'])" || tail -3 gpurun_out/ab.err
  done
done
