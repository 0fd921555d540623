#!/bin/bash
# A/B of two builds: ab/base.so (tools/build_base.sh) vs the working tree's library, alternating.
mkdir -p gpurun_out
for rep in 1 2 3; do
  for v in base new; do
    if [ "$v" = base ]; then export EMBER_LIB=ab/base.so; else unset EMBER_LIB; fi
    timeout 150 python bench.py --steps 200 --warmup 10 --no-cpu ${BENCH_ARGS} > gpurun_out/ab.json 2> gpurun_out/ab.err
    python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('$v', d['value'],d['ms_per_step'],d['phase_ms_per_step'])" || tail -3 gpurun_out/ab.err
  done
done
