#!/bin/bash
# e2e (host-batch path) vs device-resident value under environment variants: VARIANTS="NAME=VAL ..."
mkdir -p gpurun_out
for v in ${VARIANTS:-base}; do
  if [ "$v" = base ]; then envs=""; else envs="${v//__/ }"; fi
  env $envs timeout 150 python bench.py --steps 100 --warmup 10 --no-cpu > gpurun_out/e.json 2> gpurun_out/e.err
  python -c "import json;d=json.load(open('gpurun_out/e.json'));print('$v', d['value'], d['ms_per_step'], d['e2e']['value'], d['e2e']['device_span_ms_per_step'])" || tail -3 gpurun_out/e.err
done
