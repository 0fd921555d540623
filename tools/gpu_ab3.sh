#!/bin/bash
# A/B of an environment switch on the default bench (alternating, 3 runs each), plus GPU tests.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
for k in 1 2 3; do
  timeout 600 python bench.py --no-cpu > gpurun_out/ab_new_$k.json 2> gpurun_out/ab_new_$k.err
  env $AB_ENV timeout 600 python bench.py --no-cpu > gpurun_out/ab_old_$k.json 2> gpurun_out/ab_old_$k.err
done
for f in gpurun_out/ab_*.json; do python -c "import json,sys;d=json.load(open('$f'));print('$f',d['value'],d['ms_per_step'],d['phase_ms_per_step'])"; done
if [ -n "$NCU_K" ]; then
timeout 1200 ncu --profile-from-start off --set full --import-source on --clock-control none \
  -k regex:"$NCU_K" -c ${NCU_C:-1} -o gpurun_out/ab_full -f python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu_full.log 2>&1
fi
