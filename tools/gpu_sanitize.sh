#!/bin/bash
# compute-sanitizer over tools/sanitize_run.py (small configs, capped contraction grid: several items
# per CTA). One log per tool in gpurun_out/sanitizer_<tool>.log.
mkdir -p gpurun_out
export EMBER_TC_MAXGRID=3
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ "$tool" = racecheck ] && extra="--racecheck-report all"
  timeout 1500 compute-sanitizer --tool $tool $extra --print-limit 50 --error-exitcode 9 python tools/sanitize_run.py \
    > gpurun_out/sanitizer_$tool.log 2>&1
  echo "$tool rc=$?" | tee -a gpurun_out/sanitizer_summary.txt
done
