#!/bin/bash
# ncu --set full of the step's memory-bound kernels (one launch each, from bench.py's timed steps).
mkdir -p gpurun_out
timeout 1200 ncu --profile-from-start off --set full --import-source on --clock-control none \
  -k regex:"k_gather_pack|k_chain_pipe|k_segments_pipe|k_long_partial|k_long_final|k_sample_keys|k_dn_reduce" -c 7 \
  -o gpurun_out/mem_full -f python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu_mem.log 2>&1
ls -la gpurun_out/mem_full.ncu-rep
