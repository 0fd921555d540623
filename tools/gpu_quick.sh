#!/bin/bash
# Quick GPU check: selected tests (PYTEST args) + optional extra command (EXTRA).
mkdir -p gpurun_out
TAG=${TAG:-quick}
free -g > gpurun_out/host_mem.txt 2>&1; nproc >> gpurun_out/host_mem.txt
timeout ${TMO:-600} python -m pytest ${PYTEST:-tests -m gpu} -x -q > gpurun_out/pytest_${TAG}.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_${TAG}.log
tail -15 gpurun_out/pytest_${TAG}.log
if [ -n "$EXTRA" ]; then bash -c "$EXTRA"; fi
