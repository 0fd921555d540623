mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "tc" > gpurun_out/pytest_tc.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_tc.log
tail -30 gpurun_out/pytest_tc.log
if grep -q "rc=0" gpurun_out/pytest_tc.log; then
  timeout 600 python bench.py --engine tc --steps 50 --warmup 5 --no-cpu > gpurun_out/bench_fb86m_tc.json 2> gpurun_out/bench_fb86m_tc.err
  cat gpurun_out/bench_fb86m_tc.json; tail -5 gpurun_out/bench_fb86m_tc.err
fi
