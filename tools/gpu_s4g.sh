#!/bin/bash
# sorted-path operator reuse tests, plan-reuse bench lines (C5 D=7 P=2 / D=5), sanitizers on the new kernels
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_operator.py -q > gpurun_out/pytest_op.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_op.log
B="python bench.py --n 1e8 --no-e2e --no-cpu-baseline --subset 1000"
timeout 600 $B --D 7 --P 2 > gpurun_out/bench_d7p2_op.json 2> gpurun_out/bench_d7p2_op.err
timeout 600 $B --D 5 --P 4 > gpurun_out/bench_d5_op.json 2> gpurun_out/bench_d5_op.err
for t in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_cases.py 3 8 11 12 13 > gpurun_out/sanitize_$t.log 2>&1
  echo "exit $?" >> gpurun_out/sanitize_$t.log
done
echo done
