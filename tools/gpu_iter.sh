#!/bin/bash
# iteration loop on one B200: [pre-command] + GPU tests (TESTS, default all -m gpu) + quick bench line
# + optional ncu --set full capture of kernels matching NCU_K (n = NCU_N, default 1e9)
mkdir -p gpurun_out
[ -n "$PRE" ] && eval "$PRE"
if [ "$TESTS" != "none" ]; then
  timeout 1200 python -m pytest ${TESTS:-tests -m gpu} -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
fi
timeout 600 python bench.py --no-e2e --no-cpu-baseline --subset 200 ${BENCH_ARGS} > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err
if [ -n "$NCU_K" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$NCU_K" -c ${NCU_C:-2} -o gpurun_out/quick \
  python bench.py --n ${NCU_N:-1e9} --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-op --subset 0 ${BENCH_ARGS} > gpurun_out/quick_ncu.log 2>&1
fi
[ -n "$POST" ] && eval "$POST"
echo done
