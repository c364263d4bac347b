#!/bin/bash
# quick loop: GPU parity tests + one bench line (no e2e / cpu baseline) + optional ncu capture
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-e2e --no-cpu-baseline --subset 200 > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err
if [ -n "$NCU_K" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$NCU_K" -c ${NCU_C:-2} -o gpurun_out/quick \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --subset 0 > gpurun_out/quick_ncu.log 2>&1
fi
echo done
