#!/bin/bash
# round 2, call A: FP32 peak microbenchmark, compute-sanitizer runs, quick bench line
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
./tools/fp32_peak > gpurun_out/fp32_peak.jsonl 2>&1
for t in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_cases.py > gpurun_out/sanitize_$t.log 2>&1
  echo "exit $?" >> gpurun_out/sanitize_$t.log
done
timeout 600 python bench.py --no-e2e --no-cpu-baseline --subset 200 > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err
echo done
