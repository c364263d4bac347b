#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize_cases.py
mkdir -p gpurun_out
for t in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_cases.py > gpurun_out/sanitize_$t.log 2>&1
  echo "exit $?" >> gpurun_out/sanitize_$t.log
done
echo done
