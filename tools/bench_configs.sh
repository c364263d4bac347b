#!/bin/bash
# Bench lines for the other BASELINE configs (context; the headline is C4 at n = 1e9)
mkdir -p gpurun_out
run() { echo "== $*" >> gpurun_out/configs.jsonl; timeout 900 python bench.py --no-e2e --no-cpu-baseline --steps 3 "$@" 2>> gpurun_out/configs.err | tail -1 >> gpurun_out/configs.jsonl; }
run --n 1e6 --kind normal --ev 1 --subset 500
run --n 1e8 --ev 1 --subset 200
run --n 1e8 --ev 10 --subset 200
run --n 1e8 --ev 0.1 --subset 200
run --n 1e8 --P 6 --ev 1 --subset 200
run --n 1e8 --D 5 --P 4 --subset 100
run --n 1e8 --D 7 --P 2 --subset 100
echo done
