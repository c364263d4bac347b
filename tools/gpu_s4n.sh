#!/bin/bash
# D = 7 P = 3 register-blocked tiles 12 x 7 (scalar c loads, 81 % of the tile useful instead of 71 %)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -k "grid or large_grids or sharded_complete or c5_accuracy" > gpurun_out/pytest_d7p3.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_d7p3.log
timeout 900 python bench.py --n 1e8 --D 7 --P 3 --node-cap 2187 --no-e2e --no-cpu-baseline --no-op --subset 1000 > gpurun_out/bench_d7p3.json 2> gpurun_out/bench_d7p3.err
echo done
