#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -k "large_grids" -m gpu -q > gpurun_out/pytest_large.log 2>&1; echo "exit $?" >> gpurun_out/pytest_large.log
timeout 600 python bench.py --no-e2e --no-cpu-baseline --no-op --steps 3 --subset 1000 --n 1e8 --D 7 --P 3 --node-cap 2187 > gpurun_out/d7p3.json 2> gpurun_out/d7p3.err
VARIANTS=match ./tools/gpu_ab.sh
./tools/gpu_prof_secondary.sh
