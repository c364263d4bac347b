#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_msd.py -m gpu -q -x > gpurun_out/pytest_msd.log 2>&1; echo "exit $?" >> gpurun_out/pytest_msd.log
timeout 600 python bench.py --no-e2e --no-cpu-baseline --no-op --steps 5 --subset 200 --n 1e9 --ev 10 > gpurun_out/ev10.json 2> gpurun_out/ev10.err
timeout 600 python bench.py --no-e2e --no-cpu-baseline --no-op --steps 5 --subset 200 --n 1e8 --gamma 0.1 > gpurun_out/ls01.json 2> gpurun_out/ls01.err
timeout 600 python bench.py --no-e2e --no-cpu-baseline --no-op --subset 200 > gpurun_out/c4.json 2> gpurun_out/c4.err
echo done
