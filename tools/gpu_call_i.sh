#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_msd.py tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/pytest_i.log 2>&1; echo "exit $?" >> gpurun_out/pytest_i.log
B="python bench.py --no-e2e --no-cpu-baseline --no-op --steps 10 --subset 1000"
timeout 600 $B > gpurun_out/i_c4a.json 2> gpurun_out/i_c4a.err
timeout 600 $B --n 1e9 --ev 10 > gpurun_out/i_ev10.json 2> gpurun_out/i_ev10.err
timeout 600 $B > gpurun_out/i_c4b.json 2> gpurun_out/i_c4b.err
echo done
