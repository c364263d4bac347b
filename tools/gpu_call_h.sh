#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_msd.py tests/test_gpu_fullsize.py -m gpu -q -x > gpurun_out/pytest_h.log 2>&1; echo "exit $?" >> gpurun_out/pytest_h.log
B="python bench.py --no-e2e --no-cpu-baseline --no-op --steps 5 --subset 1000"
timeout 600 $B --n 1e9 --ev 10 > gpurun_out/h_ev10.json 2> gpurun_out/h_ev10.err
timeout 600 $B > gpurun_out/h_c4.json 2> gpurun_out/h_c4.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/h_launches_ev10.csv \
  python bench.py --n 1e9 --ev 10 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-op --subset 0 > gpurun_out/h_launches.log 2>&1
echo done
