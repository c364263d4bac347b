#!/bin/bash
# LSD scatter double buffering: sort-path parity tests, C5 / EV=10 lines with launch lists
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -k "parity_end_to_end or device_tree or msd or c4_ev10 or c5_uniform or grid or operator or sharded or c2_full" > gpurun_out/pytest_sort.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_sort.log
B="python bench.py --n 1e8 --no-e2e --no-cpu-baseline --no-op --subset 1000"
timeout 600 $B --D 7 --P 2 > gpurun_out/bench_d7p2.json 2> gpurun_out/bench_d7p2.err
timeout 600 $B --D 5 --P 4 > gpurun_out/bench_d5.json 2> gpurun_out/bench_d5.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_d7p2.csv \
  python bench.py --n 1e8 --D 7 --P 2 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-op --subset 0 > gpurun_out/launches_d7p2.log 2>&1
echo done
