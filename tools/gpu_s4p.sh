#!/bin/bash
# M2M split over child groups (few parents with many children): multi-level parity tests, D=7 P=3 / EV=10 / D=5 lines
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -k "msd or c4_ev10 or grid or c5 or large_grids or operator or sharded or parity_end_to_end or device_tree" > gpurun_out/pytest_m2m.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_m2m.log
B="python bench.py --no-e2e --no-cpu-baseline --no-op --subset 1000"
timeout 900 $B --n 1e8 --D 7 --P 3 --node-cap 2187 > gpurun_out/bench_d7p3.json 2> gpurun_out/bench_d7p3.err
timeout 600 $B --n 1e8 --D 5 --P 4 > gpurun_out/bench_d5.json 2> gpurun_out/bench_d5.err
timeout 600 $B --n 1e9 --ev 10 > gpurun_out/bench_ev10.json 2> gpurun_out/bench_ev10.err
echo done
