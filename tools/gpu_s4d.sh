#!/bin/bash
# complete-level (grid) M2L + multi-level D=5: parity tests, C5 bench lines, launch list D=7
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_grid.py -x -q > gpurun_out/pytest_grid.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_grid.log
timeout 900 python -m pytest tests -m gpu -x -q -k "large_grids or c5_uniform or parity_end_to_end or device_tree or sparse" > gpurun_out/pytest_d5.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_d5.log
B="python bench.py --n 1e8 --no-e2e --no-cpu-baseline --no-op --subset 1000"
timeout 600 $B --D 5 --P 4 > gpurun_out/bench_d5.json 2> gpurun_out/bench_d5.err
timeout 600 $B --D 7 --P 2 > gpurun_out/bench_d7p2.json 2> gpurun_out/bench_d7p2.err
timeout 900 $B --D 7 --P 3 --node-cap 4096 > gpurun_out/bench_d7p3.json 2> gpurun_out/bench_d7p3.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_d7.csv \
  python bench.py --n 1e8 --D 7 --P 3 --node-cap 4096 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-op --subset 0 > gpurun_out/launches_d7.log 2>&1
echo done
