#!/bin/bash
# grid M2L column kernel + D=7 P=3 register-blocked S2M/L2T: all GPU tests, C5 lines, D7P3 launch list + ncu
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
B="python bench.py --n 1e8 --no-e2e --no-cpu-baseline --no-op --subset 1000"
timeout 600 $B --D 5 --P 4 > gpurun_out/bench_d5.json 2> gpurun_out/bench_d5.err
timeout 600 $B --D 7 --P 2 > gpurun_out/bench_d7p2.json 2> gpurun_out/bench_d7p2.err
timeout 900 $B --D 7 --P 3 --node-cap 4096 > gpurun_out/bench_d7p3.json 2> gpurun_out/bench_d7p3.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_d7.csv \
  python bench.py --n 1e8 --D 7 --P 3 --node-cap 4096 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-op --subset 0 > gpurun_out/launches_d7.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"blk|grid_col" -c 12 -o gpurun_out/d7blk \
  python bench.py --n 1e8 --D 7 --P 3 --node-cap 4096 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-op --subset 0 > gpurun_out/d7_ncu.log 2>&1
echo done
