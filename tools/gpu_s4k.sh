#!/bin/bash
# blk kernels for (7,2) (4,4) (5,3) (6,3): parity; C5 D=7 P=2 line; clustered MSD vs LSD + launch list
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -k "large_grids or c5_uniform or grid or parity_end_to_end or device_tree or sparse or operator or sharded" > gpurun_out/pytest_blk.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_blk.log
B="python bench.py --no-e2e --no-cpu-baseline --no-op --subset 1000"
timeout 600 $B --n 1e8 --D 7 --P 2 > gpurun_out/bench_d7p2.json 2> gpurun_out/bench_d7p2.err
timeout 600 $B --n 1e8 --D 7 --P 2 --flags 32 > gpurun_out/bench_d7p2_mx.json 2> gpurun_out/bench_d7p2_mx.err
timeout 600 $B --n 1e8 --kind clustered > gpurun_out/bench_clu.json 2> gpurun_out/bench_clu.err
F3M_NO_LOCAL=1 timeout 600 $B --n 1e8 --kind clustered > gpurun_out/bench_clu_lsd.json 2> gpurun_out/bench_clu_lsd.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_clu.csv \
  python bench.py --n 1e8 --kind clustered --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-op --subset 0 > gpurun_out/launches_clu.log 2>&1
echo done
