#!/bin/bash
# LSD-replay gather of b for the sorted-path operator; sharded complete-level tests; op bench lines
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_operator.py tests/test_gpu_sharded.py -q > gpurun_out/pytest_op.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_op.log
B="python bench.py --n 1e8 --no-e2e --no-cpu-baseline --subset 1000"
timeout 600 $B --D 7 --P 2 > gpurun_out/bench_d7p2_op.json 2> gpurun_out/bench_d7p2_op.err
timeout 600 $B --D 5 --P 4 > gpurun_out/bench_d5_op.json 2> gpurun_out/bench_d5_op.err
timeout 900 $B --D 7 --P 3 --node-cap 4096 > gpurun_out/bench_d7p3_op.json 2> gpurun_out/bench_d7p3_op.err
timeout 900 python bench.py --n 1e9 --ev 10 --no-e2e --no-cpu-baseline --subset 1000 > gpurun_out/bench_ev10_op.json 2> gpurun_out/bench_ev10_op.err
echo done
