#!/bin/bash
# software-pipelined sorted S2M / L2T (k_s2m / k_l2t): parity subset, C5 D=7 P=2, C3 ls=0.1, C2 lines
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -k "parity_end_to_end or device_tree or c5_uniform or grid or c2_full or c4_ev10 or large_grids" > gpurun_out/pytest_far.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_far.log
B="python bench.py --no-e2e --no-cpu-baseline --no-op --subset 1000"
timeout 600 $B --n 1e8 --D 7 --P 2 > gpurun_out/bench_d7p2.json 2> gpurun_out/bench_d7p2.err
timeout 600 $B --n 1e8 --gamma 0.1 > gpurun_out/bench_ls01.json 2> gpurun_out/bench_ls01.err
timeout 600 $B --n 1e6 --kind normal > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
echo done
