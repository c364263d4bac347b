#!/bin/bash
# skew-aware LSD scatter / un-scatter: sort-path parity, App. A dataset lines, EV=10, D=7, C4
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -k "msd or parity_end_to_end or device_tree or appendix or c4_ev10 or c2_full or operator or c5_uniform or keep_empty or keys_on" > gpurun_out/pytest_skew.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_skew.log
B="python bench.py --no-e2e --no-cpu-baseline --no-op --subset 1000"
for k in clustered bm fbm; do timeout 600 $B --n 1e8 --kind $k > gpurun_out/bench_$k.json 2> gpurun_out/bench_$k.err; done
timeout 600 $B --n 1e9 --ev 10 > gpurun_out/bench_ev10.json 2> gpurun_out/bench_ev10.err
timeout 600 $B --n 1e8 --D 7 --P 2 > gpurun_out/bench_d7p2.json 2> gpurun_out/bench_d7p2.err
timeout 600 $B --n 1e8 --D 5 --P 4 > gpurun_out/bench_d5.json 2> gpurun_out/bench_d5.err
echo done
