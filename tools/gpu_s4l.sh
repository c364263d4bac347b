#!/bin/bash
# MSD decline for unbalanced buckets; (7,2) back on k_s2m/k_l2t: msd + far parity, config lines
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -k "msd or large_grids or c5_uniform or c4_ev10 or appendix" > gpurun_out/pytest_msd.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_msd.log
B="python bench.py --no-e2e --no-cpu-baseline --no-op --subset 1000"
for k in clustered bm fbm; do timeout 600 $B --n 1e8 --kind $k > gpurun_out/bench_$k.json 2> gpurun_out/bench_$k.err; done
timeout 600 $B --n 1e9 --ev 10 > gpurun_out/bench_ev10.json 2> gpurun_out/bench_ev10.err
timeout 600 $B --n 1e8 --D 7 --P 2 > gpurun_out/bench_d7p2.json 2> gpurun_out/bench_d7p2.err
echo done
