#!/bin/bash
# ncu --set full captures of the non-headline kernels (deep-tree sort passes at EV = 10,
# C5 D = 5 / 7 far-field kernels, the sparse-grid kernels); one bench step each (numbers printed under
# ncu are never bench values)
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 2 --no-e2e --no-cpu-baseline --no-op --subset 0"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"lsd_|k_m2m|k_l2l|k_s2m<|k_l2t<" -c 8 -o gpurun_out/prof_ev10 \
  $B --n 1e8 --ev 10 > gpurun_out/prof_ev10.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gen|m2l" -c 4 -o gpurun_out/prof_d5 \
  $B --n 1e7 --D 5 --P 4 > gpurun_out/prof_d5.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"m2l|s2m|l2t" -c 4 -o gpurun_out/prof_d7 \
  $B --n 1e7 --D 7 --P 2 > gpurun_out/prof_d7.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sparse|dense_rows" -c 5 -o gpurun_out/prof_sparse \
  $B --n 1e7 --D 5 --P 4 --sparse-level 2 > gpurun_out/prof_sparse.log 2>&1
echo done
