#!/bin/bash
# D = 5 register-blocked S2M / L2T: parity tests, C5 D=5 bench (blk vs the gen kernels), ncu of the new kernels
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "large_grids or c5_uniform or parity_end_to_end" > gpurun_out/pytest_d5.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_d5.log
B="python bench.py --n 1e8 --D 5 --P 4 --no-e2e --no-cpu-baseline --no-op --subset 1000"
timeout 600 $B > gpurun_out/bench_d5_blk.json 2> gpurun_out/bench_d5_blk.err
F3M_NO_BLK=1 timeout 600 $B > gpurun_out/bench_d5_gen.json 2> gpurun_out/bench_d5_gen.err
timeout 600 $B --kind normal > gpurun_out/bench_d5n_blk.json 2> gpurun_out/bench_d5n_blk.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"blk" -c 2 -o gpurun_out/d5blk \
  python bench.py --n 1e8 --D 5 --P 4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-op --subset 0 > gpurun_out/d5_ncu.log 2>&1
echo done
