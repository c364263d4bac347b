#!/bin/bash
# k_m2l_t column form: mode 0 as 16-byte accesses (P = 4): parity + C5 D=5 normal line
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -k "large_grids or parity_end_to_end or device_tree or sharded or c2_full or scale" > gpurun_out/pytest_m2l.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_m2l.log
timeout 900 python bench.py --n 1e8 --D 5 --P 4 --kind normal --steps 3 --no-e2e --no-cpu-baseline --no-op --subset 1000 > gpurun_out/bench_d5n.json 2> gpurun_out/bench_d5n.err
timeout 600 python bench.py --n 1e6 --kind normal --no-e2e --no-cpu-baseline --no-op --subset 1000 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
echo done
