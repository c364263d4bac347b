#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_msd.py tests/test_gpu_scale.py tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/pytest_f.log 2>&1; echo "exit $?" >> gpurun_out/pytest_f.log
B="python bench.py --no-e2e --no-cpu-baseline --no-op --steps 5 --subset 1000"
timeout 600 $B --n 1e9 --ev 10 > gpurun_out/f_ev10.json 2> gpurun_out/f_ev10.err
timeout 600 $B --n 1e8 --D 7 --P 2 > gpurun_out/f_d7p2.json 2> gpurun_out/f_d7p2.err
timeout 600 $B --n 1e6 --kind normal --ev 1 > gpurun_out/f_c2.json 2> gpurun_out/f_c2.err
timeout 600 $B --n 1e8 --kind bm > gpurun_out/f_bm.json 2> gpurun_out/f_bm.err
echo done
