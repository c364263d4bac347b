#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py tests/test_gpu_msd.py -m gpu -q -x > gpurun_out/pytest_k.log 2>&1; echo "exit $?" >> gpurun_out/pytest_k.log
B="python bench.py --no-e2e --no-cpu-baseline --no-op --steps 5 --subset 1000"
timeout 600 $B --n 1e8 --D 7 --P 2 > gpurun_out/k_d7p2.json 2> gpurun_out/k_d7p2.err
timeout 600 $B > gpurun_out/k_c4.json 2> gpurun_out/k_c4.err
timeout 1500 compute-sanitizer --tool racecheck --print-limit 20 python tools/sanitize_cases.py > gpurun_out/sanitize_racecheck.log 2>&1; echo "exit $?" >> gpurun_out/sanitize_racecheck.log
echo done
