#!/bin/bash
# after the m = 2187 M2M fix and the complete-level tree shortcut: all GPU tests, smoke, C5 lines, headline, ladder
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
B="python bench.py --n 1e8 --no-e2e --no-cpu-baseline --no-op --subset 1000"
timeout 600 $B --D 5 --P 4 > gpurun_out/bench_d5.json 2> gpurun_out/bench_d5.err
timeout 600 $B --D 7 --P 2 > gpurun_out/bench_d7p2.json 2> gpurun_out/bench_d7p2.err
timeout 900 $B --D 7 --P 3 --node-cap 4096 > gpurun_out/bench_d7p3.json 2> gpurun_out/bench_d7p3.err
timeout 600 python bench.py --no-e2e --no-cpu-baseline --subset 1000 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 900 python bench.py --impl reference --steps 1 --warmup 1 --oracle-ladder > gpurun_out/bench_reference_ladder.json 2> gpurun_out/bench_reference_ladder.err
echo done
