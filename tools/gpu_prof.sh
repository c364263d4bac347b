#!/bin/bash
# ncu --set full (+ source) of the C4 bench kernels named by $NCU_K; optional quick bench line first
mkdir -p gpurun_out
if [ -z "$NO_BENCH" ]; then
timeout 600 python bench.py --no-e2e --no-cpu-baseline --subset 200 > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err
fi
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${NCU_K:-s2m_ws|l2t_tma}" -c ${NCU_C:-2} -o gpurun_out/prof \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-op --subset 0 ${BENCH_ARGS} > gpurun_out/prof_ncu.log 2>&1
echo done
