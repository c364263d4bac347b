#!/bin/bash
# Bench lines for every BASELINE config besides the headline (C4, n = 1e9, EV = 1), the C5
# accuracy trade-off at D = 7, the Table 5/6 ablation shape and the App. A datasets.
# One JSON line per run in gpurun_out/configs.jsonl, preceded by a "== args" marker line.
mkdir -p gpurun_out
OUT=gpurun_out/${CONFIGS_OUT:-configs.jsonl}
run() { echo "== $*" >> $OUT; timeout 900 python bench.py --no-e2e --no-cpu-baseline --no-op --steps 3 "$@" 2>> gpurun_out/configs.err | tail -1 >> $OUT; }
# C1: n = 1e4, uniform, ls = 1, against the full exact sum
run --n 1e4 --gamma 1.0 --subset 10000
# C2: n = 1e6 normal, EV 1 / 0.1 / 10 (KeOps-style exact sum timed alongside)
run --n 1e6 --kind normal --ev 1
run --n 1e6 --kind normal --ev 0.1
run --n 1e6 --kind normal --ev 10
# C3: n = 1e8 uniform, ls sweep 0.1 .. 10 at P = 4, P sweep 3 .. 6 at EV = 1
for g in 0.1 0.3 1.0 3.0 10.0; do run --n 1e8 --gamma $g; done
for p in 3 5 6; do run --n 1e8 --P $p; done
# C4: the other effective variances at n = 1e9
run --n 1e9 --ev 0.1
run --n 1e9 --ev 10
# C5: n = 1e8, D = 5 and 7 (uniform; FALKON-style N(0, I) and planted KRR targets)
run --n 1e8 --D 5 --P 4
run --n 1e8 --D 5 --P 4 --b planted
run --n 1e8 --D 5 --P 4 --kind normal
run --n 1e8 --D 7 --P 2
run --n 1e8 --D 7 --P 2 --b planted
run --n 1e8 --D 7 --P 2 --flags 32
run --n 1e8 --D 7 --P 3 --node-cap 2187
run --n 1e8 --D 7 --P 2 --eta 0.1
# Tables 5-6 shape: FFM(GPU) = keep empty boxes, no smooth / adaptive / small;
# F^2.5M = no smooth, no adaptive; F^3M = everything on
run --n 1e7 --kind normal --flags 78
run --n 1e7 --kind normal --flags 6
run --n 1e7 --kind normal
# App. A datasets (D = 3)
for k in clustered bm fbm; do run --n 1e8 --kind $k; done
echo done
