#!/bin/bash
# C5 accuracy / time trade-off: tensor grids vs Smolyak sparse grids (reading R27), n = 1e8 unless noted
mkdir -p gpurun_out
OUT=gpurun_out/${CONFIGS_OUT:-sparse_configs.jsonl}
run() { echo "== $*" >> $OUT; timeout ${TO:-600} python bench.py --no-e2e --no-cpu-baseline --no-op --steps 3 --subset 1000 "$@" 2>> gpurun_out/sparse_configs.err | tail -1 >> $OUT; }
run --n 1e8 --D 5 --P 4
run --n 1e8 --D 5 --P 4 --sparse-level 2
run --n 1e8 --D 5 --P 4 --sparse-level 3
run --n 1e8 --D 7 --P 2
run --n 1e8 --D 7 --P 3 --node-cap 2187
run --n 1e8 --D 7 --P 4 --sparse-level 1
run --n 1e8 --D 7 --P 2 --flags 32
run --n 1e8 --D 7 --P 3 --node-cap 2187 --flags 32
TO=900 run --n 1e7 --D 7 --P 4 --sparse-level 2 --steps 1 --warmup 1
run --n 1e8 --D 3 --P 4 --sparse-level 3
echo done
