#!/bin/bash
# ncu --set full captures of the non-headline kernels (deep-tree sort passes at EV = 10,
# C5 D = 5 / 7 far-field kernels, the sparse-grid kernels); one bench step each (numbers printed under
# ncu are never bench values).  Reports are summarised on the box (tools/ncu_summary.py) and deleted.
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 2 --no-e2e --no-cpu-baseline --no-op --subset 0"
cap() {  # name kernel-regex count bench-args...
  local name=$1 k=$2 c=$3; shift 3
  timeout 900 ncu --set full --clock-control none -k regex:"$k" -c $c -o /tmp/$name $B "$@" > gpurun_out/$name.log 2>&1
  python tools/ncu_summary.py /tmp/$name.ncu-rep "ncu --set full -k regex:$k -c $c bench.py $*" > gpurun_out/$name.json 2>> gpurun_out/$name.log
  rm -f /tmp/$name.ncu-rep
}
cap prof_ev10 "lsd_|k_m2m|k_l2l|k_s2m<|k_l2t<" 8 --n 1e8 --ev 10
cap prof_d5 "gen|m2l" 4 --n 1e7 --D 5 --P 4
cap prof_d7p2 "m2l|s2m|l2t" 4 --n 1e7 --D 7 --P 2
cap prof_d7p3 "m2l_p3" 1 --n 1e7 --D 7 --P 3 --node-cap 2187
cap prof_sparse "sparse|dense_rows" 5 --n 1e7 --D 5 --P 4 --sparse-level 2
echo done
