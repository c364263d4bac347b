#!/bin/bash
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"m2l_p2" --launch-skip 1 -c 1 -o /tmp/j7 python bench.py --n 1e7 --D 7 --P 2 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-op --subset 0 > gpurun_out/j7.log 2>&1
python tools/ncu_summary.py /tmp/j7.ncu-rep "k_m2l_p2<7> depth-2 launch, n=1e7 D=7 P=2" > gpurun_out/j7.json 2>> gpurun_out/j7.log
ncu -i /tmp/j7.ncu-rep --page source --csv -k regex:m2l_p2 --print-source sass > /tmp/j7_src.csv 2>/dev/null; python tools/ncu_source.py /tmp/j7_src.csv 40 > gpurun_out/j7_source.txt 2>&1
cp /tmp/j7_src.csv gpurun_out/j7_src.csv
rm -f /tmp/j7.ncu-rep
echo done
