#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g_launches_ev10.csv \
  python bench.py --n 1e9 --ev 10 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-op --subset 0 > gpurun_out/g_launches.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"s2m_ws" -c 1 -o /tmp/gms python bench.py --n 1e9 --ev 10 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-op --subset 0 > gpurun_out/g_ms.log 2>&1
python tools/ncu_summary.py /tmp/gms.ncu-rep "ev10 s2m_ws" > gpurun_out/g_ms.json 2>> gpurun_out/g_ms.log
ncu -i /tmp/gms.ncu-rep --page source --csv -k regex:s2m_ws --print-source sass > /tmp/gms_src.csv 2>/dev/null; python tools/ncu_source.py /tmp/gms_src.csv 30 > gpurun_out/g_ms_source.txt 2>&1
rm -f /tmp/gms.ncu-rep
echo done
