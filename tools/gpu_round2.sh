#!/bin/bash
# Round-end style GPU session: all GPU tests, smoke, the default bench line, the reference arm, the
# ncu launch list, one ncu --set full capture of the headline kernels (summarised on the box), and
# every BASELINE config line.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --subset 0 > gpurun_out/launches_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"s2m_ws|l2t_fix|bbox_vec" -c 3 -o /tmp/full \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-op --subset 0 > gpurun_out/full.log 2>&1
python tools/ncu_summary.py /tmp/full.ncu-rep "ncu --set full --clock-control none --import-source on -k regex:\"s2m_ws|l2t_fix|bbox_vec\" -c 3 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-op --subset 0 (n=1e9, C4)" > gpurun_out/ncu_full.json 2>> gpurun_out/full.log
ncu -i /tmp/full.ncu-rep --page source --csv -k regex:s2m_ws --print-source sass > /tmp/s2m_src.csv 2>/dev/null; python tools/ncu_source.py /tmp/s2m_src.csv 30 > gpurun_out/ncu_source_s2m.txt 2>&1
ncu -i /tmp/full.ncu-rep --page source --csv -k regex:l2t_fix --print-source sass > /tmp/l2t_src.csv 2>/dev/null; python tools/ncu_source.py /tmp/l2t_src.csv 30 > gpurun_out/ncu_source_l2t.txt 2>&1
rm -f /tmp/full.ncu-rep
./tools/bench_configs.sh
echo done
