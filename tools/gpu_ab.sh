#!/bin/bash
# A/B of library variants on the headline bench: variants/libf3m_<name>.so swapped in for libf3m.so
mkdir -p gpurun_out
cp paper_2202_01085_b200/libf3m.so /tmp/libf3m_base.so
for v in base ${VARIANTS}; do
  if [ "$v" = base ]; then cp /tmp/libf3m_base.so paper_2202_01085_b200/libf3m.so; else cp variants/libf3m_$v.so paper_2202_01085_b200/libf3m.so; fi
  for rep in 1 2; do
    timeout 600 python bench.py --no-e2e --no-cpu-baseline --no-op --subset 0 ${BENCH_ARGS} > gpurun_out/ab_${v}_$rep.json 2> gpurun_out/ab_${v}_$rep.err
  done
done
cp /tmp/libf3m_base.so paper_2202_01085_b200/libf3m.so
echo done
