python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py -x -q 2>&1 | tail -3
python bench.py --no-e2e --no-cpu-baseline --subset 0 2>&1 | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(j['ms_per_step'], j['phase_ms'])"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"_tma" -c 2 -o gpurun_out/prof_tma3 python bench.py --n 1e8 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --subset 0 > /dev/null 2>&1
echo done
