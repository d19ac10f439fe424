# perf iteration: key parity tests, bench, trace
python -m pytest tests/test_gpu_parity.py -x -q -k "config3_full_second or cfg3_20ms or division_edge or fault_injection or split_world or bench_split_networks_match_parity_golden and not golden[8]" > gpurun_out/gputest_perf.log 2>&1
tail -2 gpurun_out/gputest_perf.log
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-extras | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', d['ms_per_step'], d['value'])"
python scripts/trace_kc.py 32 > gpurun_out/trace.txt 2>&1; tail -8 gpurun_out/trace.txt
