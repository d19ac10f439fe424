python -m pytest tests/test_gpu_parity.py -x -q -k "config3_full_second or cfg3_20ms or split_world or bench_split_networks_match_parity_golden and not golden[8]" > gpurun_out/gputest_perf.log 2>&1
tail -1 gpurun_out/gputest_perf.log
for k in rowstream ldg chain; do
SSB_DENSE_KERNEL=$k python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-extras | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', '$k', d['ms_per_step'])"
done
python scripts/trace_kc.py 32 > gpurun_out/trace.txt 2>&1; tail -8 gpurun_out/trace.txt
