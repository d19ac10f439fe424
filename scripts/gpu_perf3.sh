for r in 14 24 36 48; do
SSB_DENSE_KERNEL=chain SSB_RESERVED_SMS=$r python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-extras | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench reserved', '$r', d['ms_per_step'])"
done
for r in 24 36; do
SSB_PDL=1 SSB_DENSE_KERNEL=chain SSB_RESERVED_SMS=$r python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-extras | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench pdl reserved', '$r', d['ms_per_step'])"
done
SSB_DENSE_KERNEL=chain SSB_RESERVED_SMS=36 python scripts/trace_kc.py 32 > gpurun_out/trace.txt 2>&1; tail -8 gpurun_out/trace.txt
