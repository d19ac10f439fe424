for r in 37 44 50 60; do
SSB_RESERVED_SMS=$r python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-extras | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench reserved', '$r', d['ms_per_step'])"
done
python scripts/sweeps.py density 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l)
    if d['kernel']=='sparse_sliced': print(d['frac'], d['us'], d['frac_of_peak'], d['bit_exact_vs_fold'])"
