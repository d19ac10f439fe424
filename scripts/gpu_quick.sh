# quick GPU cycle: parity suite, short bench, KC update metrics
python -m pytest tests -m gpu -x -q -k "not kw1 and not golden[8]" > gpurun_out/gputest.log 2>&1
tail -3 gpurun_out/gputest.log
for npt in 4 2; do
SSB_QUAD_NPT=$npt python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-extras > gpurun_out/bench_quick$npt.log 2>&1
tail -1 gpurun_out/bench_quick$npt.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('npt', $npt, d['ms_per_step'], d['value'])"
SSB_QUAD_NPT=$npt ncu --metrics sm__inst_executed.sum,gpu__time_duration.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:condlif --csv --log-file gpurun_out/kc_metrics$npt.csv python scripts/profile_run.py --windows 4 > gpurun_out/kcm.log 2>&1
done
