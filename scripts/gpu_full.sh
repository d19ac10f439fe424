python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1
tail -3 gpurun_out/gputest.log
python bench.py --steps 5 --warmup 3 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', d['ms_per_step'], d['value'], d['e2e']['value'], d['config4']['ms_per_sim_second'], d['parity']['split']['match'], d['parity']['config4']['match'], d['roofline']['frac'], d['roofline'].get('frac_of_used_sms'), d['learning']['us_per_timestep'], d['recurrent']['us_per_timestep'])"
