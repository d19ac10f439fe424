python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1
tail -3 gpurun_out/gputest.log
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-extras | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', d['ms_per_step'], d['value'], d['e2e']['value'])"
python - <<'PY'
import sys; sys.path[:0]=['.','tests']
import specs
from paper_1412_0595_b200 import synscale as S
for n in (100000, 1000000):
    sp=specs.mbody_spec(n,0.05,1000.0)
    sim=S.Simulation(sp,S.StorageMode.FromSpec,S.EngineOptions(window=256))
    print("n_kc",n,"device GB",sim.device_bytes()/1e9); sim.close()
PY
