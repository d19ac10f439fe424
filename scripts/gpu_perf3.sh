for g in 8 12 16 24 48; do
SSB_GRAPH_WINDOWS=$g python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-extras | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench graphwin', '$g', d['ms_per_step'])"
done
python - <<'PY'
import sys; sys.path[:0]=['.','tests']
import specs
from paper_1412_0595_b200 import synscale as S
for g in ("8","16","48"):
    import os; os.environ["SSB_GRAPH_WINDOWS"]=g
    sp=specs.mbody_spec(100000,0.05,1000.0)
    sim=S.Simulation(sp,S.StorageMode.FromSpec,S.EngineOptions(window=256))
    print("graphwin",g,"device GB",sim.device_bytes()/1e9); sim.close()
PY
