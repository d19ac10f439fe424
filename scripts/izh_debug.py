import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import specs
from paper_1412_0595_b200 import synscale as S
variant, W = sys.argv[1], int(sys.argv[2])
spec = specs.izh_ff_spec(60.0)
if variant == "none":
    spec.synapses = [g for g in spec.synapses if g.post != "izh"]
elif variant == "in_e":
    spec.synapses = [g for g in spec.synapses if g.name != "in_i"]
elif variant == "in_i":
    spec.synapses = [g for g in spec.synapses if g.name != "in_e"]
elif variant == "n1024":
    for p in spec.populations:
        if p.name == "izh":
            p.size = 1024
            for k in ("a", "b", "c", "d", "noiseAmplitude", "biasCurrent"):
                v = list(getattr(p.params, k)); setattr(p.params, k, v + v[:23])
try:
    sim = S.Simulation(spec, S.StorageMode.FromSpec, S.EngineOptions(window=W, profile=True))
    print(variant, W, {p.name: sim.block_size(p.name) for p in spec.populations}, flush=True)
    sim.step(40)
    sim.sync()
    print(variant, W, "ok", flush=True)
except Exception as e:
    print(variant, W, "FAIL", e, flush=True)
