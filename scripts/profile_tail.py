"""Short fixed workload for ncu: config 3 + STDP on kc_dn (plastic tail kernel).
    ncu --set full -k regex:sink_step -s 1 -c 1 python scripts/profile_tail.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
from paper_1412_0595_b200 import synscale as S  # noqa: E402
import specs  # noqa: E402

spec = specs.stdp_mbody_spec(100_000, 80.0)
sim = S.Simulation(spec, S.StorageMode.FromSpec, S.EngineOptions(window=256))
sim.step(768)
sim.sync()
print("ok", sim.steps_done())
