"""Short fixed cyclic workload for ncu (the acceptance network, 4 windows)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
from paper_1412_0595_b200 import synscale as S  # noqa: E402
import specs  # noqa: E402

sim = S.Simulation(specs.izh_spec(1000, 100, 2000.0), S.StorageMode.FromSpec,
                   S.EngineOptions(window=256))
sim.step(1024)
sim.sync()
print("ok", sim.steps_done())
