"""Short config-3 run for ncu source captures of the KC pair kernel."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
from paper_1412_0595_b200 import synscale as S  # noqa: E402
import specs  # noqa: E402

spec, mode = specs.config_spec(3, 200.0)
sim = S.Simulation(spec, mode, S.EngineOptions(window=256))
sim.step(1024)
sim.sync()
print("ok")
