"""Per-kernel times (profile mode) of one shard of a virtual split world (config 3)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import specs  # noqa: E402
from paper_1412_0595_b200 import synscale as S  # noqa: E402

world = int(sys.argv[1]) if len(sys.argv) > 1 else 8
spec, mode = specs.config_spec(3, 1024 * 0.1 * 3)
sim = S.Simulation(spec, mode, S.EngineOptions(window=256, virtualWorld=world, profile=True))
sim.step(256)
sim.sync()
sim.reset_kernel_stats()
sim.step(512)
sim.sync()
for n, k, ms in sorted(sim.kernel_stats(), key=lambda x: -x[2]):
    print(f"{n:28s} {ms / k * 1e3:9.1f} us/launch")
