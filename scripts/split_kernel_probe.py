"""Per-kernel times (profile mode) of the shards of a virtual split world.

    python scripts/split_kernel_probe.py 8          # config 3 (100k KC) cut 8 ways
    python scripts/split_kernel_probe.py 8 weak     # bench's weak split: 8 x 100k KC
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import specs  # noqa: E402
from paper_1412_0595_b200 import synscale as S  # noqa: E402

world = int(sys.argv[1]) if len(sys.argv) > 1 else 8
if len(sys.argv) > 2 and sys.argv[2] == "weak":
    spec, mode = specs.mbody_spec(100_000 * world, 0.05, 1024 * 0.1 * 3), S.StorageMode.FromSpec
else:
    spec, mode = specs.config_spec(3, 1024 * 0.1 * 3)
sim = S.Simulation(spec, mode, S.EngineOptions(window=256, virtualWorld=world, profile=True))
sim.step(256)
sim.sync()
sim.reset_kernel_stats()
sim.step(512)
sim.sync()
print(f"world {world} {sys.argv[2:]}: per-shard launch times (shards run one after another)")
for n, k, ms in sorted(sim.kernel_stats(), key=lambda x: -x[2]):
    print(f"{n:28s} {ms / k * 1e3:9.1f} us/launch")
c = sim.spike_counts()
steps = 256 + 512
print("spikes/step: " + ", ".join(f"{p.name} {int(c[i]) / steps:.0f}"
                                 for i, p in enumerate(spec.populations)))
