"""Per-kernel times (profile mode, one stream) of one rank of the weak split
world of R (bench.py --gpus R: R x 100k KC) with the all-gather emulated
(SSB_EMULATE_EXCHANGE, see graph_scan.py).   python scripts/emu_probe.py 8"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
os.environ["SSB_EMULATE_EXCHANGE"] = "1"
import specs  # noqa: E402
from paper_1412_0595_b200 import synscale as S  # noqa: E402

R = int(sys.argv[1]) if len(sys.argv) > 1 else 8
spec = specs.mbody_spec(100_000 * R, 0.05, 300.0)
sim = S.Simulation(spec, S.StorageMode.FromSpec,
                   S.EngineOptions(window=256, world=R, rank=R // 2, profile=True,
                                   rasterLocal=os.environ.get("EMU_LOCAL", "1") == "1"))
sim.step(256)
sim.sync()
sim.reset_kernel_stats()
sim.step(1024)
sim.sync()
print(f"emulated rank {R // 2} of {R}: per-kernel us/launch (profile mode, one stream)")
for n, k, ms in sorted(sim.kernel_stats(), key=lambda x: -x[2]):
    print(f"{n:28s} {ms / k * 1e3:9.1f}")
