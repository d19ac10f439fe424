"""Config 3 with KC->DN learning (extension F2): sim/wall of the plastic
network (step mode) next to the static network in step mode and windowed,
plus a per-kernel profile of one learning step."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from paper_1412_0595_b200 import synscale as S  # noqa: E402
import specs  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
runs = [("learning", specs.stdp_mbody_spec(100_000, 1000.0), {}),
        ("static step mode", specs.mbody_spec(100_000, 0.05, 1000.0), {"forceStepMode": True}),
        ("static windowed", specs.mbody_spec(100_000, 0.05, 1000.0), {})]
for name, spec, kw in runs:
    sim = S.Simulation(spec, S.StorageMode.FromSpec, S.EngineOptions(**kw))
    sim.step(500)
    sim.sync()
    t = time.time()
    sim.step(N)
    sim.sync()
    dt = time.time() - t
    print(f"{name:18s} {dt / N * 1e6:8.2f} us/step  ms per simulated second {dt / N * 1e7:9.1f}"
          f"  sim/wall {N / 1e4 / dt:8.3f}  launches/step {sim.kernel_launches() / (N + 500):.1f}",
          flush=True)
    sim.close()
sim = S.Simulation(runs[0][1], S.StorageMode.FromSpec, S.EngineOptions(profile=True))
sim.step(200)
sim.sync()
sim.reset_kernel_stats()
sim.step(500)
sim.sync()
print("-- learning run, per step (us), profile mode (serialised launches):")
for name, n, ms in sorted(sim.kernel_stats(), key=lambda x: -x[2]):
    print(f"   {name:34s} {ms / n * 1000:9.2f}  x{n / 500:.0f}")
