"""Config 4 (1M KC) on one GPU: steady-state ms per simulated second and the
per-kernel profile of a few windows (BASELINE config 4's one-GPU point)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import torch  # noqa: E402
import specs  # noqa: E402
from paper_1412_0595_b200 import synscale as S  # noqa: E402

spec, mode = specs.config_spec(4, 3100.0)
t0 = time.perf_counter()
sim = S.Simulation(spec, mode, S.EngineOptions(window=256))
print(f"build {time.perf_counter() - t0:.2f} s, KC block {sim.block_size('kc')}", flush=True)
sim.step(10000)
sim.sync()
c0 = sim.spike_counts()
st = torch.cuda.ExternalStream(sim.stream())
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
sim.step(20000)
e1.record(st)
e1.synchronize()
ms = e0.elapsed_time(e1) / 2
d = sim.spike_counts() - c0
idx = {p.name: i for i, p in enumerate(spec.populations)}
ev = sum(int(d[idx[g.pre]]) * g.outDegree for g in spec.synapses) / 2
print(f"config 4: {ms:.2f} ms per simulated second, sim/wall {1000 / ms:.2f}, "
      f"{ev / (ms / 1000):.3g} synaptic events/s, KC {d[idx['kc']] / 2 / 1e6:.3g} M spikes/s")
sim.close()
sim = S.Simulation(spec, mode, S.EngineOptions(window=256, profile=True))
sim.step(512)
sim.sync()
sim.reset_kernel_stats()
sim.step(1024)
sim.sync()
print("per-kernel us per 256-step window (profile mode, one stream):")
for n, k, msk in sorted(sim.kernel_stats(), key=lambda x: -x[2]):
    print(f"  {n:28s} {msk / k * 1e3:9.1f}")
