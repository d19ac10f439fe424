"""The reference's acceptance network (1000 Izhikevich neurons, nConn = 100,
recurrent; acceptance_main.cpp:38, 139-163) on the device: us per step with
the one-block window kernel (default) and in step mode (SSB_CYCLIC_BLOCK=0)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
from paper_1412_0595_b200 import synscale as S  # noqa: E402
import specs  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
for mode in (S.StorageMode.FromSpec, S.StorageMode.ForceDense):
    spec = specs.izh_spec(1000, 100, duration_ms=(N + 2000) * 1.0)
    sim = S.Simulation(spec, mode, S.EngineOptions(window=256))
    sim.step(1000)
    sim.sync()
    t = time.time()
    sim.step(N)
    sim.sync()
    dt = time.time() - t
    print(f"izh 1000/100 {mode.name:10s} step_mode={sim.step_mode() if hasattr(sim, 'step_mode') else '?'}"
          f"  {dt / N * 1e6:8.2f} us/step  launches/step {sim.kernel_launches() / (N + 1000):.2f}",
          flush=True)
    sim.close()
spec = specs.izh_spec(1000, 100, duration_ms=4000.0)
sim = S.Simulation(spec, S.StorageMode.FromSpec, S.EngineOptions(window=256, profile=True))
sim.step(512)
sim.sync()
sim.reset_kernel_stats()
sim.step(2560)
sim.sync()
print("-- per step (us), profile mode (serialised launches):")
for name, n, ms in sorted(sim.kernel_stats(), key=lambda x: -x[2]):
    print(f"   {name:34s} {ms / 2560 * 1000:9.2f}  x{n}")
sim.close()
