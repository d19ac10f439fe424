"""Per-kernel device time of config 3 in profile mode (serialised launches)."""
import sys, os
sys.path[:0] = [os.path.dirname(os.path.dirname(os.path.abspath(__file__))), os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests")]
import specs
from paper_1412_0595_b200 import synscale as S
spec = specs.mbody_spec(100000, 0.05, 1000.0)
sim = S.Simulation(spec, S.StorageMode.FromSpec, S.EngineOptions(window=256, profile=True))
sim.step(1024); sim.sync(); sim.reset_kernel_stats()
sim.step(2560); sim.sync()
for n, l, ms in sorted(sim.kernel_stats(), key=lambda x: -x[2]):
    print(f"{n:32s} {l:5d} {ms*1000/l:9.2f} us/launch")
