import sys, time, os
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import numpy as np
from paper_1412_0595_b200 import synscale as S
import specs
for cfg, dur in ((1, 1000.0), (2, 1000.0), (3, 1000.0)):
    spec, mode = specs.config_spec(cfg, dur + 200.0)
    for W in (1, 64, 256):
        t0 = time.time(); sim = S.Simulation(spec, mode, S.EngineOptions(window=W)); tb = time.time() - t0
        sim.step(1000); sim.sync()
        t = time.time(); sim.step(10000); sim.sync(); dt = time.time() - t
        print(f"cfg{cfg} W={W} build {tb:.2f}s  1s sim in {dt*1e3:.1f} ms -> sim/wall {1.0/dt:.1f}  us/step {dt/10000*1e6:.2f}", flush=True)
        sim.close()
spec, mode = specs.config_spec(3, 300.0)
sim = S.Simulation(spec, mode, S.EngineOptions(window=64, profile=True))
sim.step(2000); sim.sync()
for k in sorted(sim.kernel_stats(), key=lambda x: -x[2]): print(k)
