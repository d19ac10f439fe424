"""Scratch timing: sim/wall per config and window, plus a per-kernel profile."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from paper_1412_0595_b200 import synscale as S  # noqa: E402
import specs  # noqa: E402

cfgs = [int(c) for c in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["1", "2", "3"])]
windows = [int(w) for w in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["64", "256"])]
for cfg in cfgs:
    spec, mode = specs.config_spec(cfg, 1200.0)
    for W in windows:
        t0 = time.time()
        sim = S.Simulation(spec, mode, S.EngineOptions(window=W))
        tb = time.time() - t0
        sim.step(1000)
        sim.sync()
        t = time.time()
        sim.step(10000)
        sim.sync()
        dt = time.time() - t
        print(f"cfg{cfg} W={W} build {tb:.2f}s  1s sim in {dt * 1e3:.1f} ms -> sim/wall "
              f"{1.0 / dt:.1f}  us/step {dt / 10000 * 1e6:.2f}  blocks "
              f"{[sim.block_size(p.name) for p in spec.populations]}", flush=True)
        sim.close()
for W in windows:
    spec, mode = specs.config_spec(3, 300.0)
    sim = S.Simulation(spec, mode, S.EngineOptions(window=W, profile=True))
    sim.step(W * 2)
    sim.sync()
    sim.reset_kernel_stats()
    sim.step(W * 8)
    sim.sync()
    print(f"-- profile W={W}, per window (us):")
    for name, n, ms in sorted(sim.kernel_stats(), key=lambda x: -x[2]):
        print(f"   {name:28s} {ms / n * 1000:9.1f}")
