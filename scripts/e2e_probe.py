import sys, time
sys.path[:0] = [".", "tests"]
import specs
from paper_1412_0595_b200 import synscale as S
spec = specs.mbody_spec(100_000, 0.05, 13000.0, seed=11)
import os
sim = S.Simulation(spec, S.StorageMode.FromSpec, S.EngineOptions(window=256, rasterPinnedMB=int(os.environ.get("PIN_MB", "0"))))
sim.step(10000); sim.drain_raster()
for i in range(3):
    t0 = time.perf_counter(); sim.step(10000); sim.sync(); t1 = time.perf_counter()
    n = sim.drain_raster(); t2 = time.perf_counter()
    print(f"step+sync {1e3*(t1-t0):.2f} ms, drain(wait) {1e3*(t2-t1):.2f} ms, events {n}")
t0 = time.perf_counter()
for i in range(4):
    sim.step(10000); sim.drain_raster(wait=False)
n = sim.drain_raster(); t1 = time.perf_counter()
print(f"pipelined 4 steps {1e3*(t1-t0):.2f} ms")
t0 = time.perf_counter()
for i in range(4):
    sim.step(10000)
sim.sync(); t1 = time.perf_counter()
print(f"4 steps no drain {1e3*(t1-t0):.2f} ms")
