"""Soak run of the plastic sink (config 3 + STDP), progress printed per
simulated 0.1 s (diagnostic; SSB_SINK_WATCH=1 prints the kernel roles'
progress from a host thread)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
from paper_1412_0595_b200 import synscale as S  # noqa: E402
import specs  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
sim = S.Simulation(specs.stdp_mbody_spec(100_000, n * 0.1 + 10), S.StorageMode.FromSpec,
                   S.EngineOptions(window=256))
t = time.time()
done = 0
while done < n:
    k = min(1000, n - done)
    sim.step(k)
    sim.sync()
    done += k
    print(f"{done} steps, {(time.time() - t) / done * 1e6:.2f} us/step", flush=True)
