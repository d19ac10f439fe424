"""Per-step phase timestamps of the plastic sink's producers (thread 32 of
sink block 0; SSB_TRACE): staged, post spikes out, learned, next rows
fetched, background in, barrier passed -- ns from the iteration's start."""
import os
import sys
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
path = os.path.join(tempfile.mkdtemp(), "trace.bin")
os.environ["SSB_TRACE"] = path
import specs  # noqa: E402
from paper_1412_0595_b200 import synscale as S  # noqa: E402

sim = S.Simulation(specs.stdp_mbody_spec(100_000, 1000.0), S.StorageMode.FromSpec,
                   S.EngineOptions(window=256))
sim.step(256 * 4)
sim.sync()
sim.step(256 * 8)
sim.sync()
sim.close()
rec = np.fromfile(path, dtype=np.uint64).reshape(-1, 4)
rec = rec[(rec[:, 0] & 0xffffffff) == 0x5200]
t0 = rec[:, 1].astype(np.int64)
per = np.diff(np.sort(t0)) / 1e3
per = per[(per > 0) & (per < 200)]
f = lambda x, sh: ((x >> sh) & 0xffff).astype(np.float64) / 1e3
cols = [("staged", f(rec[:, 2], 0)), ("post spikes out", f(rec[:, 2], 16)), ("learned", f(rec[:, 2], 32)),
        ("next rows fetched", f(rec[:, 2], 48)), ("background in", f(rec[:, 3], 0)),
        ("barrier passed", f(rec[:, 3], 16))]
print("iterations", len(rec), f"period p50 {np.median(per):.3f} us mean {per.mean():.3f}")
for name, d in cols:
    print(f"  {name:20s} p50 {np.median(d):7.3f} us  mean {d.mean():7.3f}  p90 {np.percentile(d, 90):7.3f}")
