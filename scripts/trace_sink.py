"""Per-phase device trace of the plastic sink kernel (diagnostic, SSB_TRACE):
learning config 3, block 0 (sink: post update, rows) and the first
background block (potentiation), and the grid barrier wait of each.

    python scripts/trace_sink.py [windows]
"""
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

nwin = int(sys.argv[1]) if len(sys.argv) > 1 else 8
sim = S.Simulation(specs.stdp_mbody_spec(100_000, 1000.0), S.StorageMode.FromSpec,
                   S.EngineOptions(window=256))
sim.step(256 * 4)
sim.sync()
sim.step(256 * nwin)
sim.sync()
sim.close()
rec = np.fromfile(path, dtype=np.uint64).reshape(-1, 4)
tag = rec[:, 0] & 0xffffffff
cnt = (rec[:, 0] >> 32).astype(np.float64)
tA = (rec[:, 1] & 0xffffffff).astype(np.float64) / 1e3
tB = (rec[:, 1] >> 32).astype(np.float64) / 1e3
tS = rec[:, 2].astype(np.float64) / 1e3
cy = rec[:, 3].astype(np.float64)


def stat(name, d):
    print(f"{name:22s} mean {d.mean():7.3f} us  p50 {np.median(d):7.3f}  p90 {np.percentile(d, 90):7.3f}"
          f"  p99 {np.percentile(d, 99):7.3f}")


s = tag == 0x5100
b = tag == 0x5110
print("steps", int(s.sum()), "spiking rows per step", cnt[s].mean())
stat("step (sink block)", tS[s])
stat("sink post update", tA[s])
stat("sink rows", tB[s] - tA[s])
stat("sink barrier", tS[s] - tB[s])
stat("background work", tB[b])
nq = cnt[b]
for lo, hi in [(0, 0), (1, 4), (5, 20), (21, 60), (61, 1000)]:
    m = (nq >= lo) & (nq <= hi)
    if m.any():
        print(f"   post spikes {lo:3d}-{hi:4d}: {m.mean() * 100:5.1f}% of steps, background {tB[b][m].mean():7.3f} us")
stat("background barrier", tS[b] - tB[b])
print(f"chain: {cy[s].sum() / cnt[s].sum():.2f} cycles per row")
