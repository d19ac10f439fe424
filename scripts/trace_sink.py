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
print("steps", int(s.sum()), "spiking rows per step", cnt[s].mean())
stat("step (sink block 0)", tB[s])
stat("sink post update", tA[s])
stat("  chains waiting for staged chunks", rec[s, 2].astype(np.float64) / 1e3)
stat("sink rows", tB[s] - tA[s])
print(f"chain: {cy[s].sum() / cnt[s].sum():.2f} cycles per row")
r = tag == 0x5101
if r.any():
    r0 = (rec[r, 1] & 0xffffffff).astype(np.float64) / 1e3
    r1 = (rec[r, 1] >> 32).astype(np.float64) / 1e3
    r2 = rec[r, 2].astype(np.float64) / 1e3
    r3 = rec[r, 3].astype(np.float64) / 1e3
    stat("round 0 end", r0)
    stat("round 1 end", r1)
    stat("round 2 end", r2)
    stat("round 3 end", r3)
