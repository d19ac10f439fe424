"""Per-launch timeline of config 3 windows (diagnostic): SSB_TIMELINE mode
(no graphs, the normal multi-stream schedule, events around every launch)."""
import collections
import os
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
path = os.path.join(tempfile.mkdtemp(), "tl.txt")
os.environ["SSB_TIMELINE"] = path
import specs  # noqa: E402
from paper_1412_0595_b200 import synscale as S  # noqa: E402

W = int(sys.argv[1]) if len(sys.argv) > 1 else 256
dur = (4 + int(os.environ.get("TL_WINDOWS", "8")) + 1) * W * 0.1
emu = int(os.environ.get("TL_EMULATE", "0"))  # one rank of a weak world (graph_scan.py)
if emu > 1:
    os.environ["SSB_EMULATE_EXCHANGE"] = "1"
    spec, mode = specs.mbody_spec(100_000 * emu, 0.05, dur), S.StorageMode.FromSpec
    extra = {"world": emu, "rank": emu // 2}
else:
    spec, mode = specs.config_spec(3, dur)
    split = os.environ.get("TL_SPLIT") == "1"  # exchange path on a one-rank communicator
    extra = {"world": 1, "rank": 0, "commId": S.comm_unique_id()} if split else {}
sim = S.Simulation(spec, mode, S.EngineOptions(window=W, **extra))
sim.step(W * 4)
sim.sync()
open(path, "w").close()
sim.step(W * int(os.environ.get("TL_WINDOWS", "8")))
sim.sync()
sim.kernel_stats()  # harvest
rows = [l.split() for l in open(path)]
rows = [(n, float(a), float(b)) for n, a, b in rows]
t0 = min(r[1] for r in rows)
rows = [(n, a - t0, b - t0) for n, a, b in rows]
span = max(r[2] for r in rows)
nw = int(os.environ.get("TL_WINDOWS", "8"))
print(f"{len(rows)} launches, {span:.1f} us for {nw} windows -> {span / nw:.1f} us/window, "
      f"{span / nw / W * 1e3:.1f} ns/step")
for n, a, b in sorted(rows, key=lambda r: r[1])[:int(os.environ.get("TL_ROWS", "40"))]:
    print(f"{n:28s} {a:9.1f} {b:9.1f} {b - a:8.1f}")
