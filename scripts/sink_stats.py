"""DN spike statistics of the learning run: DN spikes per step and the sink
kernel's events (steps with a spike in a 32-column block) per window."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
from paper_1412_0595_b200 import synscale as S  # noqa: E402
import specs  # noqa: E402

spec = specs.stdp_mbody_spec(100_000, 1000.0)
sim = S.Simulation(spec, S.StorageMode.FromSpec, S.EngineOptions(window=256))
sim.step(10000)
res = sim.finish()
R = res.raster
names = [p for p, _ in R.populations]
for pi, name in enumerate(names):
    sel = R.population == pi
    print(name, "spikes", int(sel.sum()), "per step", sel.sum() / 10000)
dn = names.index("DN")
sel = R.population == dn
st, nr = R.step[sel], R.neuron[sel]
for w0 in range(0, 10000, 2560):
    m = (st >= w0) & (st < w0 + 256)
    ev = {(int(s), int(n) // 32) for s, n in zip(st[m], nr[m])}
    print("window at", w0, "dn spikes", int(m.sum()), "events per block",
          [sum(1 for e in ev if e[1] == b) for b in range(4)])
