"""Phases of the single-block population kernels (LHI, DN) from the SSB_TRACE device trace."""
import os, sys, tempfile
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
path = os.path.join(tempfile.mkdtemp(), "trace.bin")
os.environ["SSB_TRACE"] = path
import specs
from paper_1412_0595_b200 import synscale as S
spec, mode = specs.config_spec(3, 60 * 25.6)
sim = S.Simulation(spec, mode, S.EngineOptions(window=256, profile=True))
sim.step(256 * 20); sim.sync(); sim.close()
rec = np.fromfile(path, dtype=np.uint64).reshape(-1, 4)
tag = rec[:, 0]; t0 = rec[:, 2].astype(np.int64); t1 = rec[:, 3].astype(np.int64)
for n, nm in ((20, "lhi"), (100, "dn")):
    i = np.where(tag == n)[0]
    a = np.where(tag == 0xfffffff0)[0]; b = np.where(tag == 0xfffffff1)[0]
    # records are appended start(tag n) then tA then tB by thread 0 in order
    print(nm, "kernel total us median", np.median((t1[i] - t0[i]) / 1e3))
# pair the 3 records per single-block launch: (n, start,end) , (f0, tA, x), (f1, tB, x)
rows = [(int(tag[k]), t0[k], t1[k]) for k in range(len(tag))]
out = {20: [], 100: []}
for k in range(len(rows) - 2):
    if rows[k][0] in out and rows[k + 1][0] == 0xfffffff0 and rows[k + 2][0] == 0xfffffff1:
        st, en = rows[k][1], rows[k][2]
        ta, tb = rows[k + 1][1], rows[k + 2][1]
        out[rows[k][0]].append(((ta - st) / 1e3, (tb - ta) / 1e3, (en - tb) / 1e3))
for n, v in out.items():
    if v:
        v = np.array(v)
        print(n, "staging %.1f us, window loop %.1f us, tail %.1f us" % tuple(np.median(v, axis=0)))
