"""Per-block device trace of config 3 in graph mode (diagnostic, SSB_TRACE):
KC update launches (131 blocks each), their block start spread, the gaps
between consecutive KC launches and what ran in them.

    python scripts/trace_kc.py [windows]
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

nwin = int(sys.argv[1]) if len(sys.argv) > 1 else 32
emu = int(os.environ.get("TR_EMULATE", "0"))
if emu > 1:
    os.environ["SSB_EMULATE_EXCHANGE"] = "1"
    spec, mode = specs.mbody_spec(100_000 * emu, 0.05, (nwin + 40) * 25.6), S.StorageMode.FromSpec
    sim = S.Simulation(spec, mode, S.EngineOptions(window=256, world=emu, rank=emu // 2,
                                                   rasterLocal=True))
else:
    spec, mode = specs.config_spec(3, (nwin + 40) * 25.6)
    sim = S.Simulation(spec, mode, S.EngineOptions(window=256))
sim.step(256 * 32)
sim.sync()
sim.step(256 * nwin)
sim.sync()
sim.close()
rec = np.fromfile(path, dtype=np.uint64).reshape(-1, 4)
tag, blk, t0, t1 = rec[:, 0], rec[:, 1], rec[:, 2].astype(np.int64), rec[:, 3].astype(np.int64)
base = t0.min()
t0, t1 = (t0 - base) / 1e3, (t1 - base) / 1e3  # us
nkc = 100_000 * max(1, emu) // max(1, emu) if emu <= 1 else None
kc_tag = max(int(x) for x in set(tag.tolist()) if x < 0xfffffff0)
names = {kc_tag: "kc", 20: "lhi", 100: "dn", 0xffffffff: "kc_dn", 0xfffffffc: "kc_dn(tma)", 0xfffffffd: "raster"}
if emu > 1:
    names[16] = "dn (local slice)"
# the last nwin windows' KC launches: split KC blocks into launches by start gaps
k = np.where(tag == kc_tag)[0]
order = k[np.argsort(t0[k])]
starts = t0[order]
cut = np.where(np.diff(starts) > 20.0)[0] + 1
launches = np.split(order, cut)[-nwin:]
print(f"{len(launches)} KC launches (tag {kc_tag}), blocks/launch {len(launches[-1])}")
prev_end = None
rows = []
for L in launches:
    s0, s1 = t0[L].min(), t0[L].max()
    e1 = t1[L].max()
    rows.append((s0, s1, e1))
for i, (s0, s1, e1) in enumerate(rows[:-1]):
    nxt = rows[i + 1][0]
    print(f"KC[{i:2d}] start {s0:9.1f} last-block-start +{s1 - s0:6.1f} end +{e1 - s0:6.1f}  "
          f"gap to next {nxt - e1:6.1f} us")
dur = np.array([r[2] - r[0] for r in rows])
per = np.diff([r[0] for r in rows])
print(f"KC duration median {np.median(dur):.1f} us, launch period median {np.median(per):.1f} us")
for tg, nm in names.items():
    m = tag == tg
    if m.any():
        d = t1[m] - t0[m]
        print(f"{nm:6s} blocks {m.sum():7d} block-duration median {np.median(d):7.1f} us  p90 {np.percentile(d, 90):7.1f}")

# what occupied SMs while the last KC blocks waited: other blocks running at
# the moment each late KC block started
late = []
for L in launches[2:]:
    s0 = t0[L].min()
    for i in L:
        if t0[i] - s0 > 5.0:
            late.append(t0[i])
if late:
    other = tag != kc_tag
    cnt = {nm: 0 for nm in names.values()}
    for x in late:
        m = other & (t0 < x) & (t1 > x - 1.0)
        for tg in set(tag[m].tolist()):
            nm = names.get(tg, f"pop of {tg}")
            cnt[nm] = cnt.get(nm, 0) + 1
    print(f"{len(late)} KC blocks started >5 us late; blocks of other kernels ending at that moment:", cnt)
