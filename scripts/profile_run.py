"""Short fixed workload for ncu: config 3 (100k KC), a few launch windows.

    ncu --set full -k regex:condlif -s 20 -c 3 python scripts/profile_run.py
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from paper_1412_0595_b200 import synscale as S  # noqa: E402
import specs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", type=int, default=3)
ap.add_argument("--window", type=int, default=256)
ap.add_argument("--windows", type=int, default=8)
ap.add_argument("--graphs", type=int, default=1)
args = ap.parse_args()

spec, mode = specs.config_spec(args.cfg, (args.windows + 1) * args.window * 0.1)
sim = S.Simulation(spec, mode, S.EngineOptions(window=args.window, useGraphs=bool(args.graphs)))
sim.step(args.windows * args.window)
sim.sync()
print("ok", sim.steps_done(), sim.spike_counts().tolist(),
      {p.name: sim.block_size(p.name) for p in spec.populations})
