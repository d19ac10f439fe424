"""µs per window vs windows per graph launch (config 3, W = 256), steps a multiple of
256 x M so every launch is a full M-window graph."""
import os
import subprocess
import sys

if len(sys.argv) > 1:  # child: one M
    ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
    import torch
    import specs
    from paper_1412_0595_b200 import synscale as S
    M = int(sys.argv[1])
    n = 256 * 64
    spec, mode = specs.config_spec(3, (n * 2 + 512) * 0.1)
    split = os.environ.get("GS_SPLIT") == "1"  # the exchange path on a one-rank communicator
    sim = S.Simulation(spec, mode, S.EngineOptions(
        window=256, blockSize=int(os.environ.get("GS_BS", "0")),
        **({"world": 1, "rank": 0, "commId": S.comm_unique_id()} if split else {})))
    sim.step(n)
    sim.sync()
    st = torch.cuda.ExternalStream(sim.stream())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    sim.step(n)
    e1.record(st)
    e1.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"M={M:2d} kc_block={sim.block_size('kc')}: {ms * 1e3 / 64:7.1f} us/window, "
          f"{ms * 1e3 / n:6.3f} us/step", flush=True)
else:
    for M in ([int(x) for x in os.environ["GS_M"].split(",")] if "GS_M" in os.environ
              else (1, 2, 4, 8, 16)):
        env = dict(os.environ, SSB_GRAPH_WINDOWS=str(M))
        subprocess.run([sys.executable, __file__, str(M)], env=env)
