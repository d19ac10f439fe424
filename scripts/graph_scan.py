"""µs per window vs windows per graph launch (config 3, W = 256), steps a multiple of
256 x M so every launch is a full M-window graph.

GS_SPLIT=1: the exchange path on a one-rank communicator.
GS_EMULATE=R: one rank of bench.py's weak split world of R (R x 100k KC, this
rank's 100k) with the all-gather emulated by copies (SSB_EMULATE_EXCHANGE:
the rank's real work, meaningless dynamics) -- weak scaling on one GPU.
"""
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
    emu = int(os.environ.get("GS_EMULATE", "0"))
    if emu > 1:
        os.environ["SSB_EMULATE_EXCHANGE"] = "1"
        spec, mode = specs.mbody_spec(100_000 * emu, 0.05, (n * 2 + 512) * 0.1), S.StorageMode.FromSpec
        extra = {"world": emu, "rank": emu // 2, "rasterLocal": os.environ.get("GS_LOCAL", "1") == "1"}
    else:
        spec, mode = specs.config_spec(3, (n * 2 + 512) * 0.1)
        split = os.environ.get("GS_SPLIT") == "1"
        extra = {"world": 1, "rank": 0, "commId": S.comm_unique_id()} if split else {}
    sim = S.Simulation(spec, mode, S.EngineOptions(
        window=256, blockSize=int(os.environ.get("GS_BS", "0")), **extra))
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
