"""Scratch: isolate timing differences between harnesses (duration, torch events, L2 flush)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch  # noqa: E402
from paper_1412_0595_b200 import synscale as S  # noqa: E402
import specs  # noqa: E402


def run(total_s, use_torch_events, flush, label):
    spec, mode = specs.config_spec(3, total_s * 1000.0)
    sim = S.Simulation(spec, mode, S.EngineOptions(window=256))
    stream = torch.cuda.ExternalStream(sim.stream())
    buf = torch.empty(64 * 1024 * 1024, device="cuda") if flush else None
    sim.step(10000)
    sim.sync()
    times = []
    for _ in range(3):
        if buf is not None:
            buf.zero_()
            torch.cuda.synchronize()
        if use_torch_events:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            sim.step(10000)
            e1.record(stream)
            e1.synchronize()
            times.append(e0.elapsed_time(e1) / 1e3)
        else:
            t = time.perf_counter()
            sim.step(10000)
            sim.sync()
            times.append(time.perf_counter() - t)
    print(f"{label:40s} " + " ".join(f"{x * 1e3:7.1f}ms" for x in times), flush=True)
    sim.close()


run(4.2, False, False, "4.2 s run, wall")
run(9.0, False, False, "9 s run, wall")
run(9.0, True, False, "9 s run, torch events")
run(9.0, True, True, "9 s run, torch events + L2 flush")

import bench  # noqa: E402
cs = bench.ClockSampler(0)
cs.start()
run(9.0, True, True, "9 s run, + nvidia-smi sampler")
print(cs.stop())
import pynvml  # noqa: E402
import threading  # noqa: E402
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
stop = threading.Event()
samples = []


def poll():
    while not stop.is_set():
        samples.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                        pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)))
        stop.wait(0.2)


th = threading.Thread(target=poll, daemon=True)
th.start()
run(9.0, True, True, "9 s run, + NVML sampler")
stop.set()
th.join()
print(samples[:5])
