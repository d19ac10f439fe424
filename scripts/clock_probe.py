"""Diagnostic: SM clock, power and clock-event reasons sampled (NVML) while config 3 runs 16 windows."""
import os, sys, threading, time, subprocess
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path[:0] = [ROOT, ROOT + "/tests"]
import torch, pynvml, specs
from paper_1412_0595_b200 import synscale as S
pynvml.nvmlInit(); h = pynvml.nvmlDeviceGetHandleByIndex(0)
samples=[]; stop=False
def run():
    while not stop:
        samples.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM), pynvml.nvmlDeviceGetPowerUsage(h)/1000.0, pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)))
        time.sleep(0.005)
spec, mode = specs.config_spec(3, 3000.0)
sim = S.Simulation(spec, mode, S.EngineOptions(window=256))
sim.step(4096); sim.sync()
t = threading.Thread(target=run, daemon=True); t.start()
t0=time.time(); sim.step(4096*4); sim.sync(); dt=time.time()-t0
stop=True; t.join()
import statistics
print("wall", dt, "us/step", dt/16384*1e6)
print("sm clk median", statistics.median(s[0] for s in samples), "min", min(s[0] for s in samples), "power median", statistics.median(s[1] for s in samples), "reasons", sorted(set(s[2] for s in samples)))
