#!/usr/bin/env python
"""Benchmark of the mushroom-body step path (BASELINE.json metric: synaptic
events/s and simulated-time / wall-time ratio).

One bench "step" = one simulated second (10,000 steps of 0.1 ms) of the
BASELINE config 3 network (100 PN / 20 LHI / 100,000 KC / 100 DN, pn_kc CRS
at 5 %, lhi_kc / kc_dn / pn_lhi dense; gScales of SURVEY.md §8(d)), continuing
one Simulation.  `value` = synaptic events / device-timed second with all
inputs resident in HBM (CUDA events on the engine's stream, L2 flushed
between steps); `e2e` = the same metric through the public C ABI with host
buffers: spec -> ssb_create (connectivity generated on the host, uploaded)
-> 1 s of steps -> ssb_finish (raster read back to the host).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

N > 1 (torchrun), default --scaling split: weak scaling of ONE network split
over the N GPUs: N x 100,000 KC (gScales per SURVEY.md §8(d):
kc_dn = 30 / nKC), KC and DN split by neuron ranges, PN / LHI replicated, each
window's KC / DN spike bitmasks all-gathered over NCCL; value = the network's
synaptic events / (max over ranks of device time).  At N = 1 this is config 3
exactly.  --scaling replicas runs independent config-3 networks instead (the
reference's own parallelism, calibration.cpp:76-84), and is the fallback when
the split run cannot start.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

DT_MS = 0.1
STEPS_PER_SIM_SECOND = 10_000
N_KC, FRAC = 100_000, 0.05
METRIC = "synaptic events/sec (mushroom body, 100k KC, dt 0.1 ms)"
UNIT = "syn_events/s"


def workload_config(window=None):
    cfg = {"workload": "mbody config 3: 100 PN / 20 LHI / 100000 KC / 100 DN, pn_kc CRS 5%, "
                       "lhi_kc+kc_dn+pn_lhi dense, dt 0.1 ms, 1 s simulated per step",
           "n_pn": 100, "n_lhi": 20, "n_kc": N_KC, "n_dn": 100, "pn_kc_out_fraction": FRAC,
           "storage": "FromSpec", "seed": 7,
           "gscales": {"pn_kc": 0.5 / FRAC, "pn_lhi": 1.0, "lhi_kc": 0.1, "kc_dn": 30.0 / N_KC}}
    if window is not None:
        cfg["window_steps"] = window
    return cfg


def scaling_config(mode, world, fallback=None):
    if mode == "split":
        return {"parallelism": f"split{world}", "n_kc_total": N_KC * world,
                "split": "KC and DN by neuron ranges, PN/LHI replicated, per-window NCCL "
                         "all-gather of spike bitmasks; each rank records its own neurons' "
                         "spikes (rank 0 also PN/LHI), events summed over ranks"}
    if mode == "replicas":
        cfg = {"parallelism": f"replicas{world}", "replicas": world}
        if fallback:
            cfg["split_failed"] = fallback
        return cfg
    return {"parallelism": "single"}


def make_spec(seconds: float, seed: int = 7):
    import specs
    return specs.mbody_spec(N_KC, FRAC, seconds * 1000.0, seed=seed)


def synaptic_events(spec, counts_per_pop):
    """Σ_groups (spikes of the pre population) × outDegree."""
    idx = {p.name: i for i, p in enumerate(spec.populations)}
    return int(sum(int(counts_per_pop[idx[g.pre]]) * g.outDegree for g in spec.synapses))


def algorithmic_bytes(spec, counts_per_pop, steps):
    """40 B per CondLif neuron-step + 8 B per sparse and 4 B
    per dense synaptic event + 4 B per spike index written."""
    idx = {p.name: i for i, p in enumerate(spec.populations)}
    b = 0
    for p in spec.populations:
        if p.model == 2:  # CondLif
            b += 40 * p.size * steps
        b += 4 * int(counts_per_pop[idx[p.name]])
    for g in spec.synapses:
        ev = int(counts_per_pop[idx[g.pre]]) * g.outDegree
        b += (4 if g.storage == 0 else 8) * ev
    return b


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

    def __init__(self, index: int = 0):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def start(self):
        try:  # NVML: ~10 ms sampling, so even a short timed region gets many samples
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            reasons = getattr(pynvml, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                pynvml.nvmlDeviceGetCurrentClocksThrottleReasons
            bits = [(0x8, "hw_slowdown"), (0x40, "hw_thermal_slowdown"),
                    (0x20, "sw_thermal_slowdown"), (0x4, "sw_power_cap")]

            def sample():
                r = reasons(h)
                return [str(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)), str(mx), "",
                        ""] + ["Active" if r & b else "Not Active" for b, _ in bits]
            sample()
            period = 0.01
        except Exception:
            q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

            def sample():
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                return [x.strip() for x in out.split(",")] if out else None
            period = 0.2

        def run():
            while not self._stop.is_set():
                try:
                    v = sample()
                    if v:
                        self.samples.append(v)
                except Exception:
                    pass
                self._stop.wait(period)
        self._t = threading.Thread(target=run, daemon=True)
        self._t.start()

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 4 + i and s[4 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def flush_l2(torch, buf):
    buf.zero_()  # 256 MiB write > 126 MB L2


def roofline_pass(S, torch, spec, window):
    """Profiled pass (CUDA events around every launch, no graphs): per-kernel
    time; algorithmic bytes of the dominant kernel per launch."""
    sim = S.Simulation(spec, S.StorageMode.FromSpec, S.EngineOptions(window=window, profile=True))
    sim.step(window * 4)  # warm-up
    sim.sync()
    sim.reset_kernel_stats()
    c0 = sim.spike_counts()
    steps = STEPS_PER_SIM_SECOND // 4
    sim.step(steps)
    sim.sync()
    c1 = sim.spike_counts()
    stats = sorted(sim.kernel_stats(), key=lambda s: -s[2])
    d = c1 - c0
    idx = {p.name: i for i, p in enumerate(spec.populations)}
    name, launches, ms = stats[0]
    kind, _, obj = name.partition(":")
    # algorithmic bytes of the dominant kernel over the pass
    if kind == "condlif_window":
        p = spec.populations[idx[obj]]
        byts = 40 * p.size * steps + 4 * int(d[idx[obj]])
        for g in spec.synapses:
            if g.post == obj and g.pre != "kc":  # inline groups (kc_dn is buffered)
                byts += (4 if g.storage == 0 else 8) * int(d[idx[g.pre]]) * g.outDegree
        unit_desc = f"40 B x {p.size} neurons x {steps} steps + inline synaptic events"
    elif kind in ("dense_window", "dense_deliver"):
        g = spec.synapses[spec.group_index(obj)]
        byts = 4 * int(d[idx[g.pre]]) * g.outDegree
        unit_desc = f"4 B x {g.pre} spikes x {g.outDegree} posts"
    else:
        byts = algorithmic_bytes(spec, d, steps)
        unit_desc = "whole-step formula"
    total_ms = sum(s[2] for s in stats)
    sim.close()
    return {"kernel": name, "launches": launches, "ms_total": ms, "share_of_step": ms / total_ms,
            "bytes_total": byts, "bytes_per_launch": byts / launches,
            "avg_launch_ms": ms / launches, "unit": unit_desc,
            "kernels": [{"name": n, "launches": l, "ms": round(m, 4)} for n, l, m in stats]}


def cpu_reference(seconds_sample: float, replicas: int):
    """The reference's own CPU engine (oracle/_ref, compiled from /root/reference)
    on a bounded sample of the same workload: `replicas` concurrent
    Simulations (calibration.cpp's parallelism model), wall time of the
    stepping phase.  Returns (events/s aggregate, sample description)."""
    from oracle import oracle as O
    from paper_1412_0595_b200 import synscale as S
    spec = make_spec(seconds_sample)
    desc = S.NetDesc(spec)
    steps = int(round(seconds_sample * STEPS_PER_SIM_SECOND))
    # events of the sample, from one reference run's raster
    sim = O.CpuSim(desc.ptr, spec, 0, ref=True)
    t0 = time.perf_counter()
    sim.step(steps)
    t1 = time.perf_counter()
    step, pop, neu = sim.finish()
    counts = np.bincount(pop, minlength=len(spec.populations))
    ev = synaptic_events(spec, counts)
    single = ev / (t1 - t0)
    if replicas > 1:
        wall, _ = O.ref_time_steps(desc.ptr, 0, steps, replicas)
        agg = ev * replicas / wall
    else:
        agg = single
    return agg, single, ev, t1 - t0


def run_reference_arm(args, rank, world):
    if rank != 0:
        return
    from oracle import oracle as O
    if not O.have_ref():
        O.build()
    cores = os.cpu_count() or 1
    sample_s = 0.02  # 20 ms simulated (200 steps) per replica per bench step
    vals = []
    for i in range(args.warmup + args.steps):
        agg, single, ev, t = cpu_reference(sample_s, cores)
        if i >= args.warmup:
            vals.append(agg)
    v = statistics.median(vals)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": workload_config(),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "reference",
                             "sample": f"{cores} concurrent reference Simulations x "
                                       f"{int(sample_s * 1e4)} steps ({sample_s * 1e3:.0f} ms "
                                       "simulated) of config 3 per bench step"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--window", type=int, default=256)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--scaling", default="split", choices=["split", "replicas"])
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        return run_reference_arm(args, rank, world)

    import torch
    from paper_1412_0595_b200 import synscale as S

    dist = None
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = local if world > 1 else 0
    torch.cuda.set_device(dev)

    total_s = args.warmup + args.steps + 1
    mode = args.scaling if world > 1 else "single"
    fallback = None

    def start(mode):
        """(spec, sim) of this rank; the split mode builds the same N x 100k
        network on every rank and the engine keeps this rank's part."""
        import specs
        if mode == "split":
            spec = specs.mbody_spec(N_KC * world, FRAC, total_s * 1000.0, seed=7)
            cid = [S.comm_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(cid, src=0)
            # each rank records its own neurons (rank 0 also PN / LHI): the
            # raster and the spike counts are the sums over ranks
            opts = S.EngineOptions(device=dev, window=args.window, world=world, rank=rank,
                                   commId=cid[0], rasterLocal=True)
        else:
            spec = make_spec(total_s, seed=7 + rank)
            opts = S.EngineOptions(device=dev, window=args.window)
        sim = S.Simulation(spec, S.StorageMode.FromSpec, opts)
        sim.step(STEPS_PER_SIM_SECOND)  # first warm-up step
        sim.sync()
        return spec, sim

    t0 = time.perf_counter()
    if mode == "split":
        err, spec, sim = "", None, None
        try:
            spec, sim = start("split")
        except Exception as exc:  # noqa: BLE001 -- reported in the JSON line
            err = f"{type(exc).__name__}: {exc}"
        bad = torch.tensor([1.0 if err else 0.0], device=f"cuda:{dev}")
        dist.all_reduce(bad, op=dist.ReduceOp.MAX)
        if bad.item() > 0:
            if sim is not None:
                sim.close()
            fallback = err or "another rank failed"
            mode = "replicas"
    if mode != "split":
        spec, sim = start(mode)
    build_s = time.perf_counter() - t0
    stream = torch.cuda.ExternalStream(sim.stream(), device=dev)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=f"cuda:{dev}")

    for _ in range(args.warmup - 1):
        sim.step(STEPS_PER_SIM_SECOND)
    sim.sync()

    c_before = sim.spike_counts()
    l_before = sim.kernel_launches()
    clocks = ClockSampler(dev)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    times = []
    for _ in range(args.steps):
        flush_l2(torch, flush)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        sim.step(STEPS_PER_SIM_SECOND)
        e1.record(stream)
        e1.synchronize()
        times.append(e0.elapsed_time(e1) / 1000.0)
    torch.cuda.synchronize()
    clk = clocks.stop()
    if dist:
        dist.barrier()
    c_after = sim.spike_counts()
    launches = sim.kernel_launches() - l_before
    t_local = sum(times)
    ev_local = synaptic_events(spec, c_after - c_before)

    t_max, ev_sum = t_local, ev_local
    if dist:
        tt = torch.tensor([t_local], device=f"cuda:{dev}", dtype=torch.float64)
        ee = torch.tensor([ev_local], device=f"cuda:{dev}", dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        # replicas: independent networks; split: each rank counted its own
        # neurons' spikes (local raster) -- either way the sum over ranks
        dist.all_reduce(ee, op=dist.ReduceOp.SUM)
        t_max, ev_sum = float(tt.item()), float(ee.item())
    value = ev_sum / t_max
    sim_seconds = args.steps
    ms_per_step = t_max / args.steps * 1000.0
    sim.close()

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return

    # -- e2e through the public C ABI with host buffers (rank 0, 1 s per step).
    # Same scope as the reference arm (which times Simulation::step, not the
    # constructor): ssb_step(10,000) per bench step with that step's raster
    # moved into host memory (ssb_raster_drain_async hands it to the copier so
    # the next step computes meanwhile; a final ssb_raster_drain waits); wall clock.  The network is uploaded once
    # at construction (like the reference, untimed) and the Poisson drive is
    # the model's own RNG stream advanced on the device (part of the step), so
    # no per-step host input exists: h2d_bytes_per_step = 0.  For reference,
    # e2e.with_build adds construction (host connectivity build + upload) and
    # ssb_finish of a fresh 1 s run.
    e2e = None
    if not args.no_e2e:
        k_e2e = 4
        spec_e = make_spec(k_e2e + 1.0, seed=11)
        # 512 MB of pinned host memory for the raster drains (allocated at
        # construction, untimed): each step's ~59 MB copies straight into it
        sim_e = S.Simulation(spec_e, S.StorageMode.FromSpec,
                             S.EngineOptions(device=dev, window=args.window, rasterPinnedMB=512))
        sim_e.step(STEPS_PER_SIM_SECOND)
        held = sim_e.drain_raster()
        c0 = sim_e.spike_counts()
        # each step's raster is handed to the background copier as soon as the
        # step is done; the next step computes while it drains; the timed
        # region ends when the last step's events are in host memory
        t0 = time.perf_counter()
        for _ in range(k_e2e):
            sim_e.step(STEPS_PER_SIM_SECOND)
            sim_e.drain_raster(wait=False)
        n = sim_e.drain_raster()
        t1 = time.perf_counter()
        vals = [synaptic_events(spec_e, sim_e.spike_counts() - c0) / (t1 - t0)]
        d2h = [4 * (n - held) / k_e2e]
        sim_e.close()
        wb = []
        for i in range(2):
            spec1 = make_spec(1.0, seed=11 + i)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            sim1 = S.Simulation(spec1, S.StorageMode.FromSpec,
                                S.EngineOptions(device=dev, window=args.window))
            r = sim1.finish()
            t1 = time.perf_counter()
            counts = np.array([np.count_nonzero(r.raster.population == k)
                               for k in range(len(spec1.populations))])
            wb.append(synaptic_events(spec1, counts) / (t1 - t0))
            sim1.close()
        e2e = {"value": statistics.median(vals), "unit": UNIT, "h2d_bytes_per_step": 0,
               "d2h_bytes_per_step": int(statistics.median(d2h)),
               "what": "4 bench steps of ssb_step(10,000), each step's raster events moved "
                       "to host memory (ssb_raster_drain_async into the engine's pinned "
                       "raster pool, overlapping the next step; the final ssb_raster_drain "
                       "inside the timed region), wall clock; network uploaded and pool "
                       "pinned once at construction (untimed, as in the reference arm)",
               "with_build": {"value": max(wb), "what": "ssb_create (host build + upload) + "
                              "10,000 steps + ssb_finish, wall clock, best of 2"}}

    # -- roofline of the dominant kernel (profiled pass)
    peaks_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    peak, peak_src = 6651.0, "fallback (B200_PROFILING.md)"
    if os.path.exists(peaks_path):
        with open(peaks_path) as f:
            peak = float(json.load(f)["hbm_gbs"])
        peak_src = "measured (MEASURED_PEAKS.json hbm_gbs)"
    rf = roofline_pass(S, torch, make_spec(1.0), args.window)
    achieved = rf["bytes_per_launch"] / (rf["avg_launch_ms"] / 1000.0) / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as f:
            per = json.load(f).get("bytes_per_launch", {})
        kname = rf["kernel"].split(":")[0]
        traffic = per.get(kname, per.get(kname + "_kernel"))
    roofline = {"bound": "hbm", "achieved": round(achieved, 2), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": traffic,
                "kernel": rf["kernel"], "peak_source": peak_src,
                "bytes_per_launch": rf["bytes_per_launch"],
                "avg_launch_us": round(rf["avg_launch_ms"] * 1000.0, 3),
                "share_of_step": round(rf["share_of_step"], 4), "algorithmic": rf["unit"],
                "kernels": rf["kernels"]}

    # -- config 3 with KC->DN learning (extension F2, step mode): a bounded
    # sample of 0.2 simulated seconds, device-timed, reported beside the
    # static headline (BASELINE config 3 names learning)
    learning = None
    if world == 1 and not os.environ.get("SSB_BENCH_NO_LEARNING"):
        import specs
        lspec = specs.stdp_mbody_spec(N_KC, 1000.0)
        lsim = S.Simulation(lspec, S.StorageMode.FromSpec, S.EngineOptions())
        lsim.step(960)
        lsim.sync()
        c0 = lsim.spike_counts().copy()
        l0 = lsim.kernel_launches()
        st = torch.cuda.ExternalStream(lsim.stream())
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        lsim.step(1920)
        e1.record(st)
        lsim.sync()
        lms = e0.elapsed_time(e1)
        lev = synaptic_events(lspec, lsim.spike_counts() - c0)
        learning = {"workload": "config 3 + pair STDP on kc_dn (step mode), 1920 steps "
                                "(0.192 s simulated, 40 graphs of 48 steps) after 960 warm-up steps",
                    "value": lev / (lms / 1e3), "unit": UNIT, "sim_wall": 0.192 / (lms / 1e3),
                    "us_per_timestep": lms * 1e3 / 1920,
                    "gpu_launches": int(lsim.kernel_launches() - l0)}
        lsim.close()

    cpu = None
    if not args.no_cpu_baseline and world == 1:
        try:
            from oracle import oracle as O
            if O.have_ref():
                cores = os.cpu_count() or 1
                agg, single, ev, t = cpu_reference(0.05, cores)
                cpu = {"value": agg, "unit": UNIT, "cores": cores, "kind": "reference",
                       "sample": f"{cores} concurrent reference Simulations x 500 steps "
                                 "(50 ms simulated) of config 3; 1-core value "
                                 f"{single:.4g} ev/s (sim/wall {0.05 / t:.4g})",
                       "value_1core": single, "sim_wall_1core": 0.05 / t}
        except Exception as exc:  # reported, not fatal
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                   "sample": f"failed: {exc}"}

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded build_mbody_net, reference RNG streams)",
            "config": dict(workload_config(args.window), l2="flushed (256 MiB write) between steps",
                           **scaling_config(mode, world, fallback)),
            "sim_wall": sim_seconds / t_max,
            "us_per_timestep": t_max / (sim_seconds * STEPS_PER_SIM_SECOND) * 1e6,
            "build_s": build_s,
            "step_ms": [round(x * 1e3, 3) for x in times],
            "gpu_launches": int(launches), "clocks": clk, "roofline": roofline,
            "cpu_baseline": cpu, "e2e": e2e, "learning": learning}
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
