"""Measurement sweeps of SURVEY.md §8(d) (BASELINE configs 3 and 5), one JSON line each.

    python scripts/sweeps.py density   # kernel level: propagate dense vs CRS, all 100 rows spiking
    python scripts/sweeps.py model     # config 5: 100k KC at pn_kc density f, ForceSparse vs ForceDense
    python scripts/sweeps.py blocks    # config 3: occupancy-chosen vs swept KC block sizes

Device times are CUDA events on the launching stream after warm-up; the
density sweep reports the kernel's algorithmic bytes / time against the
measured HBM peak (MEASURED_PEAKS.json).
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

FRACS = (0.001, 0.005, 0.01, 0.05, 0.1, 0.25, 0.5)


def peak_gbs():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"])
    return 6651.0


def density():
    import torch
    from paper_1412_0595_b200 import synscale as S
    from paper_1412_0595_b200._lib import lib
    n_pre, n_post, tile = 100, 100_000, 256
    peak = peak_gbs()
    stream = torch.cuda.current_stream()
    sp = stream.cuda_stream
    spikes = torch.arange(n_pre, dtype=torch.int32, device="cuda")
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")

    def timed(fn, prep, reps=20):
        for _ in range(3):
            prep()
            fn()
        ts = []
        for _ in range(reps):
            prep()
            # inputs cold in L2: read 256 MB (a read leaves clean lines, a
            # write-flush would make the timed kernel pay for write-backs);
            # it also keeps the GPU busy while the host enqueues the launch
            flush.sum(dtype=torch.float32)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn()
            e1.record(stream)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1) / 1e3)
        return float(np.median(ts))

    for frac in FRACS:
        k = max(1, int(round(frac * n_post)))
        w = S.gen_fixed_outdegree(n_pre, n_post, k, S.WeightDist.uniform(0.0, 0.02), 1, 1234)
        rows, cols = np.nonzero(w)
        vals = w[rows, cols].astype(np.float32)
        rs = np.zeros(n_pre + 1, np.int64)
        np.add.at(rs, rows + 1, 1)
        rs = np.cumsum(rs)
        dw = torch.from_numpy(w).cuda()
        dg = torch.from_numpy(vals).cuda()
        di = torch.from_numpy(cols.astype(np.int32)).cuda()
        drs = torch.from_numpy(rs).cuda()
        n_tiles = (n_post + tile - 1) // tile
        seg = torch.empty(n_pre * (n_tiles + 1), dtype=torch.int32, device="cuda")
        lib.ssb_crs_segments_dev(di.data_ptr(), drs.data_ptr(), n_pre, n_post, tile,
                                 seg.data_ptr(), sp)
        acc_d = torch.zeros(n_post, dtype=torch.float32, device="cuda")
        acc_s = torch.zeros(n_post, dtype=torch.float32, device="cuda")
        acc_c = torch.zeros(n_post, dtype=torch.float32, device="cuda")
        # column-sliced layout (ssb_crs_slices, host), then device copies
        import ctypes as C
        n_sl = (n_post + 31) // 32
        off = np.zeros(n_sl + 1, np.int64)
        need = C.c_int64()
        err = C.create_string_buffer(256)
        cols32 = np.ascontiguousarray(cols.astype(np.int32))
        lib.ssb_crs_slices(vals.ctypes.data, cols32.ctypes.data, rs.ctypes.data, n_pre, n_post,
                           off.ctypes.data, None, None, 0, C.byref(need), err, len(err))
        srows = np.empty(need.value, np.int32)
        svals = np.empty(need.value, np.float32)
        lib.ssb_crs_slices(vals.ctypes.data, cols32.ctypes.data, rs.ctypes.data, n_pre, n_post,
                           off.ctypes.data, srows.ctypes.data, svals.ctypes.data, need.value,
                           C.byref(need), err, len(err))
        d_sr = torch.from_numpy(srows).cuda()
        d_sv = torch.from_numpy(svals).cuda()
        d_so = torch.from_numpy(off).cuda()

        def dense():
            lib.ssb_propagate_dense_dev(dw.data_ptr(), n_pre, n_post, spikes.data_ptr(), n_pre,
                                        acc_d.data_ptr(), sp)

        def sparse():
            lib.ssb_propagate_crs_dev(dg.data_ptr(), di.data_ptr(), seg.data_ptr(), tile, n_pre,
                                      n_post, spikes.data_ptr(), n_pre, acc_s.data_ptr(), sp)

        def sliced():
            lib.ssb_propagate_crs_sliced_dev(d_sr.data_ptr(), d_sv.data_ptr(), d_so.data_ptr(),
                                             n_pre, n_post, spikes.data_ptr(), n_pre,
                                             acc_c.data_ptr(), sp)

        td, ts = timed(dense, acc_d.zero_), timed(sparse, acc_s.zero_)
        tc = timed(sliced, acc_c.zero_)
        # parity: both kernels against the reference fold (rows ascending)
        ref = np.zeros(n_post, np.float32)
        for r in range(n_pre):
            ref += w[r]
        same = bool(np.array_equal(acc_d.cpu().numpy(), ref) and
                    np.array_equal(acc_s.cpu().numpy(), ref) and
                    np.array_equal(acc_c.cpu().numpy(), ref))
        nnz = int(len(vals))
        bd = n_pre * n_post * 4 + n_post * 8      # every weight once + acc read/write
        bs = nnz * 8 + n_pre * (n_tiles + 1) * 4 + n_post * 8
        bc = int(need.value) * 8 + (n_sl + 1) * 8 + n_post * 8  # slices once + acc
        for kind, t, b in (("dense", td, bd), ("sparse", ts, bs), ("sparse_sliced", tc, bc)):
            print(json.dumps({"sweep": "density_kernel", "frac": frac, "kernel": kind,
                              "nnz": nnz, "us": round(t * 1e6, 2),
                              "synaptic_events_per_s": nnz / t, "algorithmic_bytes": b,
                              "achieved_gbs": round(b / t / 1e9, 1), "peak_gbs": peak,
                              "frac_of_peak": round(b / t / 1e9 / peak, 3),
                              "bit_exact_vs_fold": same}), flush=True)


def model(profile=False):
    import specs
    from paper_1412_0595_b200 import synscale as S
    import torch
    n_kc, secs = 100_000, 0.2
    for frac in (0.001, 0.01, 0.05, 0.1, 0.25, 0.5):
        spec = specs.mbody_spec(n_kc, frac, secs * 1000.0 + 30.0)
        for mode in (S.StorageMode.ForceSparse, S.StorageMode.ForceDense, S.StorageMode.Auto):
            sim = S.Simulation(spec, mode, S.EngineOptions(window=256))
            sim.step(256)
            sim.sync()
            c0 = sim.spike_counts()
            stream = torch.cuda.ExternalStream(sim.stream())
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            steps = int(secs * 10_000)
            e0.record(stream)
            sim.step(steps)
            e1.record(stream)
            e1.synchronize()
            t = e0.elapsed_time(e1) / 1e3
            d = sim.spike_counts() - c0
            idx = {p.name: i for i, p in enumerate(spec.populations)}
            ev = sum(int(d[idx[g.pre]]) * g.outDegree for g in spec.synapses)
            layout = "dense" if sim.group_dense("pn_kc") is not None else "sparse"
            print(json.dumps({"sweep": "density_model", "frac": frac, "mode": mode.name,
                              "pn_kc_layout": layout,
                              "us_per_step": round(t / steps * 1e6, 3),
                              "sim_wall": round(secs / t, 2), "synaptic_events_per_s": ev / t,
                              "kc_rate_hz": float(d[idx["kc"]]) / n_kc / secs}), flush=True)
            sim.close()


def modelprof():
    """Per-kernel time per window of config 5 (frac 0.01) in both storage modes."""
    import specs
    from paper_1412_0595_b200 import synscale as S
    spec = specs.mbody_spec(100_000, 0.01, 100.0)
    for mode in (S.StorageMode.ForceSparse, S.StorageMode.ForceDense):
        sim = S.Simulation(spec, mode, S.EngineOptions(window=256, profile=True))
        sim.step(256)
        sim.sync()
        sim.reset_kernel_stats()
        sim.step(512)
        sim.sync()
        print(json.dumps({"sweep": "density_model_profile", "mode": mode.name,
                          "us_per_window": {n: round(ms / k * 1e3, 1)
                                            for n, k, ms in sim.kernel_stats()}}), flush=True)
        sim.close()


def blocks():
    import specs
    from paper_1412_0595_b200 import synscale as S
    import torch
    spec, mode = specs.config_spec(3, 260.0)
    runs = [("occupancy (default: model + wave quantisation)", {}),
            ("paper occupancy model as is", {"blockPolicy": 1})]
    runs += [(f"swept {bs}", {"blockSize": bs}) for bs in (128, 256, 384, 512, 640, 704, 768,
                                                             896, 1024)]
    for label, kw in runs:
        try:
            sim = S.Simulation(spec, mode, S.EngineOptions(window=256, **kw))
        except Exception as exc:  # a plan that does not fit the SM
            print(json.dumps({"sweep": "blocks", "policy": label, "error": str(exc)}), flush=True)
            continue
        sim.step(256)
        sim.sync()
        stream = torch.cuda.ExternalStream(sim.stream())
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        sim.step(2304)
        e1.record(stream)
        e1.synchronize()
        t = e0.elapsed_time(e1) / 1e3
        print(json.dumps({"sweep": "blocks", "policy": label, "kc_block": sim.block_size("kc"),
                          "us_per_step": round(t / 2304 * 1e6, 3)}), flush=True)
        sim.close()


if __name__ == "__main__":
    what = sys.argv[1:] or ["density", "model", "blocks"]
    for w in what:
        {"density": density, "model": model, "modelprof": modelprof, "blocks": blocks}[w]()
