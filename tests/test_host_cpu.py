"""Host-side library tests that need no GPU: the C ABI surface, RNG streams,
connectivity generation (vs the reference's golden fixtures), spec
validation and builders, the occupancy model, and the no-CPU-fallback rule."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

import specs
from paper_1412_0595_b200 import _lib as L
from paper_1412_0595_b200 import synscale as S

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "synscale_b200.h")


def header_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"SSB_API\s+[\w\s\*]+?\b(ssb_\w+)\s*\(", text)))


def test_header_declares_and_library_exports_every_symbol():
    names = header_functions()
    assert len(names) > 50
    out = subprocess.run(["nm", "-D", "--defined-only", L.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    missing = [n for n in names if n not in exported]
    assert not missing, missing
    # every declared entry point has a ctypes signature and resolves
    assert sorted(L.EXPORTED) == names
    for n in names:
        assert getattr(L.lib, n) is not None


def test_library_links_cuda_statically_and_no_torch():
    out = subprocess.run(["ldd", L.LIB_PATH], capture_output=True, text=True).stdout
    assert "libtorch" not in out and "libcudart.so" not in out


def test_no_cpu_fallback_without_gpu():
    if S.device_count() > 0:
        pytest.skip("a GPU is visible")
    spec = specs.mbody_spec(1000, 0.5, 1.0)
    with pytest.raises(S.DeviceError, match="no CUDA device"):
        S.Simulation(spec)
    with pytest.raises(S.DeviceError):
        S.propagate_dense(np.ones((2, 3), np.float32), [0], np.zeros(3, np.float32))


def test_streams_and_seeds_match_reference_golden(golden):
    for key, vals in golden["streams"].items():
        g, e, label = key.split("/", 2)
        assert [str(int(x)) for x in S.stream_u64(int(g), int(e), label, len(vals))] == vals
    for key, val in golden["derive_seed"].items():
        p, label = key.split("/", 1)
        assert str(S.derive_seed(int(p), label)) == val


def test_gen_fixed_outdegree_matches_reference_golden(golden):
    for entry in golden["gen_fixed_outdegree"]:
        npre, npost, k, kind, lo, hi, value, sign, seed = [int(a) if isinstance(a, str) else a
                                                           for a in entry["args"]]
        dist = S.WeightDist("uniform", lo, hi, 0.0) if kind == L.WEIGHT_UNIFORM else \
            S.WeightDist("constant", 0.0, 0.0, value)
        m = S.gen_fixed_outdegree(npre, npost, k, dist, sign, seed)
        assert specs.sha(m) == entry["sha"]
        if "weights" in entry:
            assert m.ravel().view(np.uint32).tolist() == entry["weights"]


GOLDEN_SPECS = {
    "cfg1_1000ms": lambda: specs.config_spec(1, 1000.0),
    "cfg2_100ms": lambda: specs.config_spec(2, 100.0),
    "cfg3_20ms": lambda: specs.config_spec(3, 20.0),
    "cfg1_sparse_300ms": lambda: (specs.config_spec(1, 300.0)[0], S.StorageMode.ForceSparse),
    "cfg2_fromspec_100ms": lambda: (specs.config_spec(2, 100.0)[0], S.StorageMode.FromSpec),
    "chain_100ms": lambda: (specs.chain_spec(100.0), S.StorageMode.FromSpec),
    "recurrent_200ms": lambda: (specs.recurrent_lif_spec(), S.StorageMode.FromSpec),
}


@pytest.mark.parametrize("name", sorted(GOLDEN_SPECS))
def test_engine_connectivity_matches_reference_golden(golden, name):
    """The matrices Simulation uploads equal the reference's byte for byte."""
    spec, mode = GOLDEN_SPECS[name]()
    for gi, g in enumerate(spec.synapses):
        kind, m = S.build_group(spec, gi, mode)
        assert [kind, specs.sha(*(m if kind == "sparse" else (m,)))] == golden["runs"][name][
            "groups"][g.name], g.name


def test_gen_fixed_outdegree_invariants():
    """test_matrix.cpp:167-209."""
    m = S.gen_fixed_outdegree(50, 80, 13, S.WeightDist.uniform(0.0, 0.5), 1, 99)
    assert ((m != 0).sum(axis=1) == 13).all()
    assert (m[m != 0] > 0).all() and (m[m != 0] < 0.5).all()
    full = S.gen_fixed_outdegree(5, 5, 5, S.WeightDist.constant(1.0), 1, 1)
    assert (full == 1).all()
    neg = S.gen_fixed_outdegree(3, 4, 2, S.WeightDist.constant(2.0), -1, 7)
    assert (neg != 0).sum() == 6 and (neg[neg != 0] == -2).all()
    a = S.gen_fixed_outdegree(20, 30, 5, S.WeightDist.uniform(0.0, 1.0), 1, 4)
    b = S.gen_fixed_outdegree(20, 30, 5, S.WeightDist.uniform(0.0, 1.0), 1, 4)
    c = S.gen_fixed_outdegree(20, 30, 5, S.WeightDist.uniform(0.0, 1.0), 1, 5)
    assert np.array_equal(a, b) and not np.array_equal(a, c)
    u = S.WeightDist.uniform(0.0, 1.0)
    for args in ((3, 4, 5, u, 1, 0), (3, 4, 0, u, 1, 0), (0, 4, 1, u, 1, 0), (3, 4, 2, u, 3, 0)):
        with pytest.raises(S.SpecError):
            S.gen_fixed_outdegree(*args)
    for bad in (lambda: S.WeightDist.uniform(1.0, 1.0), lambda: S.WeightDist.uniform(-0.5, 1.0),
                lambda: S.WeightDist.constant(0.0)):
        with pytest.raises(S.SpecError):
            bad()


def test_storage_footprint_formulas():
    """test_matrix.cpp:211-231."""
    assert S.mem_sparse_elements(100000, 1000) == 201000
    assert S.mem_sparse_elements(0, 10) == 10
    assert S.mem_dense_elements(800, 200) == 160000


def test_mbody_builder_structure():
    """test_network.cpp:117-148."""
    gs = {"pn_kc": 1.0, "pn_lhi": 1.0, "lhi_kc": 1.0, "kc_dn": 1.0}
    net = S.build_mbody_net(100, 20, 1000, 100, gs, 42)
    assert [p.name for p in net.populations] == ["pn", "lhi", "kc", "dn"]
    assert net.populations[0].model == S.ModelKind.PoissonSource
    assert all(p.model == S.ModelKind.CondLif for p in net.populations[1:])
    assert [p.seed for p in net.populations] == [1, 2, 3, 4]
    assert [g.name for g in net.synapses] == ["pn_kc", "pn_lhi", "lhi_kc", "kc_dn"]
    pn_kc, pn_lhi, lhi_kc, kc_dn = net.synapses
    assert pn_kc.storage == S.StorageKind.Sparse and pn_kc.outDegree == 500
    assert pn_kc.baseWeight.kind == "uniform"
    assert lhi_kc.sign == S.SynapseSign.Inhibitory and lhi_kc.storage == S.StorageKind.Dense
    assert lhi_kc.outDegree == 1000 and kc_dn.outDegree == 100 and pn_lhi.outDegree == 20
    assert S.validate(net) == []
    with pytest.raises(S.SpecError, match="lhi_kc"):
        S.build_mbody_net(10, 2, 20, 3, {"pn_kc": 1.0, "pn_lhi": 1.0}, 1)
    with pytest.raises(S.SpecError, match="bogus"):
        S.build_mbody_net(10, 2, 20, 3, dict(gs, bogus=2.0), 1)
    with pytest.raises(S.SpecError):
        S.build_mbody_net(0, 2, 20, 3, gs, 1)


def test_izhikevich_builder_and_errors():
    net = S.build_izhikevich_net(100, 10, 0.8, 1.0, 7)
    assert [g.name for g in net.synapses] == ["exc", "inh"]
    assert net.synapses[0].preCount == 80 and net.synapses[1].preOffset == 80
    p = net.populations[0].params
    assert len(p.a) == 100 and 0.02 <= p.a[99] <= 0.1 and p.c[99] == -65.0
    for args in ((10, 11, 0.8, 1.0, 1), (10, 0, 0.8, 1.0, 1), (1, 1, 0.8, 1.0, 1),
                 (10, 5, 0.0, 1.0, 1), (10, 5, 1.0, 1.0, 1), (10, 5, 0.8, -1.0, 1)):
        with pytest.raises(S.SpecError):
            S.build_izhikevich_net(*args)
    S.build_izhikevich_net(10, 5, 0.8, 0.0, 1)


def test_validate_reports_every_problem():
    spec = specs.mbody_spec(1000, 0.5, 10.0)
    spec.dtMs = 0.0
    spec.populations[2].size = 0
    spec.synapses[0].gScale = -1.0
    spec.synapses[1].post = "nowhere"
    fields = [f for f, _ in S.validate(spec)]
    assert "dtMs" in fields and "populations[2].size" in fields
    assert "synapses[0].gScale" in fields and "synapses[1].post" in fields
    with pytest.raises(S.SpecError):
        S.require_valid(spec)


def test_occupancy_worked_examples():
    """test_occupancy.cpp:60-142."""
    cc30 = S.device_preset("cc30")
    r = S.occupancy(cc30, 256, 32, 0)
    assert (r.warpsPerBlock, r.limitWarps, r.limitBlocks, r.limitRegs) == (8, 8, 16, 8)
    assert (r.activeBlocks, r.activeWarps, r.occupancy) == (8, 64, 1.0)
    assert sorted(r.limiters) == ["registers", "warps"]
    r = S.occupancy(cc30, 256, 64, 0)
    assert (r.limitRegs, r.activeWarps, r.occupancy, r.limiters) == (4, 32, 0.5, ["registers"])
    r = S.occupancy(cc30, 32, 8, 0)
    assert (r.limitBlocks, r.limitRegs, r.activeWarps, r.limiters) == (16, 256, 16, ["blocks"])
    assert S.occupancy(cc30, 33, 0, 0).warpsPerBlock == 2
    r = S.occupancy(cc30, 33, 32, 0)
    assert (r.limitWarps, r.limitRegs) == (32, 32)
    assert [S.occupancy(cc30, 256, 0, s).limitShared for s in (1, 256, 257, 3000, 49152)] == \
        [192, 192, 96, 16, 1]
    r = S.occupancy(cc30, 256, 0, 49153)
    assert (r.limitShared, r.activeBlocks, r.occupancy, r.limiters) == (0, 0, 0.0, ["shared"])
    r = S.occupancy(cc30, 1024, 128, 0)
    assert (r.limitRegs, r.occupancy, r.limiters) == (0, 0.0, ["registers"])
    for bad in ((0, 0, 0), (-32, 0, 0), (1025, 0, 0), (256, -1, 0), (256, 0, -1)):
        with pytest.raises(S.SpecError):
            S.occupancy(cc30, *bad)
    broken = S.device_preset("cc30")
    broken.warpSize = 0
    with pytest.raises(S.SpecError):
        S.occupancy(broken, 256, 0, 0)


def _brute(dev, t, regs, shared):
    wpb = -(-t // dev.warpSize)
    sh = 0 if shared == 0 else -(-shared // dev.sharedAllocUnit) * dev.sharedAllocUnit
    rg = 0 if regs == 0 else -(-regs * dev.warpSize // dev.regAllocUnit) * dev.regAllocUnit * wpb
    for b in range(dev.maxBlocksPerSM, -1, -1):
        if b * wpb <= dev.maxWarpsPerSM and b * sh <= dev.sharedMemPerSM and b * rg <= dev.regsPerSM:
            return b
    return 0


def test_occupancy_matches_brute_force_and_recommend_is_optimal():
    """test_occupancy.cpp:160-235, including the sm100 (B200) preset."""
    assert S.device_preset_names() == ["cc20", "cc30", "cc50"]  # as the reference lists them
    rng = np.random.default_rng(0xacc)
    for name in S.device_preset_names() + ["sm100"]:
        dev = S.device_preset(name)
        for _ in range(300):
            t = int(rng.integers(1, dev.maxThreadsPerBlock + 1))
            regs, shared = int(rng.integers(0, 256)), int(rng.integers(0, 65537))
            assert S.occupancy(dev, t, regs, shared).activeBlocks == _brute(dev, t, regs, shared)
        for regs in (0, 16, 40, 64):
            for shared in (0, 2048, 32768):
                size, res = S.recommend_block_size(dev, regs, shared)
                for t in range(dev.warpSize, dev.maxThreadsPerBlock + 1, dev.warpSize):
                    r = S.occupancy(dev, t, regs, shared)
                    assert r.activeWarps <= res.activeWarps
                    if r.activeWarps == res.activeWarps:
                        assert t <= size
    size, res = S.recommend_block_size(S.device_preset("cc30"), 32, 0)
    assert (size, res.occupancy) == (1024, 1.0)
    sm100 = S.device_preset("sm100")
    assert (sm100.maxWarpsPerSM, sm100.maxBlocksPerSM, sm100.sharedMemPerSM) == (64, 32, 233472)
    with pytest.raises(S.SpecError, match="cc30"):
        S.device_preset("cc99")
    tiny = S.device_preset("cc30")
    tiny.maxThreadsPerBlock = 16
    with pytest.raises(S.SpecError):
        S.recommend_block_size(tiny, 0, 0)


def test_raster_csv_and_avg_spike():
    """io.cpp:276-287 and test_engine.cpp:520-538."""
    r = S.Raster([("a", 2), ("b", 3)], np.array([0, 3, 5, 9, 9], np.int64),
                 np.array([0, 0, 0, 0, 1], np.int32), np.array([0, 1, 0, 0, 2], np.int32))
    assert S.raster_to_csv(r).splitlines()[:2] == ["step,population,neuron", "0,a,0"]
    assert S.avg_spike(r, "a", 1000.0) == 2.0
    assert abs(S.avg_spike(r, "b", 500.0) - 1.0 / 1.5) < 1e-12
    for bad in (("missing", 1000.0), ("a", 0.0), ("a", -5.0)):
        with pytest.raises(S.SpecError):
            S.avg_spike(r, *bad)


def _sweep_builder(n, g):
    import specs
    spec = specs.mbody_spec(1000, 0.5, 20.0)
    pk = spec.synapses[spec.group_index("pn_kc")]
    pk.outDegree = n
    pk.gScale = g
    if n == 13:
        raise ValueError("builder refuses 13")
    return spec


def test_sweep_grid_validation_and_failure_rows():
    """sweep (calibration.cpp:16-86) host logic: argument errors raise; the grid
    collapses duplicates and sorts; a failing builder or run is recorded in its
    row (here every run fails without a GPU, like a run that throws)."""
    with pytest.raises(S.SpecError):
        S.sweep(_sweep_builder, S.SweepRequest([], [1.0], "kc"))
    with pytest.raises(S.SpecError):
        S.sweep(_sweep_builder, S.SweepRequest([10], [], "kc"))
    with pytest.raises(S.SpecError):
        S.sweep(_sweep_builder, S.SweepRequest([10], [1.0], ""))
    with pytest.raises(S.SpecError):
        S.sweep(_sweep_builder, S.SweepRequest([10], [float("inf")], "kc"))
    if S.device_count() > 0:
        return
    seen = []
    rows = S.sweep(_sweep_builder, S.SweepRequest([20, 13, 20], [2.0, 1.0], "kc",
                                                 onCell=lambda r, d, t: seen.append((d, t))))
    assert [(r.nConn, r.gScale) for r in rows] == [(13, 1.0), (13, 2.0), (20, 1.0), (20, 2.0)]
    assert all(r.failed and r.sumNaNs == -1 and np.isnan(r.avgSpike) for r in rows)
    assert "13" in rows[0].error and "device" in rows[2].error.lower()
    assert seen == [(1, 4), (2, 4), (3, 4), (4, 4)]


def test_storage_mode_auto_follows_density():
    """StorageMode.Auto (extension): dense iff outDegree / nPost >= the threshold
    (0.25 by default), the reference's own storage flag otherwise ignored."""
    t = S.auto_dense_threshold()
    assert 0.0 < t <= 1.0
    for frac in (0.001, 0.05, 0.2, 0.25, 0.5, 1.0):
        spec = specs.mbody_spec(4000, frac, 5.0)
        for g in spec.synapses:
            post = spec.populations[spec.pop_index(g.post)]
            kind, m = S.build_group(spec, g.name, S.StorageMode.Auto)
            assert kind == ("dense" if g.outDegree >= t * post.size else "sparse"), (frac, g.name)
            # same matrix as the explicit modes
            ref = S.build_group(spec, g.name, S.StorageMode.ForceDense if kind == "dense"
                                else S.StorageMode.ForceSparse)[1]
            if kind == "dense":
                assert np.array_equal(m, ref)
            else:
                assert all(np.array_equal(a, b) for a, b in zip(m, ref))
