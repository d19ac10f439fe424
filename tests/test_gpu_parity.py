"""Parity of the CUDA path (through the C ABI) with the reference.

Bar: bit-exact.  Rasters, spike counts and every fp32 state array (v, gExc,
gInh, excIn, inhIn) must equal the reference's bit for bit (NaN payloads
excepted: any NaN equals any NaN), because the kernels evaluate the
reference's float expressions in the same order with no FMA contraction and
sum synaptic inputs in the reference's order.  Checked against
the golden fixtures (generated from the reference) and against the oracle on
the same seeded inputs, at window sizes 1 (per-step launches) and >1 (fused
windows), in all storage modes.
"""
import os

import numpy as np
import pytest

import specs
from paper_1412_0595_b200 import synscale as S

pytestmark = pytest.mark.gpu

FIELDS = ("v", "gExc", "gInh", "excIn", "inhIn", "nanFlag")


def gpu_sim(spec, mode=S.StorageMode.FromSpec, **kw):
    return S.Simulation(spec, mode, S.EngineOptions(**kw))


def cpu_sim(O, spec, mode=S.StorageMode.FromSpec):
    d = S.NetDesc(spec)
    sim = O.CpuSim(d.ptr, spec, int(mode))
    sim._desc = d
    return sim


def assert_state_equal(g, o, spec, where=""):
    for pi, p in enumerate(spec.populations):
        for f in FIELDS:
            a, b = g.pull(pi, f), o.state(pi, f)
            if p.model == S.ModelKind.PoissonSource and f in ("v", "gExc", "gInh"):
                continue
            assert specs.bits_equal(a, b), f"{where} {p.name}.{f}"
        assert int(g.pull(pi, "flagged")[0]) == int(o.state(pi, "flagged")[0]), where


GOLDEN = {
    "cfg1_1000ms": lambda: specs.config_spec(1, 1000.0),
    "cfg2_100ms": lambda: specs.config_spec(2, 100.0),
    "cfg3_20ms": lambda: specs.config_spec(3, 20.0),
    "cfg1_sparse_300ms": lambda: (specs.config_spec(1, 300.0)[0], S.StorageMode.ForceSparse),
    "cfg2_fromspec_100ms": lambda: (specs.config_spec(2, 100.0)[0], S.StorageMode.FromSpec),
    "chain_100ms": lambda: (specs.chain_spec(100.0), S.StorageMode.FromSpec),
    "recurrent_200ms": lambda: (specs.recurrent_lif_spec(), S.StorageMode.FromSpec),
    "izh_1000_1000ms": lambda: (specs.izh_spec(), S.StorageMode.FromSpec),
    "izh_1000_dense_300ms": lambda: (specs.izh_spec(duration_ms=300.0), S.StorageMode.ForceDense),
    "izh_ff_200ms": lambda: (specs.izh_ff_spec(), S.StorageMode.FromSpec),
}


@pytest.mark.parametrize("window", [1, 7, 64])
@pytest.mark.parametrize("name", sorted(GOLDEN))
def test_runs_match_reference_golden(golden, name, window):
    spec, mode = GOLDEN[name]()
    g = golden["runs"][name]
    sim = gpu_sim(spec, mode, window=window)
    r = sim.finish()
    assert len(r.raster) == g["n_events"]
    assert specs.sha(r.raster.step, r.raster.population, r.raster.neuron) == g["raster_sha"]
    assert [r.avgSpike[p.name] for p in spec.populations] == g["rates"]
    assert r.sumNaNs == g["sum_nans"]
    for pi, p in enumerate(spec.populations):
        for f, h in g["state_sha"][p.name].items():
            if p.model == S.ModelKind.PoissonSource and f in ("v", "gExc", "gInh"):
                continue
            assert specs.sha(sim.pull(pi, f)) == h, (p.name, f)


def test_izhikevich_kat_per_step():
    """test_engine.cpp:79-111 on the device: per-step bitwise v / u of one
    bias-driven Izhikevich neuron (the noise stream is drawn, times 0)."""
    kat = np.load(os.path.join(os.path.dirname(__file__), "golden", "izh_kat.npz"))
    spec = specs.single_izh_spec()
    sim = gpu_sim(spec)
    for t in range(sim.steps_total()):
        sim.step(1)
        assert sim.pull(0, "v")[0] == kat["v"][t] and sim.pull(0, "u")[0] == kat["u"][t], t
    r = sim.finish()
    assert np.array_equal(r.raster.step, kat["step"]) and len(kat["step"]) > 0


@pytest.mark.parametrize("window", [1, 64])
def test_izhikevich_noise_stream_matches_oracle(oracle_mod, window):
    """Noisy Izhikevich inputs (Gaussian pairs straddling steps, odd sizes),
    stepwise state against the oracle."""
    spec = specs.izh_ff_spec(60.0)
    g = gpu_sim(spec, window=window)
    o = cpu_sim(oracle_mod, spec)
    for t in range(0, 120, 40):
        g.step(40)
        o.step(40)
        for pi, p in enumerate(spec.populations):
            fields = ("v", "u", "excIn", "inhIn") if p.model == S.ModelKind.Izhikevich else \
                (("v", "gExc", "gInh", "excIn", "inhIn") if p.model == S.ModelKind.CondLif else ())
            for f in fields:
                assert specs.bits_equal(g.pull(pi, f), o.state(pi, f)), (t, p.name, f)


def test_condlif_kat_per_step():
    """test_engine.cpp:183-290 on the device: per-step bitwise v/gExc/gInh."""
    kat = np.load(os.path.join(os.path.dirname(__file__), "golden", "condlif_kat.npz"))
    spec = specs.condlif_kat_spec()
    sim = gpu_sim(spec)
    for t in range(sim.steps_total()):
        sim.step(1)
        assert sim.pull(2, "v")[0].view(np.uint32) == kat["v"][t].view(np.uint32), t
        assert sim.pull(2, "gExc")[0].view(np.uint32) == kat["gExc"][t].view(np.uint32), t
        assert sim.pull(2, "gInh")[0].view(np.uint32) == kat["gInh"][t].view(np.uint32), t
    r = sim.finish()
    assert np.array_equal(r.raster.step, kat["step"])
    assert np.array_equal(r.raster.neuron, kat["neuron"])


@pytest.mark.parametrize("mode", [0, 1, 2])
def test_stepwise_state_matches_oracle(oracle_mod, mode):
    """Every state array after every call, with irregular call sizes so
    windows start and end at arbitrary steps."""
    spec = specs.mbody_spec(3000, 0.1, 40.0)
    g = gpu_sim(spec, S.StorageMode(mode), window=16)
    o = cpu_sim(oracle_mod, spec, S.StorageMode(mode))
    for n in [1, 1, 2, 3, 5, 8, 13, 21, 34, 55, 57, 100, 100]:
        g.step(n)
        o.step(n)
        assert_state_equal(g, o, spec, f"after {o.steps_done()} steps")
    rg, ro = g.finish(), o.finish()
    assert np.array_equal(rg.raster.step, ro[0]) and np.array_equal(rg.raster.neuron, ro[2])
    assert np.array_equal(rg.raster.population, ro[1])


@pytest.mark.parametrize("heavy", [8, 4096])
@pytest.mark.parametrize("block", [0, 64, 1024])
def test_chain_paths_match_oracle(oracle_mod, heavy, block):
    """Two groups on one accumulator (fold order), a pre window, a Poisson
    target, buffered (heavy=8) and inline (heavy=4096) input paths, and
    different post tile sizes."""
    spec = specs.chain_spec(40.0)
    g = gpu_sim(spec, window=11, heavyPreThreshold=heavy, blockSize=block)
    o = cpu_sim(oracle_mod, spec)
    for n in (1, 10, 11, 12, 33, 93):
        g.step(n)
        o.step(n)
        assert_state_equal(g, o, spec, f"step {o.steps_done()}")
    rg, ro = g.finish(), o.finish()
    assert np.array_equal(rg.raster.neuron, ro[2]) and np.array_equal(rg.raster.step, ro[0])


@pytest.mark.parametrize("graph_windows", ["1", "2", "4"])
def test_raster_flushes_and_multiwindow_graphs(oracle_mod, monkeypatch, graph_windows):
    """A minimal raster arena forces many background flushes (arena switches)
    while multi-window graphs overlap populations; the raster must still be
    the reference's, in order."""
    monkeypatch.setenv("SSB_GRAPH_WINDOWS", graph_windows)
    spec = specs.chain_spec(100.0)
    g = gpu_sim(spec, window=9, rasterCapacity=1)
    rg = g.finish()
    o = cpu_sim(oracle_mod, spec)
    ro = o.finish()
    assert len(rg.raster) == len(ro[0]) > 100_000
    assert np.array_equal(rg.raster.step, ro[0]) and np.array_equal(rg.raster.neuron, ro[2])
    assert np.array_equal(rg.raster.population, ro[1])


def test_fault_injection_spreads_like_reference(oracle_mod):
    """test_engine.cpp:402-434: a poisoned state written between steps."""
    spec = specs.mbody_spec(1000, 0.5, 5.0)
    for grp in spec.synapses:
        grp.gScale = 1e30
    g = gpu_sim(spec, window=8)
    o = cpu_sim(oracle_mod, spec)
    g.step(3)
    o.step(3)
    v = o.state(2, "v")
    v[3] = 1e30
    g.push(2, "v", v)
    o.set_state(2, "v", v)
    acc = o.state(3, "excIn")
    acc[7] = 5.0
    g.push(3, "excIn", acc)
    o.set_state(3, "excIn", acc)
    g.step(1)
    o.step(1)
    assert_state_equal(g, o, spec, "after injection")
    rg, ro = g.finish(), o.finish()
    assert np.array_equal(rg.raster.neuron, ro[2])
    assert rg.sumNaNs == o.sum_nans() and rg.sumNaNs > 0


def test_division_edge_numerators_rerun_exactly(oracle_mod):
    """The window kernels divide (eLeak - v) / tauM without a branch and rerun a
    chunk exactly when a numerator left the fast path's range: tiny, huge,
    infinite and NaN numerators written into a population's v (eLeak = 0, so
    v = 1e-35 gives a subnormal-range numerator) match the oracle step by step."""
    spec = specs.mbody_spec(1000, 0.5, 6.0)
    kc = spec.populations[spec.pop_index("kc")]
    kc.params.eLeakMV = 0.0
    kc.params.vResetMV = 0.0
    kc.params.vThreshMV = 15.0
    kc.params.eExcMV = 60.0
    for window in (1, 16):
        g = gpu_sim(spec, window=window)
        o = cpu_sim(oracle_mod, spec)
        g.step(5)
        o.step(5)
        v = o.state(2, "v")
        v[0], v[1], v[2], v[3], v[40] = 1e-35, -3e-38, 1e36, np.inf, np.nan
        g.push(2, "v", v)
        o.set_state(2, "v", v)
        for k in range(6):
            g.step(3)
            o.step(3)
            assert_state_equal(g, o, spec, f"window {window} after {5 + 3 * (k + 1)} steps")
        rg, ro = g.finish(), o.finish()
        assert np.array_equal(rg.raster.neuron, ro[2])


def test_storage_modes_and_windows_do_not_change_results():
    """test_engine.cpp:455-474 plus the engine's own window/graph knobs."""
    spec = specs.mbody_spec(2000, 0.2, 200.0)
    ref = None
    for mode in (0, 1, 2):
        for kw in ({"window": 1}, {"window": 64}, {"window": 50, "useGraphs": False},
                   {"forceStepMode": True}):
            r = S.run(spec, S.StorageMode(mode), S.EngineOptions(**kw))
            key = (r.raster.step.tobytes(), r.raster.population.tobytes(),
                   r.raster.neuron.tobytes(), tuple(r.avgSpike.values()))
            if ref is None:
                ref = key
                assert len(r.raster) > 1000
            assert key == ref, (mode, kw)


def test_zero_scaled_groups_are_noops():
    """test_engine.cpp:498-511 (conductance version)."""
    spec = specs.mbody_spec(1000, 0.5, 100.0)
    spec.synapses[3].gScale = 0.0  # kc_dn silent
    a = S.run(spec)
    spec2 = specs.mbody_spec(1000, 0.5, 100.0)
    spec2.synapses = spec2.synapses[:3]
    b = S.run(spec2)
    assert np.array_equal(a.raster.neuron, b.raster.neuron)
    assert a.avgSpike == b.avgSpike and a.avgSpike["dn"] == 0.0


def test_poisson_rate_and_stream():
    """test_engine.cpp:540-556: 1000 sources at 50 Hz within 5%, bit-exact raster."""
    spec = S.NetworkSpec(dtMs=1.0, durationMs=10000.0, globalSeed=77)
    spec.populations = [S.NeuronPopulation("src", 1000, S.ModelKind.PoissonSource, 1,
                                           S.PoissonParams(50.0))]
    r = S.run(spec)
    assert abs(r.avgSpike["src"] - 50.0) <= 2.5
    assert r.sumNaNs == 0
    from oracle import oracle as O
    o = cpu_sim(O, spec)
    step, pop, neu = o.finish()
    assert np.array_equal(r.raster.step, step) and np.array_equal(r.raster.neuron, neu)


def test_lifecycle_and_step_counts():
    """test_engine.cpp:558-590."""
    def steps(duration, dt):
        spec = specs.mbody_spec(100, 0.5, duration, dt_ms=dt)
        return S.Simulation(spec).steps_total()
    assert steps(1000.0, 1.0) == 1000 and steps(1000.5, 1.0) == 1001
    assert steps(0.3, 0.1) == 3 and steps(0.05, 0.1) == 1 and steps(250.0, 0.5) == 500
    spec = specs.mbody_spec(100, 0.5, 0.5)
    sim = S.Simulation(spec)
    r = sim.finish()
    assert r.steps == 5
    with pytest.raises(S.SpecError):
        sim.finish()
    with pytest.raises(S.SpecError):
        sim.step()
    sim2 = S.Simulation(specs.mbody_spec(100, 0.5, 0.2))
    sim2.step()
    sim2.step()
    with pytest.raises(S.SpecError):
        sim2.step()
    bad = specs.mbody_spec(100, 0.5, 1.0)
    bad.dtMs = 0.0
    with pytest.raises(S.SpecError):
        S.run(bad)
    over = specs.mbody_spec(100, 0.5, 1.0)
    over.synapses[0].gScale = 1e41  # U(0, 0.02) * 1e41 overflows fp32
    with pytest.raises(S.SpecError, match="overflow"):
        S.Simulation(over)


def test_propagate_hand_example_and_errors():
    """test_engine.cpp:292-333 on the device."""
    w = np.array([[0, .5, 0], [.2, 0, .3]], np.float32)
    acc = np.zeros(3, np.float32)
    S.propagate_dense(w, [0, 1], acc)
    assert acc.tolist() == np.array([.2, .5, .3], np.float32).tolist()
    g = np.array([.5, .2, .3], np.float32)
    ind = np.array([1, 0, 2], np.int32)
    rs = np.array([0, 1, 3], np.int64)
    acc2 = np.zeros(3, np.float32)
    S.propagate_crs(g, ind, rs, 3, [0, 1], acc2)
    assert acc2.tolist() == acc.tolist()
    acc3 = np.ones(3, np.float32)
    S.propagate_dense(w, [1], acc3)
    assert acc3.tolist() == np.array([1.2, 1, 1.3], np.float32).tolist()
    acc4 = np.array([1, 2, 3], np.float32)
    S.propagate_dense(w, [], acc4)
    assert acc4.tolist() == [1, 2, 3]
    with pytest.raises(S.SpecError):
        S.propagate_dense(w, [0], np.zeros(2, np.float32))
    with pytest.raises(S.SpecError):
        S.propagate_crs(g, ind, rs, 3, [2], np.zeros(3, np.float32))
    with pytest.raises(S.SpecError):
        S.propagate_dense(w, [-1], np.zeros(3, np.float32))


def test_propagate_dense_equals_sparse_and_oracle_200_seeds(oracle_mod):
    """test_engine.cpp:335-359 on the device, checked against the oracle too."""
    lib = oracle_mod.oracle_lib()
    rng = np.random.default_rng(1)
    for seed in range(200):
        npre, npost = int(rng.integers(1, 41)), int(rng.integers(1, 400))
        k = int(rng.integers(1, npost + 1))
        sign = 1 if rng.integers(2) == 0 else -1
        w = S.gen_fixed_outdegree(npre, npost, k, S.WeightDist.uniform(0.0, 2.0), sign, seed)
        rows = [np.nonzero(w[i])[0] for i in range(npre)]
        rs = np.concatenate([[0], np.cumsum([len(r) for r in rows])]).astype(np.int64)
        ind = np.concatenate(rows).astype(np.int32)
        g = np.concatenate([w[i][rows[i]] for i in range(npre)]).astype(np.float32)
        spk = np.nonzero(rng.integers(0, 3, npre) == 0)[0].astype(np.int32)
        acc0 = rng.uniform(-1, 1, npost).astype(np.float32)
        a, b, c = acc0.copy(), acc0.copy(), acc0.copy()
        S.propagate_dense(w, spk, a)
        S.propagate_crs(g, ind, rs, npost, spk, b)
        lib.or_propagate_dense(w.ctypes.data, npost, spk.ctypes.data, spk.size, c.ctypes.data)
        assert specs.bits_equal(a, b) and specs.bits_equal(a, c), seed


def test_detect_nans_on_device():
    st = S.PopulationState(np.array([1, np.inf, 3, 4], np.float32),
                           np.array([0, 0, np.nan, 0], np.float32), np.array([], np.float32),
                           np.array([], np.float32), np.zeros(4, np.float32),
                           np.zeros(4, np.float32), np.zeros(4, np.uint8), 0)
    assert S.detect_nans(st, S.ModelKind.Izhikevich) == 2
    assert st.nanFlag.tolist() == [0, 1, 1, 0] and st.flagged == 2
    assert S.detect_nans(st, S.ModelKind.Izhikevich) == 0
    st.v[1], st.u[2], st.v[3] = 0, 0, np.nan
    assert S.detect_nans(st, S.ModelKind.Izhikevich) == 1 and st.flagged == 3
    st2 = S.PopulationState(np.zeros(3, np.float32), np.array([], np.float32),
                            np.array([np.inf, 0, 0], np.float32),
                            np.array([0, np.nan, 0], np.float32), np.zeros(3, np.float32),
                            np.zeros(3, np.float32), np.zeros(3, np.uint8), 0)
    assert S.detect_nans(st2, S.ModelKind.CondLif) == 2
    assert S.detect_nans(st2, S.ModelKind.PoissonSource) == 0


def test_config3_full_size_matches_oracle(oracle_mod):
    """Config 3 (100k KC, pn_kc CRS, dense lhi_kc/kc_dn) at full size for 100 ms
    (1000 steps): bit-exact raster, rates and final state."""
    spec, mode = specs.config_spec(3, 100.0)
    g = gpu_sim(spec, mode)
    o = cpu_sim(oracle_mod, spec, mode)
    rg = g.finish()
    ro = o.finish()
    assert np.array_equal(rg.raster.step, ro[0]) and np.array_equal(rg.raster.neuron, ro[2])
    assert_state_equal(g, o, spec, "config 3 end")
    assert rg.avgSpike["kc"] > 100.0  # the network is in its active regime


def test_config4_million_kc_short_matches_oracle(oracle_mod):
    """Config 4 (1M KC) for 3 ms: bit-exact against the oracle."""
    spec, mode = specs.config_spec(4, 3.0)
    g = gpu_sim(spec, mode)
    o = cpu_sim(oracle_mod, spec, mode)
    rg = g.finish()
    ro = o.finish()
    assert np.array_equal(rg.raster.step, ro[0]) and np.array_equal(rg.raster.neuron, ro[2])
    assert_state_equal(g, o, spec, "config 4 end")


def test_block_policies_do_not_change_results():
    spec = specs.mbody_spec(20000, 0.05, 30.0)
    ref = None
    for kw in ({}, {"blockPolicy": 1}, {"blockSize": 96}, {"blockSize": 1024}):
        sim = gpu_sim(spec, **kw)
        r = sim.finish()
        key = (r.raster.neuron.tobytes(), sim.pull(2, "v").tobytes())
        ref = ref or key
        assert key == ref, kw


# ---- split populations (multi-GPU decomposition) --------------
# virtualWorld = R runs the R shards of a world inside one process on this
# GPU: the same kernels and the same per-window exchange (local bitmasks
# gathered in rank order, assembled, compacted) with device copies in place
# of the NCCL all-gather.  Results must equal the unsplit engine bit for bit.

@pytest.mark.parametrize("world", [2, 3, 8])
@pytest.mark.parametrize("name", ["cfg2_100ms", "cfg3_20ms", "cfg2_fromspec_100ms"])
def test_split_world_matches_reference_golden(golden, name, world):
    spec, mode = GOLDEN[name]()
    g = golden["runs"][name]
    sim = gpu_sim(spec, mode, window=64, virtualWorld=world)
    assert sim.world() == world
    lo, nl, ng = sim.shard_range("kc")
    assert (lo, ng) == (0, spec.populations[spec.pop_index("kc")].size) and nl < ng
    r = sim.finish()
    assert len(r.raster) == g["n_events"]
    assert specs.sha(r.raster.step, r.raster.population, r.raster.neuron) == g["raster_sha"]
    assert [r.avgSpike[p.name] for p in spec.populations] == g["rates"]
    assert r.sumNaNs == g["sum_nans"]
    for pi, p in enumerate(spec.populations):
        for f, h in g["state_sha"][p.name].items():
            if p.model == S.ModelKind.PoissonSource and f in ("v", "gExc", "gInh"):
                continue
            assert specs.sha(sim.pull(pi, f)) == h, (p.name, f)


@pytest.mark.parametrize("window", [1, 5])
def test_split_world_stepwise_state_and_fault_injection(oracle_mod, window):
    """Small windows, state pulled (gathered across shards) every few steps,
    and a NaN injected through push (scattered to its shard)."""
    spec, mode = specs.config_spec(2, 12.0)
    g = gpu_sim(spec, mode, window=window, virtualWorld=2, shardMinSize=32)
    o = cpu_sim(oracle_mod, spec, mode)
    kc = spec.pop_index("kc")
    for t in range(0, 120, 15):
        g.step(15)
        o.step(15)
        assert_state_equal(g, o, spec, f"t={t + 15}")
        if t == 45:
            v = o.state(kc, "v")
            v[7000] = np.nan  # lives on shard 1
            g.push(kc, "v", v)
            o.set_state(kc, "v", v)
    rg, ro = g.finish(), o.finish()
    assert rg.sumNaNs == o.sum_nans() >= 1
    assert np.array_equal(rg.raster.step, ro[0])
    assert np.array_equal(rg.raster.population, ro[1])
    assert np.array_equal(rg.raster.neuron, ro[2])


def test_concurrent_simulations_of_different_sizes(golden):
    """Two live engines with different shared-memory plans (the per-kernel
    dynamic shared-memory limit is process-wide; a smaller engine built
    later must not lower it under the larger one)."""
    spec3, mode3 = GOLDEN["cfg3_20ms"]()
    spec1, mode1 = GOLDEN["cfg1_1000ms"]()
    big = gpu_sim(spec3, mode3)
    small = gpu_sim(spec1, mode1)
    for sim, name in ((big, "cfg3_20ms"), (small, "cfg1_1000ms")):
        r = sim.finish()
        assert specs.sha(r.raster.step, r.raster.population, r.raster.neuron) == \
            golden["runs"][name]["raster_sha"]


def test_raster_drain_midway_keeps_results(golden):
    """ssb_raster_drain moves events to the host mid-run; the finished raster
    is unchanged (the bench's end-to-end leg relies on it)."""
    spec, mode = GOLDEN["cfg2_100ms"]()
    sim = gpu_sim(spec, mode, window=64)
    held = 0
    for n in (100, 300, 250):
        sim.step(n)
        h = sim.drain_raster()
        assert h >= held
        held = h
    r = sim.finish()
    assert len(r.raster) >= held
    assert specs.sha(r.raster.step, r.raster.population, r.raster.neuron) == \
        golden["runs"]["cfg2_100ms"]["raster_sha"]


def test_raster_pinned_pool_drains_keep_results(golden):
    """EngineOptions.rasterPinnedMB: drains that fit copy straight into pinned
    pool blocks, the rest (pool exhausted: one 32 MB block, held by the first
    drain's chunk) go through staging; async and waited drains interleave and
    the finished raster is the golden one."""
    spec, mode = GOLDEN["cfg2_100ms"]()
    sim = gpu_sim(spec, mode, window=64, rasterPinnedMB=32)
    sim.step(200)
    sim.drain_raster(wait=False)  # takes the pool's only block
    sim.step(300)
    assert sim.drain_raster() > 0  # staged: the pool is empty
    sim.step(250)
    sim.drain_raster(wait=False)
    r = sim.finish()
    assert specs.sha(r.raster.step, r.raster.population, r.raster.neuron) == \
        golden["runs"]["cfg2_100ms"]["raster_sha"]


def test_nccl_exchange_selftest():
    """The split engine's collectives (dlopen'd libnccl, one-rank communicator):
    all-gather and sum, plain and captured in a CUDA graph."""
    S.comm_selftest(0)


def test_sweep_cells_match_oracle(oracle_mod):
    """The calibration sweep on the GPU (calibration.cpp:16-86): every cell's
    target rate and NaN count equal the oracle's run of the same network;
    cells run 3 at a time on their own streams."""
    def builder(n, g):
        spec = specs.mbody_spec(1000, 0.5, 50.0)
        pk = spec.synapses[spec.group_index("pn_kc")]
        pk.outDegree = n
        pk.gScale = g
        return spec
    req = S.SweepRequest([100, 300, 500], [0.5, 1.5], "kc", parallelism=3,
                         storage=S.StorageMode.ForceDense)
    rows = S.sweep(builder, req)
    assert len(rows) == 6 and not any(r.failed for r in rows)
    kc = 2
    for r in rows:
        spec = builder(r.nConn, r.gScale)
        o = cpu_sim(oracle_mod, spec, S.StorageMode.ForceDense)
        o.finish()
        assert r.avgSpike == float(o.rates()[kc]), (r.nConn, r.gScale)
        assert r.sumNaNs == o.sum_nans()
    assert len({r.avgSpike for r in rows}) > 1


@pytest.mark.parametrize("name", ["cfg3_20ms", "cfg2_100ms", "izh_ff_200ms"])
@pytest.mark.parametrize("local", [False, True])
def test_nccl_split_path_one_rank_matches_golden(golden, name, local):
    """A communicator id with a world of one rank runs the whole split path on
    a real (one-rank) NCCL communicator: per-window all-gathers captured in the
    window graphs, assembly, compaction, gathered state pulls and the NaN sum;
    with rasterLocal the raster comes from the rank's own lists (the local
    compaction and index offset of split populations; one rank owns all)."""
    spec, mode = GOLDEN[name]()
    g = golden["runs"][name]
    sim = gpu_sim(spec, mode, window=64, world=1, rank=0, commId=S.comm_unique_id(),
                  shardMinSize=32, rasterLocal=local)
    r = sim.finish()
    assert specs.sha(r.raster.step, r.raster.population, r.raster.neuron) == g["raster_sha"]
    assert r.sumNaNs == g["sum_nans"]
    for pi, p in enumerate(spec.populations):
        for f, h in g["state_sha"][p.name].items():
            if p.model == S.ModelKind.PoissonSource and f in ("v", "gExc", "gInh"):
                continue
            assert specs.sha(sim.pull(pi, f)) == h, (p.name, f)


@pytest.mark.parametrize("kw", [{"window": 1}, {"window": 64}, {"window": 64, "virtualWorld": 2,
                                                                 "shardMinSize": 32}])
def test_traubmiles_kcs_match_restatement(oracle_mod, kw):
    """Traub-Miles HH KCs (extension F1, no reference implementation): the
    device equals the CPU restatement in oracle.c bit for bit (same custom
    exp, same operation order) -- state every 100 steps and the raster."""
    spec = specs.hh_mbody_spec()
    g = gpu_sim(spec, **kw)
    o = cpu_sim(oracle_mod, spec)
    kc = spec.pop_index("kc")
    for t in range(3):
        g.step(100)
        o.step(100)
        for f in ("v", "gExc", "gInh", "m", "h", "n", "excIn", "inhIn"):
            assert specs.bits_equal(g.pull(kc, f), o.state(kc, f)), (t, f)
    rg, ro = g.finish(), o.finish()
    assert np.array_equal(rg.raster.neuron, ro[2]) and np.array_equal(rg.raster.step, ro[0])
    assert np.count_nonzero(rg.raster.population == kc) > 100


# ---- BASELINE configs 3 and 4 at their bench horizons ------------------------

def assert_matches_golden_run(sim, r, spec, g):
    counts = [int(np.count_nonzero(r.raster.population == i)) for i in range(len(spec.populations))]
    assert counts == g["counts"]
    assert len(r.raster) == g["n_events"]
    assert specs.sha(r.raster.step, r.raster.population, r.raster.neuron) == g["raster_sha"]
    assert specs.raster_checksum(r.raster.step, r.raster.population, r.raster.neuron) == \
        int(g["checksum"])
    assert [r.avgSpike[p.name] for p in spec.populations] == g["rates"]
    assert r.sumNaNs == g["sum_nans"]
    for pi, p in enumerate(spec.populations):
        for f, h in g["state_sha"][p.name].items():
            if p.model == S.ModelKind.PoissonSource and f in ("v", "gExc", "gInh"):
                continue
            assert specs.sha(sim.pull(pi, f)) == h, (p.name, f)


def test_config3_full_second_matches_reference_golden(golden):
    """BASELINE config 3 over its whole 1 s (10,000 steps, the bench's 256-step
    windows in multi-window graphs): raster, counts, rates and every final
    state array equal the reference's own run (golden cfg3_1000ms)."""
    spec, mode = specs.config_spec(3, 1000.0)
    sim = gpu_sim(spec, mode, window=256)
    r = sim.finish()
    assert_matches_golden_run(sim, r, spec, golden["runs"]["cfg3_1000ms"])


@pytest.mark.parametrize("kw", [{}, {"virtualWorld": 8}])
def test_config4_100ms_matches_reference_golden(golden, kw):
    """BASELINE config 4 (1M KC) over 1,000 steps (four 256-step windows; the
    arena-budgeted graph path), whole and as the 8-rank decomposition of §6
    (virtual shards on one GPU): equal to the reference's own run."""
    spec, mode = specs.config_spec(4, 100.0)
    sim = gpu_sim(spec, mode, window=256, **kw)
    r = sim.finish()
    assert_matches_golden_run(sim, r, spec, golden["runs"]["cfg4_100ms"])


@pytest.mark.parametrize("world", [1, 2, 8])
def test_bench_split_networks_match_parity_golden(world):
    """The networks bench.py times at N GPUs (N x 100k KC) over its 100-ms
    parity horizon, split N ways (virtual shards): spike counts and the
    order-independent raster checksum equal the reference's
    (tests/golden/bench_parity.json)."""
    import json
    with open(os.path.join(os.path.dirname(__file__), "golden", "bench_parity.json")) as f:
        gold = json.load(f)["runs"][f"split{world}"]
    spec = specs.mbody_spec(100_000 * world, 0.05, 100.0)
    kw = {"virtualWorld": world} if world > 1 else {}
    sim = gpu_sim(spec, window=256, **kw)
    r = sim.finish()
    counts = [int(np.count_nonzero(r.raster.population == i)) for i in range(4)]
    assert counts == gold["counts"]
    assert specs.raster_checksum(r.raster.step, r.raster.population, r.raster.neuron) == \
        int(gold["checksum"])


@pytest.mark.parametrize("frac", [0.001, 0.05, 0.3, 0.5])
def test_storage_mode_auto_matches_reference_modes(oracle_mod, frac):
    """StorageMode.Auto never changes results (reference engine.hpp:15-18): at
    densities on both sides of the threshold the raster and state equal the
    oracle's FromSpec run bit for bit, and the chosen layout follows density."""
    spec = specs.mbody_spec(20_000, frac, 40.0)
    g = gpu_sim(spec, S.StorageMode.Auto, window=64)
    o = cpu_sim(oracle_mod, spec, S.StorageMode.FromSpec)
    rg = g.finish()
    ro = o.finish()
    assert np.array_equal(rg.raster.step, ro[0]) and np.array_equal(rg.raster.neuron, ro[2])
    assert np.array_equal(rg.raster.population, ro[1])
    assert_state_equal(g, o, spec, f"auto {frac}")
    dense_pn_kc = g.group_dense("pn_kc") is not None
    assert dense_pn_kc == (frac >= S.auto_dense_threshold())


@pytest.mark.parametrize("window", [16, 256])
@pytest.mark.parametrize("which", ["lif", "izh"])
def test_cyclic_block_stepwise_state_matches_oracle(oracle_mod, which, window):
    """Small recurrent networks run one block per window (cyclic.cuh): every
    state array after irregular call sizes equals the oracle, and the block
    kernel is the path that ran."""
    spec = specs.recurrent_lif_spec(200, 200.0) if which == "lif" else specs.izh_spec(300, 30, 400.0)
    g = gpu_sim(spec, window=window)
    o = cpu_sim(oracle_mod, spec)
    for n in [1, 2, 3, 5, 8, 13, 21, 34, 55, 89, 100]:
        g.step(n)
        o.step(n)
        assert_state_equal(g, o, spec, f"after {o.steps_done()} steps")
    rg, ro = g.finish(), o.finish()
    assert np.array_equal(rg.raster.step, ro[0]) and np.array_equal(rg.raster.neuron, ro[2])
    p = gpu_sim(spec, window=window, profile=True)
    p.step(64)
    p.sync()
    names = {name for name, _, _ in p.kernel_stats()}
    assert "cyclic_block" in names, names
    p.close()
