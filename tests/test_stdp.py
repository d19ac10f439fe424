"""Extension F2: KC->DN learning (pair-based STDP on a dense all-to-all group).

Not in the reference, so parity is against the repo's own
statement of the rule (include/synscale/synscale.hpp StdpRule, DESIGN.md §1
row A22): the C oracle (oracle/oracle.c or_stdp_step) is pinned here by an
independent numpy replay of the rule over the oracle's own raster, and the
CUDA path must equal the oracle bit for bit (weights, traces' effect on
weights, rasters and every state array).
"""
import numpy as np
import pytest

import specs
from paper_1412_0595_b200 import synscale as S


def cpu_sim(O, spec, mode=S.StorageMode.FromSpec):
    d = S.NetDesc(spec)
    sim = O.CpuSim(d.ptr, spec, int(mode))
    sim._desc = d
    return sim


def replay_stdp(spec, w0, raster):
    """numpy float32 restatement of the STDP rule over a recorded raster."""
    gi = spec.group_index("kc_dn")
    g = spec.synapses[gi]
    r = g.stdp
    f = np.float32
    dt = spec.dtMs
    aP, aM, wMax = f(r.aPlus), f(r.aMinus), f(r.wMax)
    dP, dM = f(np.exp(-dt / r.tauPlusMs)), f(np.exp(-dt / r.tauMinusMs))
    pre_p, post_p = spec.pop_index(g.pre), spec.pop_index(g.post)
    W = w0.astype(np.float32).copy()
    x = np.zeros(W.shape[0], np.float32)
    y = np.zeros(W.shape[1], np.float32)
    step, pop, neuron = raster
    steps = int(step.max()) + 1 if len(step) else 0
    for t in range(steps):
        sel = step == t
        pre = neuron[sel & (pop == pre_p)]
        post = neuron[sel & (pop == post_p)]
        xd = x * dP
        yd = y * dM
        touched = np.zeros(W.shape, bool)
        V = W.copy()
        if len(pre):
            V[pre, :] = V[pre, :] - aM * yd[None, :]
            touched[pre, :] = True
        if len(post):
            V[:, post] = V[:, post] + (aP * xd)[:, None]
            touched[:, post] = True
        W = np.where(touched, np.minimum(np.maximum(V, f(0)), wMax), W)
        x = xd.copy()
        x[pre] = xd[pre] + f(1)
        y = yd.copy()
        y[post] = yd[post] + f(1)
    return W


def test_oracle_stdp_matches_numpy_replay(oracle_mod):
    spec = specs.stdp_mbody_spec(1000, 150.0)
    gi = spec.group_index("kc_dn")
    o = cpu_sim(oracle_mod, spec)
    w0 = o.group(gi)[1].copy()
    raster = o.finish()
    w1 = o.group(gi)[1]
    assert not np.array_equal(w0, w1), "the rule never fired"
    post = spec.pop_index("dn")
    assert (raster[1] == post).sum() > 0
    assert np.array_equal(replay_stdp(spec, w0, raster), w1)
    assert w1.min() >= 0 and w1.max() <= np.float32(spec.synapses[gi].stdp.wMax)


def test_oracle_stdp_zero_amplitudes_is_static(oracle_mod):
    static = specs.mbody_spec(1000, 0.05, 60.0)
    plastic = specs.stdp_mbody_spec(1000, 60.0, a_plus=0.0, a_minus=0.0)
    a, b = cpu_sim(oracle_mod, static), cpu_sim(oracle_mod, plastic)
    ra, rb = a.finish(), b.finish()
    for u, v in zip(ra, rb):
        assert np.array_equal(u, v)
    gi = static.group_index("kc_dn")
    assert np.array_equal(a.group(gi)[1], b.group(gi)[1])


@pytest.mark.parametrize("mutate, field", [
    (lambda g: setattr(g, "storage", S.StorageKind.Sparse), "stdp"),
    (lambda g: setattr(g, "sign", S.SynapseSign.Inhibitory), "stdp"),
    (lambda g: setattr(g, "outDegree", 50), "stdp"),
    (lambda g: setattr(g.stdp, "wMax", 0.0), "stdp"),
    (lambda g: setattr(g.stdp, "tauPlusMs", -1.0), "stdp"),
    (lambda g: setattr(g.stdp, "aMinus", float("nan")), "stdp"),
])
def test_stdp_validation(mutate, field):
    spec = specs.stdp_mbody_spec(1000, 10.0)
    assert S.validate(spec) == []
    mutate(spec.synapses[spec.group_index("kc_dn")])
    errs = S.validate(spec)
    assert any(f.endswith(field) for f, _ in errs), errs


def test_stdp_spec_round_trips_through_the_c_abi():
    spec = specs.stdp_mbody_spec(1000, 10.0)
    back = S._spec_from_desc(S.NetDesc(spec).desc)
    assert back.synapses[back.group_index("kc_dn")].stdp == spec.synapses[spec.group_index("kc_dn")].stdp
    assert back.synapses[back.group_index("pn_kc")].stdp is None


@pytest.mark.gpu
@pytest.mark.parametrize("n_kc, ms", [(1000, 300.0), (100_000, 20.0)])
def test_gpu_stdp_bit_exact(oracle_mod, n_kc, ms):
    spec = specs.stdp_mbody_spec(n_kc, ms)
    gi = spec.group_index("kc_dn")
    g = S.Simulation(spec, S.StorageMode.FromSpec, S.EngineOptions())
    o = cpu_sim(oracle_mod, spec)
    w0 = o.group(gi)[1].copy()
    half = g.steps_total() // 2
    g.step(half)
    o.step(half)
    assert np.array_equal(g.group_weights("kc_dn"), o.group(gi)[1])
    r = g.finish()
    ro = o.finish()
    w1 = o.group(gi)[1]
    assert not np.array_equal(w0, w1)
    assert np.array_equal(g.group_weights("kc_dn"), w1)
    assert np.array_equal(r.raster.step, ro[0]) and np.array_equal(r.raster.neuron, ro[2])
    assert np.array_equal(r.raster.population, ro[1])
    for pi, p in enumerate(spec.populations):
        if p.model == S.ModelKind.PoissonSource:
            continue
        for f in ("v", "gExc", "gInh", "excIn", "inhIn"):
            assert specs.bits_equal(g.pull(pi, f), o.state(pi, f)), f"{p.name}.{f}"
    # a static group reads back its built matrix
    assert np.array_equal(g.group_weights("lhi_kc"), o.group(spec.group_index("lhi_kc"))[1])


@pytest.mark.gpu
def test_gpu_stdp_rejects_split_worlds():
    spec = specs.stdp_mbody_spec(1000, 10.0)
    with pytest.raises(S.SpecError):
        S.Simulation(spec, S.StorageMode.FromSpec, S.EngineOptions(virtualWorld=2))


@pytest.mark.gpu
@pytest.mark.parametrize("window", [64, 256])
def test_gpu_plastic_sink_matches_step_mode_config3(monkeypatch, window):
    """Config 3 + STDP over 0.3 s (DN volleys, the background's lag, many
    windows): the windowed plastic-sink path and step mode give the same
    weights, rasters and state, bit for bit."""
    spec = specs.stdp_mbody_spec(100_000, 300.0)
    runs = []
    for tail in ("1", "0"):
        monkeypatch.setenv("SSB_PLASTIC_TAIL", tail)
        sim = S.Simulation(spec, S.StorageMode.FromSpec, S.EngineOptions(window=window))
        sim.step(1234)
        w_mid = sim.group_weights("kc_dn").copy()
        sim.step(1766)
        w_end = sim.group_weights("kc_dn").copy()
        state = {(pi, f): sim.pull(pi, f) for pi, p in enumerate(spec.populations)
                 if p.model != S.ModelKind.PoissonSource for f in ("v", "gExc", "gInh", "excIn")}
        r = sim.finish()
        runs.append((w_mid, w_end, r, state))
        sim.close()
    (wa, wb, ra, sa), (wc, wd, rc, sc) = runs
    assert np.array_equal(wa, wc) and np.array_equal(wb, wd)
    assert np.array_equal(ra.raster.step, rc.raster.step)
    assert np.array_equal(ra.raster.neuron, rc.raster.neuron)
    assert np.array_equal(ra.raster.population, rc.raster.population)
    dn = [p.name for p in spec.populations].index("dn")
    assert int((ra.raster.population == dn).sum()) > 1000  # volleys happened
    for k in sa:
        assert specs.bits_equal(sa[k], sc[k]), k


@pytest.mark.gpu
@pytest.mark.parametrize("n_kc, n_dn", [(1003, 37), (4099, 65), (20000, 128)])
def test_gpu_plastic_sink_odd_sizes_match_oracle(oracle_mod, n_kc, n_dn):
    """Ragged shapes of the plastic-sink path: a partial column block, pre rows
    not a multiple of four (the scalar background path), the largest sink;
    weights, raster and state equal the oracle's."""
    spec = specs.stdp_mbody_spec(n_kc, 200.0, n_dn=n_dn, a_plus=0.3)
    gi = spec.group_index("kc_dn")
    g = S.Simulation(spec, S.StorageMode.FromSpec, S.EngineOptions(window=64))
    o = cpu_sim(oracle_mod, spec)
    g.step(g.steps_total())
    o.step(o.steps_total())
    assert np.array_equal(g.group_weights("kc_dn"), o.group(gi)[1])
    r, ro = g.finish(), o.finish()
    assert np.array_equal(r.raster.step, ro[0]) and np.array_equal(r.raster.neuron, ro[2])
    assert np.array_equal(r.raster.population, ro[1])
    for pi, p in enumerate(spec.populations):
        if p.model == S.ModelKind.PoissonSource:
            continue
        for f in ("v", "gExc", "gInh", "excIn"):
            assert specs.bits_equal(g.pull(pi, f), o.state(pi, f)), f"{p.name}.{f}"
    p = S.Simulation(spec, S.StorageMode.FromSpec, S.EngineOptions(window=64, profile=True))
    p.step(128)
    p.sync()
    assert any(name.startswith("sink_step") for name, _, _ in p.kernel_stats())
    p.close()


@pytest.mark.gpu
@pytest.mark.parametrize("window", [1, 3, 7, 250])
def test_gpu_plastic_sink_small_and_odd_windows_match_oracle(oracle_mod, window):
    """Windows of 1, 3, 7 and 250 steps (the sink's step-parity rings, the
    background's lag longer than the window) against the oracle."""
    spec = specs.stdp_mbody_spec(2000, 60.0, a_plus=0.3)
    gi = spec.group_index("kc_dn")
    g = S.Simulation(spec, S.StorageMode.FromSpec, S.EngineOptions(window=window))
    o = cpu_sim(oracle_mod, spec)
    for n in (5, 17, 100, 478):
        g.step(n)
        o.step(n)
        assert np.array_equal(g.group_weights("kc_dn"), o.group(gi)[1]), f"after {o.steps_done()} steps"
    r, ro = g.finish(), o.finish()
    assert np.array_equal(r.raster.step, ro[0]) and np.array_equal(r.raster.neuron, ro[2])
