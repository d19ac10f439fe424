"""Pins the oracle (oracle/oracle.c) before it is trusted as the parity checker.

* against the golden fixtures generated from the reference itself
  (tests/golden/make_golden.py) — always;
* against the reference library compiled here (oracle/_ref) — when present;
* re-hosts the reference's own known-answer tests for the step path
  (test_engine.cpp:183-359, 361-400).
"""
import os

import numpy as np
import pytest

import specs
from paper_1412_0595_b200 import synscale as S


def _run(O, spec, mode, ref=False):
    d = S.NetDesc(spec)
    sim = O.CpuSim(d.ptr, spec, int(mode), ref=ref)
    r = sim.finish()
    return sim, r


def test_streams_match_golden(oracle_mod, golden):
    for key, vals in golden["streams"].items():
        g, e, label = key.split("/", 2)
        got = oracle_mod.stream_u64(int(g), int(e), label, len(vals))
        assert [str(int(x)) for x in got] == vals, key


def test_derive_seed_matches_golden(oracle_mod, golden):
    lib = oracle_mod.oracle_lib()
    for key, val in golden["derive_seed"].items():
        p, label = key.split("/", 1)
        assert str(lib.or_derive_seed_c(int(p), label.encode())) == val


def test_gen_fixed_outdegree_matches_golden(oracle_mod, golden):
    for entry in golden["gen_fixed_outdegree"]:
        args = [int(a) if isinstance(a, str) else a for a in entry["args"]]
        m = oracle_mod.gen_fixed_outdegree(*args)
        assert specs.sha(m) == entry["sha"]
        assert int(np.count_nonzero(m)) == entry["nnz"]
        if "weights" in entry:
            assert m.ravel().view(np.uint32).tolist() == entry["weights"]


@pytest.mark.parametrize("name", ["cfg1_1000ms", "cfg2_100ms", "cfg3_20ms", "cfg1_sparse_300ms",
                                  "cfg2_fromspec_100ms", "chain_100ms", "recurrent_200ms",
                                  "izh_1000_1000ms", "izh_1000_dense_300ms", "izh_ff_200ms"])
def test_oracle_runs_match_golden(oracle_mod, golden, name):
    g = golden["runs"][name]
    spec, mode = {
        "cfg1_1000ms": specs.config_spec(1, 1000.0),
        "cfg2_100ms": specs.config_spec(2, 100.0),
        "cfg3_20ms": specs.config_spec(3, 20.0),
        "cfg1_sparse_300ms": (specs.config_spec(1, 300.0)[0], S.StorageMode.ForceSparse),
        "cfg2_fromspec_100ms": (specs.config_spec(2, 100.0)[0], S.StorageMode.FromSpec),
        "chain_100ms": (specs.chain_spec(100.0), S.StorageMode.FromSpec),
        "recurrent_200ms": (specs.recurrent_lif_spec(), S.StorageMode.FromSpec),
        "izh_1000_1000ms": (specs.izh_spec(), S.StorageMode.FromSpec),
        "izh_1000_dense_300ms": (specs.izh_spec(duration_ms=300.0), S.StorageMode.ForceDense),
        "izh_ff_200ms": (specs.izh_ff_spec(), S.StorageMode.FromSpec),
    }[name]
    sim, (step, pop, neu) = _run(oracle_mod, spec, mode)
    assert step.size == g["n_events"]
    assert specs.sha(step, pop, neu) == g["raster_sha"]
    assert [float(x) for x in sim.rates()] == g["rates"]
    assert sim.sum_nans() == g["sum_nans"]
    for pi, p in enumerate(spec.populations):
        for f, h in g["state_sha"][p.name].items():
            assert specs.sha(sim.state(pi, f)) == h, (p.name, f)
    for gi, grp in enumerate(spec.synapses):
        kind, m = sim.group(gi)
        assert [kind, specs.sha(*(m if kind == "sparse" else (m,)))] == g["groups"][grp.name]


def test_izhikevich_kat_per_step(oracle_mod):
    """test_engine.cpp:79-111: per-step bitwise v, u of one bias-driven
    Izhikevich neuron, against the reference's values."""
    kat = np.load(os.path.join(os.path.dirname(__file__), "golden", "izh_kat.npz"))
    spec = specs.single_izh_spec()
    d = S.NetDesc(spec)
    sim = oracle_mod.CpuSim(d.ptr, spec, 0)
    for t in range(sim.steps_total()):
        sim.step(1)
        assert sim.state(0, "v")[0] == kat["v"][t] and sim.state(0, "u")[0] == kat["u"][t], t
    step, pop, neu = sim.finish()
    assert np.array_equal(step, kat["step"]) and len(step) > 0


def test_condlif_kat_per_step(oracle_mod):
    """test_engine.cpp:183-290: per-step bitwise v, gExc, gInh of one conductance
    neuron driven by two Poisson sources, against the reference's values."""
    import os
    kat = np.load(os.path.join(os.path.dirname(__file__), "golden", "condlif_kat.npz"))
    spec = specs.condlif_kat_spec()
    d = S.NetDesc(spec)
    sim = oracle_mod.CpuSim(d.ptr, spec, 0)
    for t in range(sim.steps_total()):
        sim.step(1)
        assert sim.state(2, "v")[0].view(np.uint32) == kat["v"][t].view(np.uint32), t
        assert sim.state(2, "gExc")[0].view(np.uint32) == kat["gExc"][t].view(np.uint32), t
        assert sim.state(2, "gInh")[0].view(np.uint32) == kat["gInh"][t].view(np.uint32), t
    step, pop, neu = sim.finish()
    assert np.array_equal(step, kat["step"]) and np.array_equal(neu, kat["neuron"])
    assert np.count_nonzero(pop == 2) > 0


def test_propagate_hand_example(oracle_mod):
    """test_engine.cpp:292-333."""
    lib = oracle_mod.oracle_lib()
    w = np.array([[0, .5, 0], [.2, 0, .3]], np.float32)
    spk = np.array([0, 1], np.int32)
    acc = np.zeros(3, np.float32)
    lib.or_propagate_dense(w.ctypes.data, 3, spk.ctypes.data, 2, acc.ctypes.data)
    assert acc.tolist() == np.array([.2, .5, .3], np.float32).tolist()
    acc = np.ones(3, np.float32)
    one = np.array([1], np.int32)
    lib.or_propagate_dense(w.ctypes.data, 3, one.ctypes.data, 1, acc.ctypes.data)
    assert acc.tolist() == np.array([1.2, 1, 1.3], np.float32).tolist()


def test_dense_equals_sparse_200_seeds(oracle_mod):
    """test_engine.cpp:335-359 on the oracle: both layouts add identically."""
    lib = oracle_mod.oracle_lib()
    rng = np.random.default_rng(0)
    for seed in range(200):
        npre, npost = int(rng.integers(1, 41)), int(rng.integers(1, 51))
        k = int(rng.integers(1, npost + 1))
        sign = 1 if rng.integers(2) == 0 else -1
        w = oracle_mod.gen_fixed_outdegree(npre, npost, k, S.L.WEIGHT_UNIFORM, 0.0, 2.0, 0.0,
                                           sign, seed)
        rs = np.zeros(npre + 1, np.int64)
        rows = [np.nonzero(w[i])[0] for i in range(npre)]
        rs[1:] = np.cumsum([len(r) for r in rows])
        ind = np.concatenate(rows).astype(np.int32)
        g = np.concatenate([w[i][rows[i]] for i in range(npre)]).astype(np.float32)
        spk = np.nonzero(rng.integers(0, 3, npre) == 0)[0].astype(np.int32)
        acc0 = rng.uniform(-1, 1, npost).astype(np.float32)
        a, b = acc0.copy(), acc0.copy()
        lib.or_propagate_dense(w.ctypes.data, npost, spk.ctypes.data, spk.size, a.ctypes.data)
        lib.or_propagate_crs(g.ctypes.data, ind.ctypes.data, rs.ctypes.data, spk.ctypes.data,
                             spk.size, b.ctypes.data)
        assert specs.bits_equal(a, b), seed


def test_detect_nans_sticky(oracle_mod):
    """test_engine.cpp:361-400."""
    lib = oracle_mod.oracle_lib()
    v = np.array([1, np.inf, 3, 4], np.float32)
    u = np.array([0, 0, np.nan, 0], np.float32)
    fl = np.zeros(4, np.uint8)
    assert lib.or_detect_nans(0, v.ctypes.data, u.ctypes.data, None, None, fl.ctypes.data, 4) == 2
    assert fl.tolist() == [0, 1, 1, 0]
    assert lib.or_detect_nans(0, v.ctypes.data, u.ctypes.data, None, None, fl.ctypes.data, 4) == 0
    v[1], u[2], v[3] = 0, 0, np.nan
    assert lib.or_detect_nans(0, v.ctypes.data, u.ctypes.data, None, None, fl.ctypes.data, 4) == 1
    assert fl.tolist() == [0, 1, 1, 1]
    z = np.zeros(3, np.float32)
    ge = np.array([np.inf, 0, 0], np.float32)
    gi = np.array([0, np.nan, 0], np.float32)
    fl = np.zeros(3, np.uint8)
    assert lib.or_detect_nans(2, z.ctypes.data, None, ge.ctypes.data, gi.ctypes.data,
                              fl.ctypes.data, 3) == 2


@pytest.fixture(scope="module")
def ref_available(oracle_mod):
    if not oracle_mod.have_ref():
        pytest.skip("reference build oracle/_ref not present (golden fixtures still pin)")
    return True


@pytest.mark.parametrize("mode", [0, 1, 2])
def test_oracle_matches_reference_stepwise(oracle_mod, ref_available, mode):
    """Oracle and the compiled reference agree on every state array after every
    step of a short mushroom-body run, and on the raster."""
    spec = specs.mbody_spec(2000, 0.1, 30.0)
    d = S.NetDesc(spec)
    a = oracle_mod.CpuSim(d.ptr, spec, mode)
    b = oracle_mod.CpuSim(d.ptr, spec, mode, ref=True)
    for _ in range(a.steps_total()):
        a.step(1)
        b.step(1)
        for pi in range(4):
            for f in ("v", "gExc", "gInh", "excIn", "inhIn", "nanFlag"):
                assert specs.bits_equal(a.state(pi, f), b.state(pi, f))
    ra, rb = a.finish(), b.finish()
    assert all(np.array_equal(x, y) for x, y in zip(ra, rb))


def test_oracle_matches_reference_fault_injection(oracle_mod, ref_available):
    """test_engine.cpp:402-434 style: a poisoned state spreads identically."""
    spec = specs.mbody_spec(1000, 0.5, 5.0)
    for g in spec.synapses:
        g.gScale = 1e30
    d = S.NetDesc(spec)
    a = oracle_mod.CpuSim(d.ptr, spec, 0)
    b = oracle_mod.CpuSim(d.ptr, spec, 0, ref=True)
    v = a.state(2, "v")
    v[3] = 1e30
    a.set_state(2, "v", v)
    b.set_state(2, "v", v)
    ra, rb = a.finish(), b.finish()
    assert all(np.array_equal(x, y) for x, y in zip(ra, rb))
    assert a.sum_nans() == b.sum_nans()
