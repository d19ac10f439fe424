"""Network specs shared by the tests, the golden generator, smoke() and bench.py.

The mushroom-body configs follow SURVEY.md §8(d) / BASELINE.md §2:
build_mbody_net(nPN=100, nLHI=20, nKC, nDN=100, seed=7) with dtMs=0.1,
pnRateHz=50 and gScales pn_lhi=1.0, lhi_kc=0.1, pn_kc=0.5/frac, kc_dn=30/nKC.
"""
from __future__ import annotations

import hashlib

import numpy as np

from paper_1412_0595_b200 import synscale as S

# BASELINE.json configs -> (nKC, pnKcOutFraction, storage mode)
CONFIGS = {
    1: (1_000, 0.5, S.StorageMode.ForceDense),
    2: (10_000, 0.05, S.StorageMode.ForceSparse),
    3: (100_000, 0.05, S.StorageMode.FromSpec),
    4: (1_000_000, 0.05, S.StorageMode.FromSpec),
}


def mbody_gscales(n_kc: int, frac: float) -> dict:
    return {"pn_kc": 0.5 / frac, "pn_lhi": 1.0, "lhi_kc": 0.1, "kc_dn": 30.0 / n_kc}


def mbody_spec(n_kc: int, frac: float, duration_ms: float, dt_ms: float = 0.1, seed: int = 7,
               n_pn: int = 100, n_lhi: int = 20, n_dn: int = 100) -> S.NetworkSpec:
    opt = S.MBodyBuildOptions(dtMs=dt_ms, durationMs=duration_ms, pnKcOutFraction=frac)
    return S.build_mbody_net(n_pn, n_lhi, n_kc, n_dn, mbody_gscales(n_kc, frac), seed, opt)


def config_spec(cfg: int, duration_ms: float):
    n_kc, frac, mode = CONFIGS[cfg]
    return mbody_spec(n_kc, frac, duration_ms), mode


def condlif_kat_spec() -> S.NetworkSpec:
    """The conductance-neuron known-answer network of test_engine.cpp:183-238."""
    spec = S.NetworkSpec(dtMs=1.0, durationMs=400.0, globalSeed=11)
    spec.populations = [
        S.NeuronPopulation("drive", 1, S.ModelKind.PoissonSource, 1, S.PoissonParams(200.0)),
        S.NeuronPopulation("damp", 1, S.ModelKind.PoissonSource, 2, S.PoissonParams(80.0)),
        S.NeuronPopulation("cell", 1, S.ModelKind.CondLif, 3, S.CondLifParams()),
    ]
    spec.synapses = [
        S.SynapseGroupSpec("exc", "drive", "cell", S.SynapseSign.Excitatory, 1,
                           S.WeightDist.constant(0.05)),
        S.SynapseGroupSpec("inh", "damp", "cell", S.SynapseSign.Inhibitory, 1,
                           S.WeightDist.constant(0.03)),
    ]
    return spec


def recurrent_lif_spec(n: int = 200, duration_ms: float = 200.0, seed: int = 3) -> S.NetworkSpec:
    """A CondLif population with self-connections (cyclic graph: one step per launch),
    driven by Poisson input through a sparse group; exercises windows of 1."""
    spec = S.NetworkSpec(dtMs=0.5, durationMs=duration_ms, globalSeed=seed)
    spec.populations = [
        S.NeuronPopulation("src", 50, S.ModelKind.PoissonSource, 1, S.PoissonParams(80.0)),
        S.NeuronPopulation("net", n, S.ModelKind.CondLif, 2, S.CondLifParams()),
    ]
    spec.synapses = [
        S.SynapseGroupSpec("drive", "src", "net", S.SynapseSign.Excitatory, n // 4,
                           S.WeightDist.uniform(0.0, 0.4), 1.0, S.StorageKind.Sparse),
        S.SynapseGroupSpec("rec_e", "net", "net", S.SynapseSign.Excitatory, n // 10,
                           S.WeightDist.uniform(0.0, 0.05), 1.0, S.StorageKind.Dense, 0, n // 2),
        S.SynapseGroupSpec("rec_i", "net", "net", S.SynapseSign.Inhibitory, n // 10,
                           S.WeightDist.uniform(0.0, 0.08), 1.0, S.StorageKind.Sparse, n // 2, -1),
    ]
    return spec


def chain_spec(duration_ms: float = 100.0) -> S.NetworkSpec:
    """Feed-forward chain with two groups on one accumulator (fold order across
    groups), a windowed pre range, a Poisson target and mixed storage."""
    spec = S.NetworkSpec(dtMs=0.25, durationMs=duration_ms, globalSeed=19)
    spec.populations = [
        S.NeuronPopulation("in_a", 64, S.ModelKind.PoissonSource, 1, S.PoissonParams(120.0)),
        S.NeuronPopulation("in_b", 300, S.ModelKind.PoissonSource, 2, S.PoissonParams(40.0)),
        S.NeuronPopulation("mid", 700, S.ModelKind.CondLif, 3, S.CondLifParams()),
        S.NeuronPopulation("out", 90, S.ModelKind.CondLif, 4,
                           S.CondLifParams(tauMMs=8.0, tauSynMs=3.0)),
        S.NeuronPopulation("sink", 40, S.ModelKind.PoissonSource, 5, S.PoissonParams(5.0)),
    ]
    spec.synapses = [
        S.SynapseGroupSpec("a_mid", "in_a", "mid", S.SynapseSign.Excitatory, 200,
                           S.WeightDist.uniform(0.0, 0.05), 2.0, S.StorageKind.Sparse),
        S.SynapseGroupSpec("b_mid", "in_b", "mid", S.SynapseSign.Excitatory, 120,
                           S.WeightDist.uniform(0.01, 0.03), 1.5, S.StorageKind.Dense, 20, 250),
        S.SynapseGroupSpec("a_mid_i", "in_a", "mid", S.SynapseSign.Inhibitory, 50,
                           S.WeightDist.constant(0.02), 1.0, S.StorageKind.Dense),
        S.SynapseGroupSpec("mid_out", "mid", "out", S.SynapseSign.Excitatory, 30,
                           S.WeightDist.uniform(0.0, 0.01), 3.0, S.StorageKind.Sparse),
        S.SynapseGroupSpec("mid_out2", "mid", "out", S.SynapseSign.Excitatory, 90,
                           S.WeightDist.constant(0.002), 1.0, S.StorageKind.Dense),
        S.SynapseGroupSpec("out_sink", "out", "sink", S.SynapseSign.Inhibitory, 10,
                           S.WeightDist.constant(0.5), 1.0, S.StorageKind.Sparse),
    ]
    return spec


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def bits_equal(a: np.ndarray, b: np.ndarray) -> bool:
    """Bitwise equality of float arrays, any NaN equal to any NaN."""
    a = np.asarray(a)
    b = np.asarray(b)
    if a.shape != b.shape:
        return False
    if a.dtype.kind != "f":
        return bool(np.array_equal(a, b))
    na, nb = np.isnan(a), np.isnan(b)
    if not np.array_equal(na, nb):
        return False
    return bool(np.array_equal(a[~na].view(np.uint32), b[~nb].view(np.uint32)))


def izh_spec(n: int = 1000, n_conn: int = 100, duration_ms: float = 1000.0,
             storage=S.StorageKind.Sparse, g_scale: float = 6.0, seed: int = 1) -> S.NetworkSpec:
    """The reference's acceptance network (acceptance_main.cpp:139-163):
    recurrent Izhikevich population, noise-driven, dt 1 ms."""
    opt = S.IzhBuildOptions(dtMs=1.0, durationMs=duration_ms, storage=storage)
    return S.build_izhikevich_net(n, n_conn, 0.8, g_scale, seed, opt)


def single_izh_spec(bias: float = 10.0, duration_ms: float = 300.0, seed: int = 99) -> S.NetworkSpec:
    """test_engine.cpp:21-41: one regular-spiking neuron with a constant bias."""
    spec = S.NetworkSpec(dtMs=1.0, durationMs=duration_ms, globalSeed=seed)
    spec.populations = [S.NeuronPopulation("n", 1, S.ModelKind.Izhikevich, 3, S.IzhikevichParams(
        a=[0.02], b=[0.2], c=[-65.0], d=[8.0], noiseAmplitude=[0.0], biasCurrent=[bias]))]
    return spec


def izh_ff_spec(duration_ms: float = 200.0) -> S.NetworkSpec:
    """Feed-forward mix (windowed path): Poisson -> noisy Izhikevich (odd size, so
    Gaussian pairs straddle steps) -> CondLif, dense and sparse groups."""
    import numpy as _np
    rng = _np.random.default_rng(5)
    n = 1001
    r = rng.random(n)
    spec = S.NetworkSpec(dtMs=0.5, durationMs=duration_ms, globalSeed=23)
    spec.populations = [
        S.NeuronPopulation("src", 200, S.ModelKind.PoissonSource, 1, S.PoissonParams(30.0)),
        S.NeuronPopulation("izh", n, S.ModelKind.Izhikevich, 2, S.IzhikevichParams(
            a=[float(x) for x in 0.02 + 0.08 * r], b=[float(x) for x in 0.25 - 0.05 * r],
            c=[-65.0] * n, d=[float(x) for x in 2.0 + 6.0 * r], noiseAmplitude=[3.0] * n,
            biasCurrent=[float(x) for x in 2.0 * r])),
        S.NeuronPopulation("out", 100, S.ModelKind.CondLif, 3, S.CondLifParams()),
    ]
    spec.synapses = [
        S.SynapseGroupSpec("in_e", "src", "izh", S.SynapseSign.Excitatory, 100,
                           S.WeightDist.uniform(0.0, 3.0), 1.0, S.StorageKind.Sparse),
        S.SynapseGroupSpec("in_i", "src", "izh", S.SynapseSign.Inhibitory, 50,
                           S.WeightDist.uniform(0.0, 2.0), 1.0, S.StorageKind.Dense, 100, 100),
        S.SynapseGroupSpec("fwd", "izh", "out", S.SynapseSign.Excitatory, 20,
                           S.WeightDist.uniform(0.0, 0.05), 1.0, S.StorageKind.Dense),
    ]
    return spec


def hh_mbody_spec(n_kc: int = 300, duration_ms: float = 30.0, seed: int = 7) -> S.NetworkSpec:
    """Mushroom body with Traub-Miles HH KCs (extension)."""
    o = S.MBodyBuildOptions(dtMs=0.1, durationMs=duration_ms, pnKcOutFraction=0.5,
                            kcModel=S.ModelKind.TraubMiles)
    return S.build_mbody_net(100, 20, n_kc, 100, {"pn_kc": 2.0, "pn_lhi": 1.0, "lhi_kc": 0.1,
                                                  "kc_dn": 30.0 / n_kc}, seed, o)


def stdp_mbody_spec(n_kc: int, duration_ms: float, frac: float = 0.05, seed: int = 7,
                    a_plus: float = 0.1, a_minus: float = 0.12, w_max: float = 3.0,
                    n_dn: int = 100):
    """Extension F2: the mushroom body with STDP on kc_dn (amplitudes and wMax
    relative to the built kc_dn weight)."""
    spec = mbody_spec(n_kc, frac, duration_ms, seed=seed, n_dn=n_dn)
    g = spec.synapses[spec.group_index("kc_dn")]
    w0 = g.baseWeight.value * g.gScale
    g.stdp = S.StdpRule(aPlus=a_plus * w0, aMinus=a_minus * w0, tauPlusMs=20.0,
                        tauMinusMs=15.0, wMax=w_max * w0)
    return spec


def spec_from_ref_desc(desc) -> S.NetworkSpec:
    """The product-side NetworkSpec view of a flat ssb_net_desc that the
    REFERENCE's own builder produced (oracle.RefDesc); a pure data conversion."""
    import ctypes as C
    from paper_1412_0595_b200 import _lib as L
    return S._spec_from_desc(C.cast(desc.ptr, C.POINTER(L.ssb_net_desc)).contents)


def spec_key(spec: S.NetworkSpec):
    """Every field of a spec as a comparable tuple (float arrays by their bytes)."""
    def val(x):
        if isinstance(x, (list, tuple, np.ndarray)):
            return np.ascontiguousarray(x, np.float64).tobytes()
        return x

    def fields(obj):
        if obj is None:
            return None
        return tuple((k, val(v) if not hasattr(v, "__dataclass_fields__") else fields(v))
                     for k, v in sorted(vars(obj).items()))
    return (spec.dtMs, spec.durationMs, spec.globalSeed,
            tuple(fields(p) for p in spec.populations), tuple(fields(g) for g in spec.synapses))


def ref_mbody_spec(n_kc: int, frac: float, duration_ms: float, seed: int = 7):
    """(RefDesc, spec view) of the mushroom body built by the reference's
    build_mbody_net (network.cpp:286-362) with the §8(d) gScales."""
    from oracle import oracle as O
    d = O.ref_mbody_desc(n_kc, frac, duration_ms, seed=seed)
    return d, spec_from_ref_desc(d)


def raster_checksum(step, pop, neuron) -> int:
    """Order-independent raster checksum (sum of mix64(step<<40 ^ pop<<32 ^ neuron)
    mod 2^64); the same function as bench.raster_checksum and the shim's
    ref_pool_raster_checksum."""
    import bench
    return bench.raster_checksum(step, pop, neuron)
