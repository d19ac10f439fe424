"""Generates the golden fixtures in tests/golden/ from the REFERENCE itself.

Run in the build container (it needs oracle/_ref/libsynscale_ref.so, which is
compiled from /root/reference/proj by oracle/Makefile):

    python tests/golden/make_golden.py

Everything recorded here comes out of the unmodified reference library
through its public C++ API (Simulation / gen_fixed_outdegree / RandomStream /
derive_seed, via oracle/ref_shim.cpp).  The fixtures pin the oracle
restatement and the CUDA path on machines where /root/reference is absent.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from oracle import oracle as O  # noqa: E402
from paper_1412_0595_b200 import synscale as S  # noqa: E402
import specs  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))

STREAMS = [(7, 1, "pn/source"), (11, 1, "drive/source"), (11, 2, "damp/source"),
           (42, 7, "pop/noise"), (0, 0, "gen/targets")]
SEEDS = [(7, "pn_kc"), (7, "pn_lhi"), (7, "lhi_kc"), (7, "kc_dn"), (9, "exc"), (9, "inh")]
GENS = [  # nPre, nPost, k, kind, lo, hi, value, sign, seed
    (5, 8, 3, S.L.WEIGHT_UNIFORM, 0.0, 0.5, 0.0, 1, 99),
    (3, 4, 2, S.L.WEIGHT_CONSTANT, 0.0, 0.0, 2.0, -1, 7),
    (50, 80, 13, S.L.WEIGHT_UNIFORM, 0.0, 0.5, 0.0, 1, 99),
    (100, 1000, 500, S.L.WEIGHT_UNIFORM, 0.0, 0.02, 0.0, 1, 2921146032820891623),
]


def run_ref(spec, mode, desc=None, light=False):
    """One reference run.  `desc`: a flat spec the reference's own builder made
    (the mushroom-body and Izhikevich runs); otherwise `spec` flattened."""
    d = desc if desc is not None else S.NetDesc(spec)
    sim = O.CpuSim(d.ptr, spec, int(mode), ref=True)
    step, pop, neu = sim.finish()
    out = {
        "n_events": int(step.size),
        "raster_sha": specs.sha(step, pop, neu),
        "rates": [float(x) for x in sim.rates()],
        "sum_nans": sim.sum_nans(),
        "counts": [int(np.count_nonzero(pop == i)) for i in range(len(spec.populations))],
        "state_sha": {},
        "groups": {},
        "head": [[int(a), int(b), int(c)] for a, b, c in zip(step[:40], pop[:40], neu[:40])],
        "checksum": str(specs.raster_checksum(step, pop, neu)),
    }
    if light:
        del out["groups"]
    for pi, p in enumerate(spec.populations):
        fields = ("v", "gExc", "gInh", "excIn", "inhIn", "nanFlag")
        if p.model == S.ModelKind.Izhikevich:
            fields = ("v", "u", "excIn", "inhIn", "nanFlag")
        out["state_sha"][p.name] = {f: specs.sha(sim.state(pi, f)) for f in fields}
    for gi, g in enumerate(spec.synapses if not light else []):
        kind, m = sim.group(gi)
        out["groups"][g.name] = [kind, specs.sha(*(m if kind == "sparse" else (m,)))]
    return out


def main():
    if not O.have_ref():
        O.build()
    gold = {"source": "reference (oracle/_ref/libsynscale_ref.so from /root/reference/proj)"}
    gold["streams"] = {f"{g}/{e}/{lab}": [str(int(x)) for x in O.stream_u64(g, e, lab, 16, ref=True)]
                       for g, e, lab in STREAMS}
    gold["derive_seed"] = {f"{p}/{lab}": str(int(O.ref_lib().ref_derive_seed(p, lab.encode())))
                           for p, lab in SEEDS}
    gens = []
    for args in GENS:
        m = O.gen_fixed_outdegree(*args, ref=True)
        entry = {"args": [str(a) if isinstance(a, int) and a > 2**31 else a for a in args],
                 "sha": specs.sha(m), "nnz": int(np.count_nonzero(m))}
        if m.size <= 64:
            entry["weights"] = m.ravel().view(np.uint32).tolist()
        gens.append(entry)
    gold["gen_fixed_outdegree"] = gens

    def mbody(cfg, ms):
        """(desc, spec) of BASELINE config `cfg` from the reference's build_mbody_net."""
        n_kc, frac, _ = specs.CONFIGS[cfg]
        return specs.ref_mbody_spec(n_kc, frac, ms)

    def izh(duration_ms=1000.0, dense=False):
        d = O.ref_izh_desc(1000, 100, 0.8, 6.0, 1, duration_ms=duration_ms, dense=dense)
        return d, specs.spec_from_ref_desc(d)

    M = S.StorageMode
    runs = {}
    for name, (built, mode, light) in {
        "cfg1_1000ms": (mbody(1, 1000.0), M.ForceDense, False),
        "cfg2_100ms": (mbody(2, 100.0), M.ForceSparse, False),
        "cfg3_20ms": (mbody(3, 20.0), M.FromSpec, False),
        "cfg1_sparse_300ms": (mbody(1, 300.0), M.ForceSparse, False),
        "cfg2_fromspec_100ms": (mbody(2, 100.0), M.FromSpec, False),
        "chain_100ms": ((None, specs.chain_spec(100.0)), M.FromSpec, False),
        "recurrent_200ms": ((None, specs.recurrent_lif_spec()), M.FromSpec, False),
        "izh_1000_1000ms": (izh(), M.FromSpec, False),
        "izh_1000_dense_300ms": (izh(300.0), M.ForceDense, False),
        "izh_ff_200ms": ((None, specs.izh_ff_spec()), M.FromSpec, False),
        # BASELINE config 3 over its whole 1 s (10,000 steps) and config 4
        # (1M KC) over 100 ms (1,000 steps, four 256-step windows)
        "cfg3_1000ms": (mbody(3, 1000.0), M.FromSpec, True),
        "cfg4_100ms": (mbody(4, 100.0), M.FromSpec, True),
    }.items():
        print("reference run", name, flush=True)
        desc, spec = built
        runs[name] = run_ref(spec, mode, desc, light)
    gold["runs"] = runs

    # bench.py's end-of-run parity check: the split network of N x 100k KC
    # (and config 4) over 100 ms, as spike counts + order-independent raster
    # checksum (bench.raster_checksum); the reference's own builder and engine
    bp = {"source": gold["source"], "duration_ms": 100.0,
          "checksum": "sum of mix64(step<<40 ^ pop<<32 ^ neuron) mod 2^64 (bench.raster_checksum)",
          "runs": {}}
    for key, n_kc in (("split1", 100_000), ("split2", 200_000), ("split4", 400_000),
                      ("split8", 800_000), ("cfg4", 1_000_000)):
        print("reference parity run", key, flush=True)
        pool = O.RefPool(n_kc, 0.05, 100.0, 1)
        pool.step(pool.steps_total())
        bp["runs"][key] = {"n_kc": n_kc, "counts": [int(c) for c in pool.counts(0, 1 << 62)],
                           "checksum": str(pool.raster_checksum())}
        pool.close()
    with open(os.path.join(OUT, "bench_parity.json"), "w") as f:
        json.dump(bp, f, indent=1, sort_keys=True)

    # CondLif + Poisson known-answer network (test_engine.cpp:183-290): the
    # reference's per-step v / gExc / gInh of the single conductance neuron.
    kat = specs.condlif_kat_spec()
    d = S.NetDesc(kat)
    sim = O.CpuSim(d.ptr, kat, 0, ref=True)
    v, ge, gi = [], [], []
    for _ in range(sim.steps_total()):
        sim.step(1)
        v.append(sim.state(2, "v")[0])
        ge.append(sim.state(2, "gExc")[0])
        gi.append(sim.state(2, "gInh")[0])
    step, pop, neu = sim.finish()
    np.savez_compressed(os.path.join(OUT, "condlif_kat.npz"), v=np.array(v, np.float32),
                        gExc=np.array(ge, np.float32), gInh=np.array(gi, np.float32),
                        step=step, pop=pop, neuron=neu)

    # Izhikevich known answer (test_engine.cpp:79-111): one bias-driven neuron,
    # per-step v / u from the reference.
    one = specs.single_izh_spec()
    d = S.NetDesc(one)
    sim = O.CpuSim(d.ptr, one, 0, ref=True)
    v, u = [], []
    for _ in range(sim.steps_total()):
        sim.step(1)
        v.append(sim.state(0, "v")[0])
        u.append(sim.state(0, "u")[0])
    step, pop, neu = sim.finish()
    np.savez_compressed(os.path.join(OUT, "izh_kat.npz"), v=np.array(v, np.float32),
                        u=np.array(u, np.float32), step=step, pop=pop, neuron=neu)

    with open(os.path.join(OUT, "golden.json"), "w") as f:
        json.dump(gold, f, indent=1, sort_keys=True)
    print("wrote", os.path.join(OUT, "golden.json"))


if __name__ == "__main__":
    main()
