"""The product's spec builders against the REFERENCE's own builders
(build_mbody_net network.cpp:286-362, build_izhikevich_net :198-284, compiled
into oracle/_ref), field by field, and the bench's reference arm plumbing."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

import specs
from paper_1412_0595_b200 import synscale as S

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def O(oracle_mod):
    if not oracle_mod.have_ref():
        pytest.skip("oracle/_ref not built (reference sources absent)")
    return oracle_mod


@pytest.mark.parametrize("n_kc,frac,ms,seed", [
    (1_000, 0.5, 1000.0, 7), (10_000, 0.05, 100.0, 7), (100_000, 0.05, 1000.0, 7),
    (1_000_000, 0.05, 100.0, 7), (800_000, 0.05, 100.0, 7), (37, 0.3, 12.5, 123456789),
    (5, 0.0001, 1.0, 2**64 - 1)])
def test_mbody_builder_equals_reference(O, n_kc, frac, ms, seed):
    d, ref = specs.ref_mbody_spec(n_kc, frac, ms, seed=seed)
    mine = specs.mbody_spec(n_kc, frac, ms, seed=seed)
    assert specs.spec_key(mine) == specs.spec_key(ref)
    # the flattened forms too (what the engine and the reference consume)
    assert [g.outDegree for g in mine.synapses] == [g.outDegree for g in ref.synapses]
    assert [p.seed for p in mine.populations] == [p.seed for p in ref.populations]


@pytest.mark.parametrize("n,conn,exc,g,seed,dense", [
    (1000, 100, 0.8, 6.0, 1, False), (1000, 100, 0.8, 6.0, 1, True), (257, 13, 0.31, 0.5, 99, False)])
def test_izhikevich_builder_equals_reference(O, n, conn, exc, g, seed, dense):
    d = O.ref_izh_desc(n, conn, exc, g, seed, dense=dense, duration_ms=300.0)
    ref = specs.spec_from_ref_desc(d)
    opt = S.IzhBuildOptions(dtMs=1.0, durationMs=300.0,
                            storage=S.StorageKind.Dense if dense else S.StorageKind.Sparse)
    mine = S.build_izhikevich_net(n, conn, exc, g, seed, opt)
    assert specs.spec_key(mine) == specs.spec_key(ref)


def test_builder_errors_match_reference(O):
    for args in ((0, 0.05), (10, float("nan"))):
        with pytest.raises(ValueError):
            O.ref_mbody_desc(args[0], 0.05, 10.0, gscales=(args[1], 1.0, 0.1, 0.1))
        with pytest.raises((ValueError, S.SpecError)):
            S.build_mbody_net(100, 20, args[0], 100, {"pn_kc": args[1], "pn_lhi": 1.0,
                                                      "lhi_kc": 0.1, "kc_dn": 0.1}, 7,
                              S.MBodyBuildOptions())


def test_bench_checksum_equals_reference_shim(O):
    """bench.raster_checksum (numpy) == the shim's checksum of the same reference raster."""
    pool = O.RefPool(2000, 0.05, 30.0, 1)
    pool.step(pool.steps_total())
    d, spec = specs.ref_mbody_spec(2000, 0.05, 30.0)
    sim = O.CpuSim(d.ptr, spec, 0, ref=True)
    step, pop, neu = sim.finish()
    assert step.size > 100
    assert specs.raster_checksum(step, pop, neu) == pool.raster_checksum()
    assert list(pool.counts(0, 1 << 62)) == [int(np.count_nonzero(pop == i)) for i in range(4)]


def test_bench_parity_golden_matches_reference_runs(O):
    """bench_parity.json's split1 entry equals golden.json's cfg3 prefix data
    source: a fresh reference run over 100 ms of config 3 (the unsplit network)."""
    with open(os.path.join(ROOT, "tests", "golden", "bench_parity.json")) as f:
        bp = json.load(f)["runs"]
    assert set(bp) == {"split1", "split2", "split4", "split8", "cfg4"}
    pool = O.RefPool(100_000, 0.05, 100.0, 1)
    pool.step(pool.steps_total())
    assert [int(c) for c in pool.counts(0, 1 << 62)] == bp["split1"]["counts"]
    assert pool.raster_checksum() == int(bp["split1"]["checksum"])


def test_bench_reference_arm_imports_no_product_code(O):
    """--impl reference runs the reference library alone: after a (shrunk)
    run, no module of the product package is loaded and no product .so is
    mapped into the process."""
    code = (
        "import sys, json; sys.argv=['bench.py','--impl','reference','--steps','1',"
        "'--warmup','3']; import bench; bench.N_KC=2000; bench.main(); "
        "mods=[m for m in sys.modules if m.startswith('paper_1412_0595_b200')]; "
        "maps=open('/proc/self/maps').read(); "
        "print(json.dumps({'mods': mods, 'so': 'libsynscale_b200' in maps}))")
    out = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True,
                         timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(x) for x in out.stdout.splitlines() if x.startswith("{")]
    line, probe = lines[0], lines[-1]
    assert probe == {"mods": [], "so": False}
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "reference"
    import bench
    assert line["config"] == json.loads(json.dumps(bench.bench_config(1, 256) | {
        "n_kc": 2000, "gscales": bench.gscales(2000),
        "workload": line["config"]["workload"]}))


def test_bench_gpus_flag_launches_ranks():
    """bench.py --gpus 2 without WORLD_SIZE re-launches itself under
    torch.distributed.run with two ranks (RANK / LOCAL_RANK / WORLD_SIZE set)."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--launch-probe"], cwd=ROOT,
                         capture_output=True, text=True, timeout=300, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    ranks = sorted((json.loads(x)["rank"], json.loads(x)["local_rank"], json.loads(x)["world"])
                   for x in out.stdout.splitlines() if x.startswith("{"))
    assert ranks == [(0, 0, 2), (1, 1, 2)]


def test_bench_config_identical_in_both_arms():
    import bench
    for world in (1, 2, 8):
        a = bench.bench_config(world, 256)
        assert a["n_kc"] == 100_000 * world
        assert a["gscales"]["kc_dn"] == 30.0 / (100_000 * world)
