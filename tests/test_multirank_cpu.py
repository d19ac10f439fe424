"""Multi-process (gloo, CPU) tests of the split step path.

world_size 2 and 3 processes each hold one rank's shard -- the populations
the product library's ssb_shard_plan splits, the column slices ssb_shard_group
hands that rank -- advance it with the numpy restatement in shard_sim.py and
exchange spikes with torch.distributed all-gathers, as the NCCL path does per
window on the GPU.  The merged raster must equal the unsplit oracle's bit for
bit, and the ranks' slices must tile every group exactly.
"""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_path):
    sys.path[:0] = [ROOT, HERE]
    import specs
    from shard_sim import ShardSim
    from paper_1412_0595_b200 import synscale as S

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        spec = specs.mbody_spec(2000, 0.2, 20.0)
        mode = S.StorageMode.FromSpec
        plan = S.shard_plan(spec, world)
        assert plan["pn"] is None and plan["lhi"] is None  # small / Poisson: replicated
        assert plan["kc"] is not None and plan["dn"] is not None

        # the rank pipeline: dn (fed only by kc_dn) is owned by rank 0 and
        # kc_dn is split by kc rows
        assert plan["dn"] == [0] + [100] * world
        # the ranks' column (row) slices tile every group exactly
        for gi, g in enumerate(spec.synapses):
            kind, m = S.shard_group(spec, gi, world, rank, mode)
            parts = [None] * world
            dist.all_gather_object(parts, (kind, m))
            fk, full = S.build_group(spec, gi, mode)
            assert all(k == fk for k, _ in parts)
            b = plan[g.post]
            if g.name == "kc_dn":  # rows of each rank's kc range, in rank order
                assert np.array_equal(np.concatenate([p for _, p in parts], axis=0), full)
            elif b is None:  # whole post population: every rank holds the whole group
                for _, p in parts:
                    if fk == "dense":
                        assert np.array_equal(p, full)
                    else:
                        assert all(np.array_equal(x, y) for x, y in zip(p, full))
            elif fk == "dense":
                assert np.array_equal(np.concatenate([p for _, p in parts], axis=1), full)
            else:
                vals, ind, rs = full
                for r in range(len(rs) - 1):
                    got_i = np.concatenate([p[1][p[2][r]:p[2][r + 1]] + b[k]
                                            for k, (_, p) in enumerate(parts)])
                    got_v = np.concatenate([p[0][p[2][r]:p[2][r + 1]] for _, p in parts])
                    assert np.array_equal(got_i, ind[rs[r]:rs[r + 1]])
                    assert np.array_equal(got_v, vals[rs[r]:rs[r + 1]])

        def exchange(local):
            got = [None] * world
            dist.all_gather_object(got, local)
            return got

        def send(arr, dst):
            dist.send(torch.from_numpy(np.ascontiguousarray(arr, np.float32)), dst)

        def recv(n, src):
            t = torch.empty(n, dtype=torch.float32)
            dist.recv(t, src)
            return t.numpy()

        sim = ShardSim(spec, mode, world, rank, exchange, send=send, recv=recv)
        events = np.array(sim.run(), np.int64).reshape(-1, 3)
        flagged = [None] * world
        dist.all_gather_object(flagged, sim.flagged)
        if rank == 0:
            np.savez(out_path, events=events, flagged=np.array(flagged))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_split_ranks_match_unsplit_oracle(tmp_path, oracle_mod, world):
    import specs
    from paper_1412_0595_b200 import synscale as S

    out = str(tmp_path / "rank0.npz")
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    got = np.load(out)
    spec = specs.mbody_spec(2000, 0.2, 20.0)
    d = S.NetDesc(spec)
    o = oracle_mod.CpuSim(d.ptr, spec, int(S.StorageMode.FromSpec))
    step, pop, neuron = o.finish()
    ref = np.stack([step, pop, neuron], axis=1).astype(np.int64)
    assert len(ref) > 1000
    assert np.array_equal(got["events"], ref)
    assert int(got["flagged"].sum()) == o.sum_nans()
