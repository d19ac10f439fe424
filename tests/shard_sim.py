"""One rank of a split run, restated on the CPU with numpy (test infrastructure).

Checks the multi-GPU decomposition itself -- which populations a world
splits, each rank's column (or row) slices (both taken from the product
library's host code: ssb_shard_plan / ssb_shard_group), the spike exchange in
rank order and the rank pipeline of row-split groups (each rank continues the
previous rank's partial sums over its own pre rows, the last rank hands them
to rank 0, which owns the sink population) -- with real multi-process
communication (torch.distributed, gloo).  The
per-step arithmetic follows the reference step (engine.cpp:316-356) in numpy
float32, which rounds every operation like the reference's -ffp-contract=off
build; the merged raster is compared with the unsplit oracle in the test.
"""
from __future__ import annotations

import math

import numpy as np

from paper_1412_0595_b200 import synscale as S


class ShardSim:
    def __init__(self, spec: S.NetworkSpec, mode: S.StorageMode, world: int, rank: int,
                 exchange, min_size: int = 0, send=None, recv=None):
        """exchange(list_of_local_arrays) -> list (per rank) of those lists;
        send(float32 array, dst) / recv(n, src): the pipeline's point to point."""
        self.spec, self.world, self.rank, self.exchange = spec, world, rank, exchange
        self.send, self.recv = send, recv
        self.plan = S.shard_plan(spec, world, min_size)
        self.dt = np.float32(spec.dtMs)
        self.steps = max(1, math.ceil(spec.durationMs / spec.dtMs - 1e-9))
        self.pops = []
        for p in spec.populations:
            b = self.plan[p.name]
            lo, hi = (0, p.size) if b is None else (b[rank], b[rank + 1])
            st = {"name": p.name, "model": p.model, "lo": lo, "n": hi - lo, "N": p.size,
                  "split": b is not None, "bounds": b}
            if p.model == S.ModelKind.PoissonSource:
                st["p"] = p.params.rateHz * spec.dtMs / 1000.0
                # draw (t, i) is output t*N + i of the population's stream
                st["u"] = S.stream_u64(spec.globalSeed, p.seed, p.name + "/source",
                                       self.steps * p.size)
            else:
                c = p.params
                f = np.float32
                st.update(tauM=f(c.tauMMs), eLeak=f(c.eLeakMV), eExc=f(c.eExcMV),
                          eInh=f(c.eInhMV), vT=f(c.vThreshMV), vR=f(c.vResetMV),
                          decay=f(math.exp(-spec.dtMs / c.tauSynMs)))
                n = hi - lo
                st["v"] = np.full(n, st["eLeak"], np.float32)
                st["gE"] = np.zeros(n, np.float32)
                st["gI"] = np.zeros(n, np.float32)
                st["flag"] = np.zeros(n, np.uint8)
            st["exc"] = np.zeros(hi - lo, np.float32)
            st["inh"] = np.zeros(hi - lo, np.float32)
            self.pops.append(st)
        self.groups = []
        for gi, g in enumerate(spec.synapses):
            kind, m = S.shard_group(spec, gi, world, rank, mode, min_size)
            pre, post = spec.pop_index(g.pre), spec.pop_index(g.post)
            pb, qb = self.plan[g.pre], self.plan[g.post]
            # row split (rank pipeline): rank 0 owns the post population, this
            # rank holds its own pre rows x every post column
            rows = (kind == "dense" and pb is not None and qb is not None and world > 1 and
                    qb[1] == spec.populations[post].size and
                    m.shape == (pb[rank + 1] - pb[rank], spec.populations[post].size))
            self.groups.append({"pre": pre, "post": post,
                                "inh": g.sign == S.SynapseSign.Inhibitory,
                                "off": g.preOffset, "kind": kind, "m": m, "rows": rows})
        self.events = []  # (step, pop, neuron), global ids
        self.t = 0
        self.flagged = 0

    def _poisson(self, st):
        n = st["N"]
        u = st["u"][self.t * n:(self.t + 1) * n]
        # uniform01() < p  (random.hpp:48)
        return np.nonzero((u >> np.uint64(11)).astype(np.float64) * 2.0 ** -53 < st["p"])[0]

    def step(self):
        local = []
        for st in self.pops:  # advance, flag, threshold (engine.cpp:251-314)
            if st["model"] == S.ModelKind.PoissonSource:
                local.append(self._poisson(st))
                continue
            v, gE, gI = st["v"], st["gE"], st["gI"]
            ge = gE * st["decay"] + st["exc"]
            gi = gI * st["decay"] - st["inh"]
            v = v + self.dt * (((st["eLeak"] - v) / st["tauM"] + ge * (st["eExc"] - v)) +
                               gi * (st["eInh"] - v))
            bad = ~(np.isfinite(v) & np.isfinite(ge) & np.isfinite(gi)) & (st["flag"] == 0)
            st["flag"][bad] = 1
            self.flagged += int(bad.sum())
            spk = np.nonzero(v >= st["vT"])[0]
            v[spk] = st["vR"]
            st["v"], st["gE"], st["gI"] = v, ge, gi
            local.append(spk)
        # the exchange: split populations' local spikes, all ranks, rank order
        gathered = self.exchange([s + st["lo"] for s, st in zip(local, self.pops)])
        spikes = []
        for pi, st in enumerate(self.pops):
            if st["split"]:
                spikes.append(np.concatenate([g[pi] for g in gathered]).astype(np.int64))
            else:
                spikes.append(local[pi].astype(np.int64))
        for pi, s in enumerate(spikes):  # record (engine.cpp:328-333)
            self.events.extend((self.t, pi, int(i)) for i in s)
        for st in self.pops:  # zero (engine.cpp:336-339)
            st["exc"][:] = 0
            st["inh"][:] = 0
        for g in self.groups:  # propagate in spec order (engine.cpp:343-355)
            acc = self.pops[g["post"]]["inh" if g["inh"] else "exc"]
            if g["rows"]:  # rank pipeline over this rank's own (local) spiking rows
                n = g["m"].shape[1]
                part = (np.zeros(n, np.float32) if self.rank == 0
                        else self.recv(n, self.rank - 1))
                for r in local[g["pre"]]:
                    part += g["m"][r]
                self.send(part, self.rank + 1 if self.rank < self.world - 1 else 0)
                if self.rank == 0:
                    acc += self.recv(n, self.world - 1)  # acc is +0: exact
                continue
            rows = spikes[g["pre"]] - g["off"]
            if g["kind"] == "dense":
                W = g["m"]
                rows = rows[(rows >= 0) & (rows < W.shape[0])]
                for r in rows:
                    acc += W[r]  # zero entries add +0 (the fold never holds -0)
            else:
                vals, ind, rs = g["m"]
                rows = rows[(rows >= 0) & (rows < len(rs) - 1)]
                for r in rows:
                    a, b = rs[r], rs[r + 1]
                    acc[ind[a:b]] += vals[a:b]
        self.t += 1

    def run(self):
        while self.t < self.steps:
            self.step()
        return self.events
