"""Python mirror of the reference's model-definition and run API.

Same names and argument meaning as the reference C++ API
(/root/reference/proj/include/synscale/{network,engine,matrix,occupancy}.hpp):
``NetworkSpec``, ``build_mbody_net``, ``build_izhikevich_net``, ``validate``,
``Simulation`` (``step``/``population_state``/``group_dense``/
``group_sparse``/``finish``), ``run``, ``propagate``, ``detect_nans``,
``avg_spike``, ``raster_to_csv`` and the occupancy model.  Misuse raises
``SpecError`` exactly where the reference throws ``SpecError``.

Everything below is a thin layer over the C ABI (``_lib``); spec building,
connectivity generation and validation run in the C++ host library, the
simulation step runs in the sm_100a kernels.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple, Union

import numpy as np

from . import _lib as L

lib = L.lib


class SpecError(ValueError):
    """The reference's SpecError (common.hpp:20-23): bad input or misuse."""


class DeviceError(RuntimeError):
    """CUDA / internal failure (SSB_ERR_INTERNAL)."""


def _raise(rc: int, msg: str) -> None:
    if rc == L.SSB_OK:
        return
    if rc == L.SSB_ERR_SPEC:
        raise SpecError(msg)
    raise DeviceError(msg)


def _err() -> C.Array:
    return C.create_string_buffer(2048)


def _fptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_float))


def _iptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_int32))


def _lptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_int64))


# ---- model definition (network.hpp) -------------------------------------------


class ModelKind(enum.IntEnum):
    Izhikevich = L.MODEL_IZHIKEVICH
    PoissonSource = L.MODEL_POISSON
    CondLif = L.MODEL_CONDLIF
    TraubMiles = L.MODEL_TRAUBMILES  # extension (F1): Traub-Miles HH


class SynapseSign(enum.IntEnum):
    Excitatory = L.SIGN_EXC
    Inhibitory = L.SIGN_INH


class StorageKind(enum.IntEnum):
    Dense = L.STORAGE_DENSE
    Sparse = L.STORAGE_SPARSE


class StorageMode(enum.IntEnum):
    FromSpec = L.MODE_FROM_SPEC
    ForceDense = L.MODE_FORCE_DENSE
    ForceSparse = L.MODE_FORCE_SPARSE
    Auto = L.MODE_AUTO  # extension: dense iff outDegree / nPost >= auto_dense_threshold()


@dataclass
class WeightDist:
    kind: str = "constant"  # "constant" | "uniform"
    lo: float = 0.0
    hi: float = 0.0
    value: float = 0.0

    @staticmethod
    def uniform(lo: float, hi: float) -> "WeightDist":
        if not (np.isfinite(lo) and np.isfinite(hi)) or lo < 0.0 or not lo < hi:
            raise SpecError(f"uniform weight range [{lo}, {hi}) needs finite 0 <= lo < hi")
        return WeightDist("uniform", lo, hi, 0.0)

    @staticmethod
    def constant(value: float) -> "WeightDist":
        if not np.isfinite(value) or not value > 0.0:
            raise SpecError(f"constant weight {value} must be finite and > 0")
        return WeightDist("constant", 0.0, 0.0, value)


@dataclass
class PoissonParams:
    rateHz: float = 0.0


@dataclass
class CondLifParams:
    tauMMs: float = 10.0
    eLeakMV: float = -60.0
    vThreshMV: float = -45.0
    vResetMV: float = -60.0
    eExcMV: float = 0.0
    eInhMV: float = -80.0
    tauSynMs: float = 5.0


@dataclass
class IzhikevichParams:
    a: Sequence[float] = ()
    b: Sequence[float] = ()
    c: Sequence[float] = ()
    d: Sequence[float] = ()
    noiseAmplitude: Sequence[float] = ()
    biasCurrent: Sequence[float] = ()


@dataclass
class NeuronPopulation:
    name: str
    size: int
    model: ModelKind = ModelKind.Izhikevich
    seed: int = 0
    params: Union[IzhikevichParams, PoissonParams, CondLifParams] = field(
        default_factory=IzhikevichParams)


@dataclass
class StdpRule:
    """Extension F2 (not in the reference): pair-based STDP on a
    dense all-to-all excitatory group; the rule is include/synscale/synscale.hpp
    StdpRule's (DESIGN.md §1 row A22)."""
    aPlus: float = 0.0
    aMinus: float = 0.0
    tauPlusMs: float = 20.0
    tauMinusMs: float = 20.0
    wMax: float = 0.0


@dataclass
class SynapseGroupSpec:
    name: str
    pre: str
    post: str
    sign: SynapseSign = SynapseSign.Excitatory
    outDegree: int = 0
    baseWeight: WeightDist = field(default_factory=WeightDist)
    gScale: float = 1.0
    storage: StorageKind = StorageKind.Sparse
    preOffset: int = 0
    preCount: int = -1
    stdp: Optional[StdpRule] = None  # extension F2


@dataclass
class NetworkSpec:
    populations: List[NeuronPopulation] = field(default_factory=list)
    synapses: List[SynapseGroupSpec] = field(default_factory=list)
    dtMs: float = 1.0
    durationMs: float = 1000.0
    globalSeed: int = 0

    def find_population(self, name: str) -> Optional[NeuronPopulation]:
        for p in self.populations:
            if p.name == name:
                return p
        return None

    def pop_index(self, name: str) -> int:
        for i, p in enumerate(self.populations):
            if p.name == name:
                return i
        raise SpecError(f"unknown population '{name}'")

    def group_index(self, name: str) -> int:
        for i, g in enumerate(self.synapses):
            if g.name == name:
                return i
        raise SpecError(f"unknown synapse group '{name}'")


@dataclass
class TraubMilesParams:
    """Extension: GeNN's Traub-Miles HH neuron with CondLif-style
    conductance synapses; not in the reference (parity is against oracle.c)."""
    gNa: float = 7.15
    ENa: float = 50.0
    gK: float = 1.43
    EK: float = -95.0
    gl: float = 0.02672
    El: float = -63.563
    C: float = 0.143
    eExcMV: float = 0.0
    eInhMV: float = -92.0
    tauSynMs: float = 3.0
    substeps: int = 25


@dataclass
class MBodyBuildOptions:
    dtMs: float = 1.0
    durationMs: float = 1000.0
    pnRateHz: float = 50.0
    pnKcOutFraction: float = 0.5
    lif: CondLifParams = field(default_factory=CondLifParams)
    pnKcWeightHi: float = 0.02
    pnLhiWeight: float = 0.02
    lhiKcWeight: float = 0.01
    kcDnWeight: float = 0.01
    kcModel: "ModelKind" = None  # extension: ModelKind.TraubMiles for HH KCs
    kcHH: TraubMilesParams = field(default_factory=TraubMilesParams)


@dataclass
class IzhBuildOptions:
    dtMs: float = 1.0
    durationMs: float = 1000.0
    noiseExc: float = 5.0
    noiseInh: float = 2.0
    excWeightHi: float = 0.5
    inhWeightHi: float = 1.0
    biasCurrent: float = 0.0
    storage: StorageKind = StorageKind.Sparse


class NetDesc:
    """A NetworkSpec flattened into the C ABI's ssb_net_desc (keeps its buffers alive)."""

    def __init__(self, spec: NetworkSpec):
        self._keep = []
        pops = (L.ssb_pop_desc * max(1, len(spec.populations)))()
        for i, p in enumerate(spec.populations):
            d = pops[i]
            d.name = p.name.encode()
            d.size = int(p.size)
            d.model = int(p.model)
            d.seed = int(p.seed) & 0xFFFFFFFFFFFFFFFF
            prm = p.params
            if isinstance(prm, PoissonParams):
                d.rate_hz = float(prm.rateHz)
            elif isinstance(prm, CondLifParams):
                d.tau_m_ms, d.e_leak_mv, d.v_thresh_mv = prm.tauMMs, prm.eLeakMV, prm.vThreshMV
                d.v_reset_mv, d.e_exc_mv, d.e_inh_mv = prm.vResetMV, prm.eExcMV, prm.eInhMV
                d.tau_syn_ms = prm.tauSynMs
            elif isinstance(prm, TraubMilesParams):
                d.hh_gna, d.hh_ena, d.hh_gk, d.hh_ek = prm.gNa, prm.ENa, prm.gK, prm.EK
                d.hh_gl, d.hh_el, d.hh_c = prm.gl, prm.El, prm.C
                d.e_exc_mv, d.e_inh_mv, d.tau_syn_ms = prm.eExcMV, prm.eInhMV, prm.tauSynMs
                d.hh_substeps = int(prm.substeps)
            elif isinstance(prm, IzhikevichParams):
                for attr, key in (("izh_a", "a"), ("izh_b", "b"), ("izh_c", "c"), ("izh_d", "d"),
                                  ("izh_noise", "noiseAmplitude"), ("izh_bias", "biasCurrent")):
                    arr = np.ascontiguousarray(getattr(prm, key), dtype=np.float64)
                    self._keep.append(arr)
                    setattr(d, attr, arr.ctypes.data_as(C.POINTER(C.c_double)))
        groups = (L.ssb_group_desc * max(1, len(spec.synapses)))()
        for i, g in enumerate(spec.synapses):
            d = groups[i]
            d.name, d.pre, d.post = g.name.encode(), g.pre.encode(), g.post.encode()
            d.sign = int(g.sign)
            d.out_degree = int(g.outDegree)
            d.weight_kind = L.WEIGHT_UNIFORM if g.baseWeight.kind == "uniform" else L.WEIGHT_CONSTANT
            d.weight_lo, d.weight_hi = g.baseWeight.lo, g.baseWeight.hi
            d.weight_value = g.baseWeight.value
            d.g_scale = float(g.gScale)
            d.storage = int(g.storage)
            d.pre_offset = int(g.preOffset)
            d.pre_count = int(g.preCount)
            if g.stdp is not None:
                d.plasticity = L.PLASTICITY_STDP
                d.stdp_a_plus, d.stdp_a_minus = float(g.stdp.aPlus), float(g.stdp.aMinus)
                d.stdp_tau_plus_ms = float(g.stdp.tauPlusMs)
                d.stdp_tau_minus_ms = float(g.stdp.tauMinusMs)
                d.stdp_w_max = float(g.stdp.wMax)
        self._pops, self._groups = pops, groups
        self.desc = L.ssb_net_desc(len(spec.populations), pops, len(spec.synapses), groups,
                                   float(spec.dtMs), float(spec.durationMs),
                                   int(spec.globalSeed) & 0xFFFFFFFFFFFFFFFF)

    @property
    def ptr(self):
        return C.byref(self.desc)


def _spec_from_desc(d: L.ssb_net_desc) -> NetworkSpec:
    spec = NetworkSpec(dtMs=d.dt_ms, durationMs=d.duration_ms, globalSeed=d.global_seed)
    for i in range(d.n_pops):
        p = d.pops[i]
        model = ModelKind(p.model)
        if model == ModelKind.PoissonSource:
            prm = PoissonParams(p.rate_hz)
        elif model == ModelKind.CondLif:
            prm = CondLifParams(p.tau_m_ms, p.e_leak_mv, p.v_thresh_mv, p.v_reset_mv,
                                p.e_exc_mv, p.e_inh_mv, p.tau_syn_ms)
        elif model == ModelKind.TraubMiles:
            prm = TraubMilesParams(p.hh_gna, p.hh_ena, p.hh_gk, p.hh_ek, p.hh_gl, p.hh_el, p.hh_c,
                                   p.e_exc_mv, p.e_inh_mv, p.tau_syn_ms, p.hh_substeps)
        else:
            n = p.size
            prm = IzhikevichParams(*[np.ctypeslib.as_array(getattr(p, f), (n,)).copy()
                                     for f in ("izh_a", "izh_b", "izh_c", "izh_d", "izh_noise",
                                               "izh_bias")])
        spec.populations.append(NeuronPopulation(p.name.decode(), p.size, model, p.seed, prm))
    for i in range(d.n_groups):
        g = d.groups[i]
        w = (WeightDist("uniform", g.weight_lo, g.weight_hi, 0.0)
             if g.weight_kind == L.WEIGHT_UNIFORM else WeightDist("constant", 0.0, 0.0,
                                                                  g.weight_value))
        spec.synapses.append(SynapseGroupSpec(
            g.name.decode(), g.pre.decode(), g.post.decode(), SynapseSign(g.sign), g.out_degree,
            w, g.g_scale, StorageKind(g.storage), g.pre_offset, g.pre_count,
            StdpRule(g.stdp_a_plus, g.stdp_a_minus, g.stdp_tau_plus_ms, g.stdp_tau_minus_ms,
                     g.stdp_w_max) if g.plasticity == L.PLASTICITY_STDP else None))
    return spec


def build_mbody_net(nPN: int, nLHI: int, nKC: int, nDN: int, gScales: Dict[str, float],
                    seed: int, opt: Optional[MBodyBuildOptions] = None) -> NetworkSpec:
    """build_mbody_net (reference network.cpp:286-362), via the C++ builder."""
    opt = opt or MBodyBuildOptions()
    extra = set(gScales) - {"pn_kc", "pn_lhi", "lhi_kc", "kc_dn"}
    if extra:
        raise SpecError(f"gScales names an unknown synapse group '{sorted(extra)[0]}'")
    for g in ("pn_kc", "pn_lhi", "lhi_kc", "kc_dn"):
        if g not in gScales:
            raise SpecError(f"gScales has no entry for synapse group '{g}'")
    o = L.ssb_mbody_opts()
    o.dt_ms, o.duration_ms, o.pn_rate_hz = opt.dtMs, opt.durationMs, opt.pnRateHz
    o.pn_kc_out_fraction = opt.pnKcOutFraction
    o.tau_m_ms, o.e_leak_mv, o.v_thresh_mv = opt.lif.tauMMs, opt.lif.eLeakMV, opt.lif.vThreshMV
    o.v_reset_mv, o.e_exc_mv, o.e_inh_mv = opt.lif.vResetMV, opt.lif.eExcMV, opt.lif.eInhMV
    o.tau_syn_ms = opt.lif.tauSynMs
    o.pn_kc_weight_hi, o.pn_lhi_weight = opt.pnKcWeightHi, opt.pnLhiWeight
    o.lhi_kc_weight, o.kc_dn_weight = opt.lhiKcWeight, opt.kcDnWeight
    o.kc_model = int(opt.kcModel) if opt.kcModel is not None else L.MODEL_CONDLIF
    h = opt.kcHH
    o.hh_gna, o.hh_ena, o.hh_gk, o.hh_ek = h.gNa, h.ENa, h.gK, h.EK
    o.hh_gl, o.hh_el, o.hh_c, o.hh_e_inh_mv, o.kc_tau_syn_ms = h.gl, h.El, h.C, h.eInhMV, h.tauSynMs
    o.hh_substeps = h.substeps
    if o.kc_model == L.MODEL_TRAUBMILES and h.eExcMV != opt.lif.eExcMV:
        raise SpecError("the HH KCs share eExcMV with the CondLif populations in this builder")
    gs = (C.c_double * 4)(gScales["pn_kc"], gScales["pn_lhi"], gScales["lhi_kc"], gScales["kc_dn"])
    out = C.POINTER(L.ssb_net_desc)()
    err = _err()
    _raise(lib.ssb_build_mbody(nPN, nLHI, nKC, nDN, gs, seed & 0xFFFFFFFFFFFFFFFF, C.byref(o),
                               C.byref(out), err, len(err)), err.value.decode())
    try:
        return _spec_from_desc(out.contents)
    finally:
        lib.ssb_net_desc_free(out)


def build_izhikevich_net(nNeurons: int, nConn: int, excFraction: float, gScale: float, seed: int,
                         opt: Optional[IzhBuildOptions] = None) -> NetworkSpec:
    """build_izhikevich_net (reference network.cpp:198-284), via the C++ builder."""
    opt = opt or IzhBuildOptions()
    o = L.ssb_izh_opts(opt.dtMs, opt.durationMs, opt.noiseExc, opt.noiseInh, opt.excWeightHi,
                       opt.inhWeightHi, opt.biasCurrent, int(opt.storage))
    out = C.POINTER(L.ssb_net_desc)()
    err = _err()
    _raise(lib.ssb_build_izhikevich(nNeurons, nConn, excFraction, gScale,
                                    seed & 0xFFFFFFFFFFFFFFFF, C.byref(o), C.byref(out), err,
                                    len(err)), err.value.decode())
    try:
        return _spec_from_desc(out.contents)
    finally:
        lib.ssb_net_desc_free(out)


def validate(spec: NetworkSpec) -> List[Tuple[str, str]]:
    """validate (reference network.hpp:89-91): every violation as (field, message)."""
    buf = C.create_string_buffer(1 << 16)
    desc = NetDesc(spec)  # keeps the flattened arrays alive across the call
    n = lib.ssb_validate(desc.ptr, buf, len(buf))
    if n < 0:
        raise SpecError(buf.value.decode())
    out = []
    for line in buf.value.decode().splitlines():
        f, _, m = line.partition(": ")
        out.append((f, m))
    return out


def require_valid(spec: NetworkSpec) -> None:
    v = validate(spec)
    if v:
        raise SpecError("invalid network spec:\n" + "\n".join(f"  {f}: {m}" for f, m in v))


# ---- engine (engine.hpp) ----------------------------------------------------------


@dataclass
class EngineOptions:
    """B200 engine knobs (no reference counterpart); 0 = default."""
    device: int = 0
    window: int = 0
    blockSize: int = 0
    blockPolicy: int = 0
    useGraphs: bool = True
    heavyPreThreshold: int = 0
    rasterCapacity: int = 0
    profile: bool = False
    forceStepMode: bool = False
    # multi-GPU: one process per GPU, rank of world, NCCL id
    # from comm_unique_id() on rank 0 (broadcast by the caller); virtualWorld > 1
    # runs that many shards in this process on one GPU (tests the split path)
    rank: int = 0
    world: int = 1
    virtualWorld: int = 0
    shardMinSize: int = 0
    commId: Optional[bytes] = None
    # pinned host memory (MB) allocated at creation for raster drains: a drain
    # that fits copies straight into it at PCIe speed (0 = staged drains)
    rasterPinnedMB: int = 0
    # split runs: each rank records only its own neurons (rank 0 also the
    # replicated populations); the raster and spike counts sum over ranks
    rasterLocal: bool = False

    def to_c(self) -> L.ssb_engine_opts:
        o = L.ssb_engine_opts()
        lib.ssb_engine_default_opts(C.byref(o))
        o.device = self.device
        if self.window:
            o.window = self.window
        o.block_size = self.blockSize
        o.block_policy = self.blockPolicy
        o.use_graphs = 1 if self.useGraphs else -1
        if self.heavyPreThreshold:
            o.heavy_pre_threshold = self.heavyPreThreshold
        o.raster_capacity = self.rasterCapacity
        o.profile = int(self.profile)
        o.force_step_mode = int(self.forceStepMode)
        o.rank = self.rank
        o.world_size = max(1, self.world)
        o.virtual_world = self.virtualWorld
        o.raster_pinned_mb = max(0, self.rasterPinnedMB)
        o.raster_local = 1 if self.rasterLocal else 0
        if self.shardMinSize:
            o.shard_min_size = self.shardMinSize
        if self.commId is not None:
            if len(self.commId) != 128:
                raise ValueError("commId must be 128 bytes (comm_unique_id())")
            o.has_comm_id = 1
            C.memmove(o.comm_id, bytes(self.commId), 128)
        return o


@dataclass
class PopulationState:
    v: np.ndarray
    u: np.ndarray
    gExc: np.ndarray
    gInh: np.ndarray
    excIn: np.ndarray
    inhIn: np.ndarray
    nanFlag: np.ndarray
    flagged: int


@dataclass
class Raster:
    populations: List[Tuple[str, int]]
    step: np.ndarray    # int64
    population: np.ndarray  # int32
    neuron: np.ndarray  # int32

    def __len__(self) -> int:
        return int(self.step.shape[0])


@dataclass
class RunResult:
    raster: Raster
    avgSpike: Dict[str, float]
    sumNaNs: int
    steps: int
    durationMs: float
    wallTimeMs: float


_FIELDS = {"v": L.FIELD_V, "u": L.FIELD_U, "gExc": L.FIELD_GEXC, "gInh": L.FIELD_GINH,
           "excIn": L.FIELD_EXCIN, "inhIn": L.FIELD_INHIN}
_HH_FIELDS = {"m": L.FIELD_M, "h": L.FIELD_H, "n": L.FIELD_N}  # Traub-Miles (extension)


class Simulation:
    """Simulation (reference engine.hpp:75-99) over the device engine."""

    def __init__(self, spec: NetworkSpec, mode: StorageMode = StorageMode.FromSpec,
                 options: Optional[EngineOptions] = None):
        self.spec = spec
        self.mode = StorageMode(mode)
        self.options = options or EngineOptions()
        self._desc = NetDesc(spec)
        self._opts = self.options.to_c()
        h = C.c_void_p()
        err = _err()
        _raise(lib.ssb_create(self._desc.ptr, int(self.mode), C.byref(self._opts), C.byref(h), err,
                              len(err)), err.value.decode())
        self._h = h
        self._finished = False
        self.result: Optional[RunResult] = None

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and lib is not None:  # lib is None during interpreter shutdown
            lib.ssb_destroy(h)
            self._h = None

    def close(self) -> None:
        self.__del__()

    def _check(self, rc: int) -> None:
        if rc:
            _raise(rc, lib.ssb_last_error(self._h).decode())

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    def step(self, n: int = 1) -> None:
        self._check(lib.ssb_step(self._h, int(n)))

    def steps_total(self) -> int:
        return int(lib.ssb_steps_total(self._h))

    def world(self) -> int:
        """Ranks (or virtual shards) the network is split over (1: whole)."""
        return int(lib.ssb_world(self._h))

    def shard_range(self, pop: Union[int, str]) -> Tuple[int, int, int]:
        """(lo, n_local, n_global): this process's neurons of population pop."""
        pi = pop if isinstance(pop, int) else self.spec.pop_index(pop)
        lo, nl, ng = C.c_int64(), C.c_int64(), C.c_int64()
        self._check(lib.ssb_shard_range(self._h, pi, C.byref(lo), C.byref(nl), C.byref(ng)))
        return lo.value, nl.value, ng.value

    def steps_done(self) -> int:
        return int(lib.ssb_steps_done(self._h))

    def sync(self) -> None:
        self._check(lib.ssb_sync(self._h))

    def pull(self, pop: Union[int, str], fieldname: str) -> np.ndarray:
        pi = pop if isinstance(pop, int) else self.spec.pop_index(pop)
        n = self.spec.populations[pi].size
        if fieldname == "nanFlag":
            out = np.empty(n, np.uint8)
            self._check(lib.ssb_pull_state(self._h, pi, L.FIELD_NANFLAG, out.ctypes.data, n))
            return out
        if fieldname == "flagged":
            out = np.empty(1, np.int64)
            self._check(lib.ssb_pull_state(self._h, pi, L.FIELD_FLAGGED, out.ctypes.data, 1))
            return out
        out = np.empty(n, np.float32)
        fid = _FIELDS.get(fieldname, _HH_FIELDS.get(fieldname))
        if fid is None:
            raise SpecError(f"unknown state field '{fieldname}'")
        self._check(lib.ssb_pull_state(self._h, pi, fid, out.ctypes.data, n))
        return out

    def push(self, pop: Union[int, str], fieldname: str, values) -> None:
        pi = pop if isinstance(pop, int) else self.spec.pop_index(pop)
        n = self.spec.populations[pi].size
        if fieldname == "nanFlag":
            a = np.ascontiguousarray(values, np.uint8)
            fid = L.FIELD_NANFLAG
        elif fieldname == "flagged":
            a = np.ascontiguousarray([values], np.int64).reshape(1)
            fid, n = L.FIELD_FLAGGED, 1
        else:
            a = np.ascontiguousarray(values, np.float32)
            fid = _FIELDS.get(fieldname, _HH_FIELDS.get(fieldname))
            if fid is None:
                raise SpecError(f"unknown state field '{fieldname}'")
        if a.size != n:
            raise SpecError(f"state field '{fieldname}' holds {n} values, {a.size} given")
        self._check(lib.ssb_push_state(self._h, pi, fid, a.ctypes.data, n))

    def population_state(self, name: str) -> PopulationState:
        """Snapshot of the device state (push edits back with push_state)."""
        pi = self.spec.pop_index(name)
        return PopulationState(*(self.pull(pi, f) for f in _FIELDS), self.pull(pi, "nanFlag"),
                               int(self.pull(pi, "flagged")[0]))

    def push_state(self, name: str, st: PopulationState) -> None:
        for f in _FIELDS:
            self.push(name, f, getattr(st, f))
        self.push(name, "nanFlag", st.nanFlag)
        self.push(name, "flagged", st.flagged)

    def group_dense(self, name: str) -> Optional[np.ndarray]:
        gi = self.spec.group_index(name)
        st, npre, npost, nnz = C.c_int32(), C.c_int32(), C.c_int32(), C.c_int64()
        self._check(lib.ssb_group_info(self._h, gi, C.byref(st), C.byref(npre), C.byref(npost),
                                       C.byref(nnz)))
        if st.value != L.STORAGE_DENSE:
            return None
        w = np.empty((npre.value, npost.value), np.float32)
        self._check(lib.ssb_group_dense(self._h, gi, _fptr(w), w.size))
        return w

    def group_weights(self, name: str) -> np.ndarray:
        """A dense group's weights now: a plastic group's learned weights read
        from the device (extension F2), a static group's group_dense()."""
        gi = self.spec.group_index(name)
        st, npre, npost, nnz = C.c_int32(), C.c_int32(), C.c_int32(), C.c_int64()
        self._check(lib.ssb_group_info(self._h, gi, C.byref(st), C.byref(npre), C.byref(npost),
                                       C.byref(nnz)))
        w = np.empty((npre.value, npost.value), np.float32)
        self._check(lib.ssb_group_weights(self._h, gi, _fptr(w), w.size))
        return w

    def group_sparse(self, name: str):
        """(gValues, postInd, rowStart) or None when the group is stored dense."""
        gi = self.spec.group_index(name)
        st, npre, npost, nnz = C.c_int32(), C.c_int32(), C.c_int32(), C.c_int64()
        self._check(lib.ssb_group_info(self._h, gi, C.byref(st), C.byref(npre), C.byref(npost),
                                       C.byref(nnz)))
        if st.value != L.STORAGE_SPARSE:
            return None
        g = np.empty(nnz.value, np.float32)
        ind = np.empty(nnz.value, np.int32)
        rs = np.empty(npre.value + 1, np.int64)
        self._check(lib.ssb_group_sparse(self._h, gi, _fptr(g), _iptr(ind), _lptr(rs)))
        return g, ind, rs

    def finish(self) -> RunResult:
        s = L.ssb_run_summary()
        self._check(lib.ssb_finish(self._h, C.byref(s)))
        npops = len(self.spec.populations)
        rates = np.empty(npops, np.float64)
        self._check(lib.ssb_result_rates(self._h, rates.ctypes.data_as(C.POINTER(C.c_double)),
                                         npops))
        ne = int(lib.ssb_result_n_events(self._h))
        step = np.empty(ne, np.int64)
        pop = np.empty(ne, np.int32)
        neu = np.empty(ne, np.int32)
        self._check(lib.ssb_result_raster(self._h, _lptr(step), _iptr(pop), _iptr(neu), ne))
        r = Raster([(p.name, p.size) for p in self.spec.populations], step, pop, neu)
        self.result = RunResult(r, {p.name: float(rates[i]) for i, p in
                                    enumerate(self.spec.populations)},
                                int(s.sum_nans), int(s.steps), float(s.duration_ms),
                                float(s.wall_time_ms))
        self._finished = True
        return self.result

    def spike_counts(self) -> np.ndarray:
        n = len(self.spec.populations)
        out = np.empty(n, np.int64)
        self._check(lib.ssb_spike_counts(self._h, _lptr(out), n))
        return out

    def window(self) -> int:
        return int(lib.ssb_window(self._h))

    def block_size(self, pop: Union[int, str]) -> int:
        pi = pop if isinstance(pop, int) else self.spec.pop_index(pop)
        return int(lib.ssb_block_size(self._h, pi))

    def grid_size(self, pop: Union[int, str]) -> int:
        """Blocks of the population's update kernel."""
        pi = pop if isinstance(pop, int) else self.spec.pop_index(pop)
        return int(lib.ssb_grid_size(self._h, pi))

    def stream(self) -> int:
        return int(lib.ssb_stream(self._h) or 0)

    def kernel_stats(self) -> List[Tuple[str, int, float]]:
        n = lib.ssb_n_kernel_stats(self._h)
        arr = (L.ssb_kernel_stat * max(1, n))()
        self._check(lib.ssb_kernel_stats(self._h, arr, n))
        return [(arr[i].name.decode(), int(arr[i].launches), float(arr[i].total_ms))
                for i in range(n)]

    def reset_kernel_stats(self) -> None:
        self._check(lib.ssb_kernel_stats_reset(self._h))

    def discard_raster(self) -> None:
        self._check(lib.ssb_raster_discard(self._h))

    def drain_raster(self, wait: bool = True) -> int:
        """Moves every recorded event to host memory.  wait=True returns the
        number of events held on the host once they are there; wait=False starts
        the copy in the background (steps issued next overlap it), returns -1."""
        if not wait:
            self._check(lib.ssb_raster_drain_async(self._h))
            return -1
        n = C.c_int64()
        self._check(lib.ssb_raster_drain(self._h, C.byref(n)))
        return n.value

    def device_bytes(self) -> int:
        return int(lib.ssb_device_bytes(self._h))

    def kernel_launches(self) -> int:
        return int(lib.ssb_kernel_launches(self._h))


def run(spec: NetworkSpec, mode: StorageMode = StorageMode.FromSpec,
        options: Optional[EngineOptions] = None) -> RunResult:
    """run (reference engine.hpp:102)."""
    sim = Simulation(spec, mode, options)
    try:
        return sim.finish()
    finally:
        sim.close()


# ---- free functions ------------------------------------------------------------------


def propagate_dense(weights: np.ndarray, spikes, acc: np.ndarray) -> None:
    """propagate(DenseMatrix) (engine.cpp:53-67), in place on acc, on the GPU."""
    w = np.ascontiguousarray(weights, np.float32)
    if w.ndim != 2:
        raise SpecError("dense weights must be 2-D [nPre, nPost]")
    s = np.ascontiguousarray(spikes, np.int32)
    if acc.dtype != np.float32 or not acc.flags.c_contiguous:
        raise SpecError("acc must be a contiguous float32 array")
    err = _err()
    _raise(lib.ssb_propagate_dense(_fptr(w), w.shape[0], w.shape[1], _iptr(s), s.size, _fptr(acc),
                                   acc.size, err, len(err)), err.value.decode())


def propagate_crs(gValues: np.ndarray, postInd: np.ndarray, rowStart: np.ndarray, nPost: int,
                  spikes, acc: np.ndarray) -> None:
    """propagate(CrsMatrix) (engine.cpp:69-80), in place on acc, on the GPU."""
    g = np.ascontiguousarray(gValues, np.float32)
    ind = np.ascontiguousarray(postInd, np.int32)
    rs = np.ascontiguousarray(rowStart, np.int64)
    s = np.ascontiguousarray(spikes, np.int32)
    if acc.dtype != np.float32 or not acc.flags.c_contiguous:
        raise SpecError("acc must be a contiguous float32 array")
    err = _err()
    _raise(lib.ssb_propagate_crs(_fptr(g), _iptr(ind), _lptr(rs), rs.size - 1, nPost, _iptr(s),
                                 s.size, _fptr(acc), acc.size, err, len(err)), err.value.decode())


def detect_nans(st: PopulationState, model: ModelKind) -> int:
    """detect_nans (engine.cpp:27-51) on a state snapshot, on the GPU; returns newly flagged."""
    n = st.nanFlag.size
    flags = np.ascontiguousarray(st.nanFlag, np.uint8)

    def arr(a):
        if a is None or len(a) == 0:
            return None
        return np.ascontiguousarray(a, np.float32)

    v, u, ge, gi = arr(st.v), arr(st.u), arr(st.gExc), arr(st.gInh)
    fl, nw = C.c_int64(st.flagged), C.c_int64()
    err = _err()
    _raise(lib.ssb_detect_nans(int(model), *(None if x is None else _fptr(x) for x in (v, u, ge, gi)),
                               flags.ctypes.data_as(C.POINTER(C.c_uint8)), n, C.byref(fl),
                               C.byref(nw), err, len(err)), err.value.decode())
    st.nanFlag[:] = flags
    st.flagged = fl.value
    return nw.value


def avg_spike(raster: Raster, population: str, durationMs: float) -> float:
    """avg_spike (engine.cpp:82-99)."""
    if not np.isfinite(durationMs) or not durationMs > 0.0:
        raise SpecError("durationMs must be finite and > 0")
    for i, (name, size) in enumerate(raster.populations):
        if name == population:
            if size < 1:
                raise SpecError(f"population '{population}' has a non-positive size")
            return float(np.count_nonzero(raster.population == i)) / (size * (durationMs / 1000.0))
    raise SpecError(f"raster has no population named '{population}'")


def raster_to_csv(raster: Raster) -> str:
    """raster_to_csv (io.cpp:276-287): 'step,population,neuron' lines."""
    names = [n for n, _ in raster.populations]
    lines = ["step,population,neuron"]
    lines += [f"{s},{names[p]},{n}" for s, p, n in zip(raster.step.tolist(),
                                                        raster.population.tolist(),
                                                        raster.neuron.tolist())]
    return "\n".join(lines) + "\n"


# ---- RNG / connectivity helpers ------------------------------------------------------


def derive_seed(parent: int, label: str) -> int:
    return int(lib.ssb_derive_seed(parent & 0xFFFFFFFFFFFFFFFF, label.encode()))


def stream_u64(globalSeed: int, entitySeed: int, label: str, n: int) -> np.ndarray:
    out = np.empty(n, np.uint64)
    _raise(lib.ssb_stream_u64(globalSeed & 0xFFFFFFFFFFFFFFFF, entitySeed & 0xFFFFFFFFFFFFFFFF,
                              label.encode(), n, out.ctypes.data_as(C.POINTER(C.c_uint64))),
           "stream failed")
    return out


def gen_fixed_outdegree(nPre: int, nPost: int, k: int, dist: WeightDist, sign: int,
                        seed: int) -> np.ndarray:
    out = np.empty((max(nPre, 0), max(nPost, 0)), np.float32)
    err = _err()
    _raise(lib.ssb_gen_fixed_outdegree(nPre, nPost, k, L.WEIGHT_UNIFORM if dist.kind == "uniform"
                                       else L.WEIGHT_CONSTANT, dist.lo, dist.hi, dist.value, sign,
                                       seed & 0xFFFFFFFFFFFFFFFF, _fptr(out), err, len(err)),
           err.value.decode())
    return out


def build_group(spec: NetworkSpec, group: Union[int, str],
                mode: StorageMode = StorageMode.FromSpec):
    """Connectivity of one group as Simulation's constructor builds it (host setup).

    Returns ("dense", W[nPre, nPost]) or ("sparse", (gValues, postInd, rowStart)).
    """
    gi = group if isinstance(group, int) else spec.group_index(group)
    desc = NetDesc(spec)
    st, npre, npost, nnz = C.c_int32(), C.c_int32(), C.c_int32(), C.c_int64()
    err = _err()
    _raise(lib.ssb_build_group(desc.ptr, int(mode), gi, C.byref(st), C.byref(npre),
                               C.byref(npost), C.byref(nnz), None, None, None, 0, err, len(err)),
           err.value.decode())
    vals = np.empty(nnz.value, np.float32)
    if st.value == L.STORAGE_DENSE:
        _raise(lib.ssb_build_group(desc.ptr, int(mode), gi, C.byref(st), C.byref(npre),
                                   C.byref(npost), C.byref(nnz), _fptr(vals), None, None,
                                   vals.size, err, len(err)), err.value.decode())
        return "dense", vals.reshape(npre.value, npost.value)
    ind = np.empty(nnz.value, np.int32)
    rs = np.empty(npre.value + 1, np.int64)
    _raise(lib.ssb_build_group(desc.ptr, int(mode), gi, C.byref(st), C.byref(npre),
                               C.byref(npost), C.byref(nnz), _fptr(vals), _iptr(ind), _lptr(rs),
                               vals.size, err, len(err)), err.value.decode())
    return "sparse", (vals, ind, rs)


# ---- calibration sweep (reference calibration.hpp:12-42) -------------------------------


@dataclass
class SweepRow:
    nConn: int = 0
    gScale: float = 0.0
    avgSpike: float = 0.0
    sumNaNs: int = 0
    failed: bool = False
    error: str = ""


@dataclass
class SweepRequest:
    nConnValues: Sequence[int] = ()
    gScaleValues: Sequence[float] = ()
    targetPopulation: str = ""
    parallelism: int = 1
    storage: "StorageMode" = None
    onCell: Optional[object] = None  # called (row, done, total) after each cell, in order
    engine: Optional["EngineOptions"] = None  # B200 extension


def sweep(builder, req: SweepRequest) -> List[SweepRow]:
    """sweep (reference calibration.cpp:16-86): every (nConn, gScale) grid cell
    (duplicates collapsed, ascending) built by builder(nConn, gScale) and run to
    its end on the GPU, req.parallelism cells at a time.  A cell whose build or
    run fails is recorded (failed, avgSpike NaN, sumNaNs -1), not raised."""
    if builder is None:
        raise SpecError("sweep needs a network builder")
    if not req.nConnValues:
        raise SpecError("sweep needs at least one nConn value")
    if not req.gScaleValues:
        raise SpecError("sweep needs at least one gScale value")
    if not req.targetPopulation:
        raise SpecError("sweep needs a target population name")
    if any(not np.isfinite(g) for g in req.gScaleValues):
        raise SpecError("sweep gScale values must be finite")
    rows, descs, which = [], [], []
    for n in sorted(set(int(x) for x in req.nConnValues)):
        for g in sorted(set(float(x) for x in req.gScaleValues)):
            row = SweepRow(n, g)
            try:
                descs.append(NetDesc(builder(n, g)))
                which.append(len(rows))
            except Exception as exc:  # noqa: BLE001 -- recorded like the reference
                row.failed, row.error, row.avgSpike, row.sumNaNs = True, str(exc), float("nan"), -1
            rows.append(row)
    if descs:
        k = len(descs)
        arr = (C.POINTER(L.ssb_net_desc) * k)(*[C.pointer(d.desc) for d in descs])
        avg = np.empty(k, np.float64)
        nans = np.empty(k, np.int64)
        failed = np.empty(k, np.int32)
        stride = 512
        errs = C.create_string_buffer(k * stride)
        opts = (req.engine or EngineOptions()).to_c()
        mode = int(req.storage if req.storage is not None else StorageMode.FromSpec)
        err = _err()
        _raise(lib.ssb_sweep(arr, k, mode, req.targetPopulation.encode(), max(1, req.parallelism),
                             C.byref(opts), avg.ctypes.data_as(C.POINTER(C.c_double)),
                             _lptr(nans), _iptr(failed), errs, stride, err, len(err)),
               err.value.decode())
        for j, i in enumerate(which):
            r = rows[i]
            r.avgSpike, r.sumNaNs, r.failed = float(avg[j]), int(nans[j]), bool(failed[j])
            if r.failed:
                r.error = errs.raw[j * stride:(j + 1) * stride].split(b"\0", 1)[0].decode()
    if req.onCell:
        for d, r in enumerate(rows, 1):
            req.onCell(r, d, len(rows))
    return rows


def shard_plan(spec: NetworkSpec, world: int, minSize: int = 0) -> Dict[str, Optional[List[int]]]:
    """Neuron ranges of a world of `world` ranks per population (None: whole,
    replicated on every rank), as the engine splits it (host, no GPU)."""
    desc = NetDesc(spec)
    npop = len(spec.populations)
    b = np.empty(npop * (world + 1), np.int64)
    err = _err()
    _raise(lib.ssb_shard_plan(desc.ptr, world, minSize, _lptr(b), err, len(err)),
           err.value.decode())
    b = b.reshape(npop, world + 1)
    return {p.name: (None if b[i, 0] < 0 else [int(x) for x in b[i]])
            for i, p in enumerate(spec.populations)}


def shard_group(spec: NetworkSpec, group: Union[int, str], world: int, rank: int,
                mode: StorageMode = StorageMode.FromSpec, minSize: int = 0):
    """Group connectivity as rank `rank` of `world` holds it (column slice of a
    split post population); same return shape as build_group."""
    gi = group if isinstance(group, int) else spec.group_index(group)
    desc = NetDesc(spec)
    st, npre, npost, nnz = C.c_int32(), C.c_int32(), C.c_int32(), C.c_int64()
    err = _err()
    args = (desc.ptr, int(mode), gi, world, rank, minSize, C.byref(st), C.byref(npre),
            C.byref(npost), C.byref(nnz))
    _raise(lib.ssb_shard_group(*args, None, None, None, 0, err, len(err)), err.value.decode())
    vals = np.empty(nnz.value, np.float32)
    if st.value == L.STORAGE_DENSE:
        _raise(lib.ssb_shard_group(*args, _fptr(vals), None, None, vals.size, err, len(err)),
               err.value.decode())
        return "dense", vals.reshape(npre.value, npost.value)
    ind = np.empty(nnz.value, np.int32)
    rs = np.empty(npre.value + 1, np.int64)
    _raise(lib.ssb_shard_group(*args, _fptr(vals), _iptr(ind), _lptr(rs), vals.size, err,
                               len(err)), err.value.decode())
    return "sparse", (vals, ind, rs)


def comm_selftest(device: int = 0) -> None:
    """Runs the split engine's NCCL calls on a one-rank communicator (raises on failure)."""
    err = _err()
    _raise(lib.ssb_comm_selftest(device, err, len(err)), err.value.decode())


def comm_unique_id() -> bytes:
    """NCCL unique id for EngineOptions.commId (rank 0 creates, the caller
    broadcasts it, e.g. with torch.distributed.broadcast_object_list)."""
    out = (C.c_uint8 * 128)()
    err = _err()
    _raise(lib.ssb_comm_unique_id(out, err, len(err)), err.value.decode())
    return bytes(out)


def mem_sparse_elements(nnz: int, nPost: int) -> int:
    return int(lib.ssb_mem_sparse_elements(nnz, nPost))


def mem_dense_elements(nPre: int, nPost: int) -> int:
    return int(lib.ssb_mem_dense_elements(nPre, nPost))


# ---- occupancy model (occupancy.hpp) ---------------------------------------------------


@dataclass
class DeviceSpec:
    name: str
    warpSize: int = 32
    maxWarpsPerSM: int = 64
    maxBlocksPerSM: int = 16
    maxThreadsPerBlock: int = 1024
    sharedMemPerSM: int = 49152
    regsPerSM: int = 65536
    regAllocUnit: int = 256
    sharedAllocUnit: int = 256

    def to_c(self) -> L.ssb_device_spec:
        return L.ssb_device_spec(self.name.encode()[:31], self.warpSize, self.maxWarpsPerSM,
                                 self.maxBlocksPerSM, self.maxThreadsPerBlock, self.sharedMemPerSM,
                                 self.regsPerSM, self.regAllocUnit, self.sharedAllocUnit)

    @staticmethod
    def from_c(d: L.ssb_device_spec) -> "DeviceSpec":
        return DeviceSpec(d.name.decode(), d.warp_size, d.max_warps_per_sm, d.max_blocks_per_sm,
                          d.max_threads_per_block, d.shared_mem_per_sm, d.regs_per_sm,
                          d.reg_alloc_unit, d.shared_alloc_unit)


LIMITERS = ("warps", "blocks", "shared", "registers")


@dataclass
class OccupancyResult:
    warpsPerBlock: int
    limitWarps: int
    limitBlocks: int
    limitShared: int
    limitRegs: int
    activeBlocks: int
    activeWarps: int
    occupancy: float
    limiters: List[str]


def _occ(r: L.ssb_occupancy_result) -> OccupancyResult:
    return OccupancyResult(r.warps_per_block, r.limit_warps, r.limit_blocks, r.limit_shared,
                           r.limit_regs, r.active_blocks, r.active_warps, r.occupancy,
                           [LIMITERS[i] for i in range(4) if r.limiter_mask >> i & 1])


def device_preset(name: str) -> DeviceSpec:
    d = L.ssb_device_spec()
    err = _err()
    _raise(lib.ssb_device_preset(name.encode(), C.byref(d), err, len(err)), err.value.decode())
    return DeviceSpec.from_c(d)


def auto_dense_threshold() -> float:
    """StorageMode.Auto's density threshold (extension; env SSB_AUTO_DENSITY)."""
    return float(lib.ssb_auto_dense_threshold())


def device_preset_names() -> List[str]:
    return lib.ssb_device_preset_names().decode().split(",")


def device_query(device: int = 0) -> DeviceSpec:
    d = L.ssb_device_spec()
    err = _err()
    _raise(lib.ssb_device_query(device, C.byref(d), err, len(err)), err.value.decode())
    return DeviceSpec.from_c(d)


def occupancy(dev: DeviceSpec, threadsPerBlock: int, regsPerThread: int = 0,
              sharedMemPerBlock: int = 0) -> OccupancyResult:
    r = L.ssb_occupancy_result()
    err = _err()
    _raise(lib.ssb_occupancy(C.byref(dev.to_c()), threadsPerBlock, regsPerThread,
                             sharedMemPerBlock, C.byref(r), err, len(err)), err.value.decode())
    return _occ(r)


def recommend_block_size(dev: DeviceSpec, regsPerThread: int,
                         sharedMemPerBlock: int) -> Tuple[int, OccupancyResult]:
    r = L.ssb_occupancy_result()
    bs = C.c_int64()
    err = _err()
    _raise(lib.ssb_recommend_block_size(C.byref(dev.to_c()), regsPerThread, sharedMemPerBlock,
                                        C.byref(bs), C.byref(r), err, len(err)), err.value.decode())
    return bs.value, _occ(r)


def kernel_attributes(name: str) -> Tuple[int, int, int]:
    r, s, m = C.c_int32(), C.c_int32(), C.c_int32()
    _raise(lib.ssb_kernel_attributes(name.encode(), C.byref(r), C.byref(s), C.byref(m)),
           f"no attributes for kernel '{name}' (unknown, or no GPU)")
    return r.value, s.value, m.value


def device_count() -> int:
    return int(lib.ssb_device_count())
