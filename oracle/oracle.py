"""TEST INFRASTRUCTURE ONLY — ctypes bindings of the parity checkers.

* ``liboracle.so``: the C restatement of the reference step path (oracle.c).
* ``_ref/libsynscale_ref.so``: the unmodified reference library compiled from
  /root/reference/proj by oracle/Makefile, driven through ref_shim.cpp.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg may
import this module.  Both libraries take the product's flat ``ssb_net_desc``
(include/synscale_b200.h) as a plain data format.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_LIB = os.path.join(HERE, "liboracle.so")
REF_LIB = os.path.join(HERE, "_ref", "libsynscale_ref.so")
REF_SRC = "/root/reference/proj"

FIELD_IDS = {"v": 0, "u": 1, "gExc": 2, "gInh": 3, "excIn": 4, "inhIn": 5, "nanFlag": 6,
             "m": 8, "h": 9, "n": 10,
             "flagged": 7}


def build(quiet: bool = True) -> None:
    """Builds liboracle.so, and _ref/ when the reference sources are present."""
    out = subprocess.run(["make", "-C", HERE], capture_output=True, text=True)
    if out.returncode:
        raise RuntimeError("oracle build failed:\n" + out.stdout + out.stderr)
    if not quiet:
        print(out.stdout)


def have_ref() -> bool:
    return os.path.exists(REF_LIB)


_P = C.POINTER
_vp, _i32, _i64, _u64, _dbl = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64, C.c_double


def _bind(path: str, prefix: str) -> C.CDLL:
    lib = C.CDLL(path)
    sig = {
        "create": (_vp, [_vp, C.c_int, C.c_char_p, C.c_size_t]),
        "destroy": (None, [_vp]),
        "step": (C.c_int, [_vp, C.c_longlong]),
        "steps_total": (C.c_longlong, [_vp]),
        "steps_done": (C.c_longlong, [_vp]),
        "n_events": (C.c_longlong, [_vp]),
        "raster": (C.c_int, [_vp, _vp, _vp, _vp, C.c_longlong]),
        "get_state": (C.c_int, [_vp, C.c_int, C.c_int, _vp, C.c_longlong]),
        "set_state": (C.c_int, [_vp, C.c_int, C.c_int, _vp, C.c_longlong]),
        "group_info": (C.c_int, [_vp, C.c_int, _vp, _vp, _vp, _vp]),
        "group_dense": (C.c_int, [_vp, C.c_int, _vp]),
        "group_sparse": (C.c_int, [_vp, C.c_int, _vp, _vp, _vp]),
        "gen_fixed_outdegree": (C.c_int, [_i32, _i32, _i32, C.c_int, _dbl, _dbl, _dbl, C.c_int,
                                          _u64, _vp] + ([C.c_char_p, C.c_size_t]
                                                        if prefix == "ref_" else [])),
        "stream_u64": (None, [_u64, _u64, C.c_char_p, C.c_longlong, _vp]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, prefix + name)
        fn.restype, fn.argtypes = res, args
    if prefix == "or_":
        lib.or_flagged.restype, lib.or_flagged.argtypes = C.c_longlong, [_vp, C.c_int]
        lib.or_spike_count.restype, lib.or_spike_count.argtypes = C.c_longlong, [_vp, C.c_int]
        lib.or_derive_seed_c.restype, lib.or_derive_seed_c.argtypes = _u64, [_u64, C.c_char_p]
        lib.or_propagate_dense.argtypes = [_vp, _i32, _vp, _i64, _vp]
        lib.or_propagate_crs.argtypes = [_vp, _vp, _vp, _vp, _i64, _vp]
        lib.or_detect_nans.restype = _i64
        lib.or_detect_nans.argtypes = [C.c_int, _vp, _vp, _vp, _vp, _vp, _i64]
    else:
        lib.ref_finish.restype, lib.ref_finish.argtypes = C.c_int, [_vp]
        lib.ref_rates.restype, lib.ref_rates.argtypes = C.c_int, [_vp, _vp, C.c_int]
        lib.ref_sum_nans.restype, lib.ref_sum_nans.argtypes = C.c_longlong, [_vp]
        lib.ref_derive_seed.restype, lib.ref_derive_seed.argtypes = _u64, [_u64, C.c_char_p]
        lib.ref_propagate_dense.restype = C.c_int
        lib.ref_propagate_dense.argtypes = [_vp, _i32, _i32, _vp, C.c_longlong, _vp, C.c_longlong]
        lib.ref_propagate_crs.restype = C.c_int
        lib.ref_propagate_crs.argtypes = [_vp, _vp, _vp, _i32, _i32, _vp, C.c_longlong, _vp,
                                          C.c_longlong]
        lib.ref_time_steps.restype = _dbl
        lib.ref_time_steps.argtypes = [_vp, C.c_int, C.c_longlong, C.c_int, _P(_dbl), _P(C.c_longlong)]
    return lib


_libs = {}


def oracle_lib() -> C.CDLL:
    if "or_" not in _libs:
        if not os.path.exists(ORACLE_LIB):
            build()
        _libs["or_"] = _bind(ORACLE_LIB, "or_")
    return _libs["or_"]


def ref_lib() -> C.CDLL:
    if "ref_" not in _libs:
        if not os.path.exists(REF_LIB):
            raise RuntimeError("reference build missing: oracle/_ref/libsynscale_ref.so")
        _libs["ref_"] = _bind(REF_LIB, "ref_")
    return _libs["ref_"]


class CpuSim:
    """One CPU simulation (oracle restatement, or the reference itself with ref=True)."""

    def __init__(self, desc_ptr, spec, mode: int = 0, ref: bool = False):
        self.ref = ref
        self.lib = ref_lib() if ref else oracle_lib()
        self.p = "ref_" if ref else "or_"
        self.spec = spec
        err = C.create_string_buffer(1024)
        self.h = getattr(self.lib, self.p + "create")(C.cast(desc_ptr, C.c_void_p), mode, err,
                                                      len(err))
        if not self.h:
            raise ValueError(err.value.decode())
        self._finished = False

    def _f(self, name):
        return getattr(self.lib, self.p + name)

    def __del__(self):
        if getattr(self, "h", None):
            self._f("destroy")(self.h)
            self.h = None

    def step(self, n: int = 1) -> None:
        rc = self._f("step")(self.h, n)
        if rc:
            raise ValueError(f"step failed ({rc})")

    def steps_total(self) -> int:
        return int(self._f("steps_total")(self.h))

    def steps_done(self) -> int:
        return int(self._f("steps_done")(self.h))

    def state(self, pop: int, field: str) -> np.ndarray:
        n = self.spec.populations[pop].size
        if field == "flagged":
            out = np.zeros(1, np.int64)
            n = 1
        else:
            out = np.zeros(n, np.uint8 if field == "nanFlag" else np.float32)
        rc = self._f("get_state")(self.h, pop, FIELD_IDS[field], out.ctypes.data, n)
        if rc:
            raise ValueError(f"get_state failed ({rc})")
        return out

    def set_state(self, pop: int, field: str, values) -> None:
        a = np.ascontiguousarray(values, np.int64 if field == "flagged" else np.float32)
        rc = self._f("set_state")(self.h, pop, FIELD_IDS[field], a.ctypes.data, a.size)
        if rc:
            raise ValueError(f"set_state failed ({rc})")

    def finish(self):
        """Runs the remaining steps; returns (step, pop, neuron) arrays."""
        if self.ref:
            if self._f("finish")(self.h):
                raise ValueError("finish failed")
        else:
            self.step(self.steps_total() - self.steps_done())
        self._finished = True
        return self.raster()

    def raster(self):
        n = int(self._f("n_events")(self.h))
        s = np.empty(n, np.int64)
        p = np.empty(n, np.int32)
        q = np.empty(n, np.int32)
        if self._f("raster")(self.h, s.ctypes.data, p.ctypes.data, q.ctypes.data, n):
            raise ValueError("raster failed")
        return s, p, q

    def rates(self):
        """avgSpike per population (reference: from RunResult; oracle: from counts)."""
        npops = len(self.spec.populations)
        if self.ref:
            out = np.empty(npops, np.float64)
            self.lib.ref_rates(self.h, out.ctypes.data, npops)
            return out
        dur = self.spec.durationMs
        return np.array([self.lib.or_spike_count(self.h, i) /
                         (self.spec.populations[i].size * (dur / 1000.0)) for i in range(npops)])

    def sum_nans(self) -> int:
        if self.ref:
            return int(self.lib.ref_sum_nans(self.h))
        return int(sum(self.lib.or_flagged(self.h, i) for i in range(len(self.spec.populations))))

    def group(self, gi: int):
        dense, npre, npost, nnz = C.c_int32(), C.c_int32(), C.c_int32(), C.c_int64()
        self._f("group_info")(self.h, gi, C.byref(dense), C.byref(npre), C.byref(npost),
                              C.byref(nnz))
        if dense.value:
            w = np.empty((npre.value, npost.value), np.float32)
            self._f("group_dense")(self.h, gi, w.ctypes.data)
            return ("dense", w)
        g = np.empty(nnz.value, np.float32)
        ind = np.empty(nnz.value, np.int32)
        rs = np.empty(npre.value + 1, np.int64)
        self._f("group_sparse")(self.h, gi, g.ctypes.data, ind.ctypes.data, rs.ctypes.data)
        return ("sparse", (g, ind, rs))


def stream_u64(g: int, e: int, label: str, n: int, ref: bool = False) -> np.ndarray:
    lib = ref_lib() if ref else oracle_lib()
    out = np.empty(n, np.uint64)
    getattr(lib, ("ref_" if ref else "or_") + "stream_u64")(g, e, label.encode(), n,
                                                           out.ctypes.data)
    return out


def gen_fixed_outdegree(nPre, nPost, k, kind, lo, hi, value, sign, seed, ref=False):
    lib = ref_lib() if ref else oracle_lib()
    out = np.empty((nPre, nPost), np.float32)
    if ref:
        err = C.create_string_buffer(512)
        rc = lib.ref_gen_fixed_outdegree(nPre, nPost, k, kind, lo, hi, value, sign, seed,
                                         out.ctypes.data, err, len(err))
    else:
        rc = lib.or_gen_fixed_outdegree(nPre, nPost, k, kind, lo, hi, value, sign, seed,
                                        out.ctypes.data)
    if rc:
        raise ValueError(f"gen_fixed_outdegree rejected its arguments ({rc})")
    return out


def ref_time_steps(desc_ptr, mode: int, steps: int, replicas: int):
    """Wall seconds for `replicas` concurrent reference Simulations x `steps` steps."""
    build_s = C.c_double()
    ev = C.c_longlong()
    t = ref_lib().ref_time_steps(C.cast(desc_ptr, C.c_void_p), mode, steps, replicas,
                                 C.byref(build_s), C.byref(ev))
    return t, build_s.value


# ---- the reference's own builders and replica pools (ref_shim.cpp) ------------------

def mbody_gscales(n_kc: int, frac: float):
    """SURVEY.md §8(d) gScales: pn_kc, pn_lhi, lhi_kc, kc_dn."""
    return (0.5 / frac, 1.0, 0.1, 30.0 / n_kc)


def _bind_builders(lib: C.CDLL) -> None:
    if getattr(lib, "_builders_bound", False):
        return
    d4 = _P(_dbl)
    lib.ref_build_mbody.restype = _vp
    lib.ref_build_mbody.argtypes = [_i32, _i32, _i32, _i32, d4, _u64, _dbl, _dbl, _dbl, _dbl,
                                    C.c_char_p, C.c_size_t]
    lib.ref_build_izhikevich.restype = _vp
    lib.ref_build_izhikevich.argtypes = [_i32, _i32, _dbl, _dbl, _u64, _dbl, _dbl, _dbl, _dbl,
                                         _dbl, _dbl, _dbl, C.c_int, C.c_char_p, C.c_size_t]
    lib.ref_desc_free.restype, lib.ref_desc_free.argtypes = None, [_vp]
    lib.ref_pool_mbody.restype = _vp
    lib.ref_pool_mbody.argtypes = [_i32, _i32, _i32, _i32, d4, _u64, _dbl, _dbl, _dbl, _dbl,
                                   C.c_int, C.c_int, _P(_dbl), C.c_char_p, C.c_size_t]
    lib.ref_pool_step.restype, lib.ref_pool_step.argtypes = _dbl, [_vp, C.c_longlong]
    lib.ref_pool_counts.restype = C.c_int
    lib.ref_pool_counts.argtypes = [_vp, C.c_longlong, C.c_longlong, _vp, C.c_int]
    lib.ref_pool_groups.restype = C.c_int
    lib.ref_pool_groups.argtypes = [_vp, _vp, _vp, C.c_int]
    lib.ref_pool_steps_total.restype, lib.ref_pool_steps_total.argtypes = C.c_longlong, [_vp]
    lib.ref_pool_destroy.restype, lib.ref_pool_destroy.argtypes = None, [_vp]
    lib.ref_pool_raster_checksum.restype = _u64
    lib.ref_pool_raster_checksum.argtypes = [_vp, C.c_int, C.c_longlong]
    lib._builders_bound = True


class RefDesc:
    """A flat ssb_net_desc built by the REFERENCE's own builder (build_mbody_net /
    build_izhikevich_net, network.cpp:198-362), owned by the shim."""

    def __init__(self, ptr):
        self.ptr = ptr
        self._lib = ref_lib()

    def __del__(self):
        if getattr(self, "ptr", None):
            self._lib.ref_desc_free(self.ptr)
            self.ptr = None


def ref_mbody_desc(n_kc: int, frac: float, duration_ms: float, seed: int = 7,
                   dt_ms: float = 0.1, n_pn: int = 100, n_lhi: int = 20, n_dn: int = 100,
                   rate_hz: float = 50.0, gscales=None) -> RefDesc:
    lib = ref_lib()
    _bind_builders(lib)
    g = (_dbl * 4)(*(gscales or mbody_gscales(n_kc, frac)))
    err = C.create_string_buffer(1024)
    p = lib.ref_build_mbody(n_pn, n_lhi, n_kc, n_dn, g, seed, dt_ms, duration_ms, rate_hz, frac,
                            err, len(err))
    if not p:
        raise ValueError(err.value.decode())
    return RefDesc(p)


def ref_izh_desc(n: int, n_conn: int, exc_fraction: float, g_scale: float, seed: int,
                 dt_ms: float = 1.0, duration_ms: float = 1000.0, noise_exc: float = 5.0,
                 noise_inh: float = 2.0, exc_hi: float = 0.5, inh_hi: float = 1.0,
                 bias: float = 0.0, dense: bool = False) -> RefDesc:
    lib = ref_lib()
    _bind_builders(lib)
    err = C.create_string_buffer(1024)
    p = lib.ref_build_izhikevich(n, n_conn, exc_fraction, g_scale, seed, dt_ms, duration_ms,
                                 noise_exc, noise_inh, exc_hi, inh_hi, bias, int(dense), err,
                                 len(err))
    if not p:
        raise ValueError(err.value.decode())
    return RefDesc(p)


class RefPool:
    """`replicas` reference Simulations of the reference-built mushroom body,
    stepped concurrently on host threads (calibration.cpp:76-84's model)."""

    def __init__(self, n_kc: int, frac: float, duration_ms: float, replicas: int, seed: int = 7,
                 mode: int = 0, dt_ms: float = 0.1):
        self.lib = ref_lib()
        _bind_builders(self.lib)
        g = (_dbl * 4)(*mbody_gscales(n_kc, frac))
        err = C.create_string_buffer(1024)
        b = C.c_double()
        self.h = self.lib.ref_pool_mbody(100, 20, n_kc, 100, g, seed, dt_ms, duration_ms, 50.0,
                                         frac, mode, replicas, C.byref(b), err, len(err))
        if not self.h:
            raise ValueError(err.value.decode())
        self.build_s = b.value
        self.replicas = replicas
        pre = np.zeros(16, np.int32)
        deg = np.zeros(16, np.int32)
        n = self.lib.ref_pool_groups(self.h, pre.ctypes.data, deg.ctypes.data, 16)
        self.group_pre, self.group_out = pre[:n], deg[:n]

    def step(self, steps: int) -> float:
        t = self.lib.ref_pool_step(self.h, steps)
        if t < 0:
            raise RuntimeError("reference step failed")
        return t

    def counts(self, lo: int, hi: int) -> np.ndarray:
        """Spikes per population with step in [lo, hi), summed over replicas
        (finishes the replicas on first use)."""
        out = np.zeros(16, np.int64)
        n = self.lib.ref_pool_counts(self.h, lo, hi, out.ctypes.data, 16)
        if n < 0:
            raise RuntimeError("reference finish failed")
        return out[:n]

    def synaptic_events(self, lo: int, hi: int) -> int:
        c = self.counts(lo, hi)
        return int(sum(int(c[p]) * int(d) for p, d in zip(self.group_pre, self.group_out)))

    def raster_checksum(self, replica: int = 0, up_to: int = 1 << 62) -> int:
        self.counts(0, 0)
        return int(self.lib.ref_pool_raster_checksum(self.h, replica, up_to))

    def steps_total(self) -> int:
        return int(self.lib.ref_pool_steps_total(self.h))

    def close(self):
        if getattr(self, "h", None):
            self.lib.ref_pool_destroy(self.h)
            self.h = None

    __del__ = close
