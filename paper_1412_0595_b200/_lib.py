"""ctypes binding of libsynscale_b200.so (the C ABI in include/synscale_b200.h).

The shared library is built in-tree by ``__graft_entry__.build()``
(``make -C paper_1412_0595_b200/csrc``).  There is no Python or CPU fallback:
importing this module fails loudly when the library is missing, and every
simulation call fails with a CUDA error when no GPU is visible.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libsynscale_b200.so")

SSB_OK, SSB_ERR_INTERNAL, SSB_ERR_SPEC = 0, 1, 2
MODEL_IZHIKEVICH, MODEL_POISSON, MODEL_CONDLIF, MODEL_TRAUBMILES = 0, 1, 2, 3
SIGN_EXC, SIGN_INH = 0, 1
STORAGE_DENSE, STORAGE_SPARSE = 0, 1
MODE_FROM_SPEC, MODE_FORCE_DENSE, MODE_FORCE_SPARSE, MODE_AUTO = 0, 1, 2, 3
WEIGHT_CONSTANT, WEIGHT_UNIFORM = 0, 1
(FIELD_V, FIELD_U, FIELD_GEXC, FIELD_GINH, FIELD_EXCIN, FIELD_INHIN, FIELD_NANFLAG,
 FIELD_FLAGGED, FIELD_M, FIELD_H, FIELD_N) = range(11)


class ssb_pop_desc(C.Structure):
    _fields_ = [
        ("name", C.c_char_p), ("size", C.c_int32), ("model", C.c_int32), ("seed", C.c_uint64),
        ("rate_hz", C.c_double),
        ("tau_m_ms", C.c_double), ("e_leak_mv", C.c_double), ("v_thresh_mv", C.c_double),
        ("v_reset_mv", C.c_double), ("e_exc_mv", C.c_double), ("e_inh_mv", C.c_double),
        ("tau_syn_ms", C.c_double),
        ("izh_a", C.POINTER(C.c_double)), ("izh_b", C.POINTER(C.c_double)),
        ("izh_c", C.POINTER(C.c_double)), ("izh_d", C.POINTER(C.c_double)),
        ("izh_noise", C.POINTER(C.c_double)), ("izh_bias", C.POINTER(C.c_double)),
        ("hh_gna", C.c_double), ("hh_ena", C.c_double), ("hh_gk", C.c_double),
        ("hh_ek", C.c_double), ("hh_gl", C.c_double), ("hh_el", C.c_double),
        ("hh_c", C.c_double), ("hh_substeps", C.c_int32),
    ]


PLASTICITY_NONE, PLASTICITY_STDP = 0, 1


class ssb_group_desc(C.Structure):
    _fields_ = [
        ("name", C.c_char_p), ("pre", C.c_char_p), ("post", C.c_char_p),
        ("sign", C.c_int32), ("out_degree", C.c_int32), ("weight_kind", C.c_int32),
        ("weight_lo", C.c_double), ("weight_hi", C.c_double), ("weight_value", C.c_double),
        ("g_scale", C.c_double), ("storage", C.c_int32), ("pre_offset", C.c_int32),
        ("pre_count", C.c_int32),
        # extension F2 (STDP); zero = static, as in the reference
        ("plasticity", C.c_int32), ("stdp_a_plus", C.c_double), ("stdp_a_minus", C.c_double),
        ("stdp_tau_plus_ms", C.c_double), ("stdp_tau_minus_ms", C.c_double),
        ("stdp_w_max", C.c_double),
    ]


class ssb_net_desc(C.Structure):
    _fields_ = [
        ("n_pops", C.c_int32), ("pops", C.POINTER(ssb_pop_desc)),
        ("n_groups", C.c_int32), ("groups", C.POINTER(ssb_group_desc)),
        ("dt_ms", C.c_double), ("duration_ms", C.c_double), ("global_seed", C.c_uint64),
    ]


class ssb_mbody_opts(C.Structure):
    _fields_ = [(n, C.c_double) for n in (
        "dt_ms", "duration_ms", "pn_rate_hz", "pn_kc_out_fraction", "tau_m_ms", "e_leak_mv",
        "v_thresh_mv", "v_reset_mv", "e_exc_mv", "e_inh_mv", "tau_syn_ms", "pn_kc_weight_hi",
        "pn_lhi_weight", "lhi_kc_weight", "kc_dn_weight")] + [("kc_model", C.c_int32)] + [
        (n, C.c_double) for n in ("hh_gna", "hh_ena", "hh_gk", "hh_ek", "hh_gl", "hh_el", "hh_c",
                                  "hh_e_inh_mv", "kc_tau_syn_ms")] + [("hh_substeps", C.c_int32)]


class ssb_izh_opts(C.Structure):
    _fields_ = [(n, C.c_double) for n in (
        "dt_ms", "duration_ms", "noise_exc", "noise_inh", "exc_weight_hi", "inh_weight_hi",
        "bias_current")] + [("storage", C.c_int32)]


class ssb_engine_opts(C.Structure):
    _fields_ = [
        ("device", C.c_int32), ("window", C.c_int32), ("block_size", C.c_int32),
        ("block_policy", C.c_int32), ("use_graphs", C.c_int32),
        ("heavy_pre_threshold", C.c_int32), ("raster_capacity", C.c_int64),
        ("profile", C.c_int32), ("force_step_mode", C.c_int32),
        ("rank", C.c_int32), ("world_size", C.c_int32), ("virtual_world", C.c_int32),
        ("shard_min_size", C.c_int32), ("has_comm_id", C.c_int32),
        ("comm_id", C.c_uint8 * 128), ("raster_pinned_mb", C.c_int32),
        ("raster_local", C.c_int32),
    ]


class ssb_run_summary(C.Structure):
    _fields_ = [("steps", C.c_int64), ("steps_done", C.c_int64), ("duration_ms", C.c_double),
                ("sum_nans", C.c_int64), ("n_events", C.c_int64), ("wall_time_ms", C.c_double)]


class ssb_device_spec(C.Structure):
    _fields_ = [("name", C.c_char * 32)] + [(n, C.c_int64) for n in (
        "warp_size", "max_warps_per_sm", "max_blocks_per_sm", "max_threads_per_block",
        "shared_mem_per_sm", "regs_per_sm", "reg_alloc_unit", "shared_alloc_unit")]


class ssb_occupancy_result(C.Structure):
    _fields_ = [(n, C.c_int64) for n in (
        "warps_per_block", "limit_warps", "limit_blocks", "limit_shared", "limit_regs",
        "active_blocks", "active_warps")] + [("occupancy", C.c_double),
                                              ("limiter_mask", C.c_int32)]


class ssb_kernel_stat(C.Structure):
    _fields_ = [("name", C.c_char * 48), ("launches", C.c_int64), ("total_ms", C.c_double),
                ("bytes", C.c_double)]


P = C.POINTER
_i32, _i64, _u64, _dbl, _f32, _u8 = C.c_int32, C.c_int64, C.c_uint64, C.c_double, C.c_float, C.c_uint8
_vp, _cp, _sz = C.c_void_p, C.c_char_p, C.c_size_t

# name: (restype, argtypes)
_SIGNATURES = {
    "ssb_version": (_cp, []),
    "ssb_auto_dense_threshold": (C.c_double, []),
    "ssb_device_count": (C.c_int, []),
    "ssb_validate": (C.c_int, [P(ssb_net_desc), _cp, _sz]),
    "ssb_build_mbody": (C.c_int, [_i32, _i32, _i32, _i32, P(_dbl), _u64, P(ssb_mbody_opts),
                                  P(P(ssb_net_desc)), _cp, _sz]),
    "ssb_build_izhikevich": (C.c_int, [_i32, _i32, _dbl, _dbl, _u64, P(ssb_izh_opts),
                                       P(P(ssb_net_desc)), _cp, _sz]),
    "ssb_net_desc_free": (None, [P(ssb_net_desc)]),
    "ssb_mbody_default_opts": (None, [P(ssb_mbody_opts)]),
    "ssb_izh_default_opts": (None, [P(ssb_izh_opts)]),
    "ssb_engine_default_opts": (None, [P(ssb_engine_opts)]),
    "ssb_fnv1a64": (_u64, [_cp]),
    "ssb_splitmix64": (_u64, [_u64]),
    "ssb_derive_seed": (_u64, [_u64, _cp]),
    "ssb_stream_u64": (C.c_int, [_u64, _u64, _cp, _i64, P(_u64)]),
    "ssb_gen_fixed_outdegree": (C.c_int, [_i32, _i32, _i32, _i32, _dbl, _dbl, _dbl, _i32, _u64,
                                          P(_f32), _cp, _sz]),
    "ssb_build_group": (C.c_int, [P(ssb_net_desc), _i32, _i32, P(_i32), P(_i32), P(_i32), P(_i64),
                                  P(_f32), P(_i32), P(_i64), _i64, _cp, _sz]),
    "ssb_sweep": (C.c_int, [P(P(ssb_net_desc)), _i32, _i32, _cp, _i32, P(ssb_engine_opts), P(_dbl),
                            P(_i64), P(_i32), _cp, _sz, _cp, _sz]),
    "ssb_shard_plan": (C.c_int, [P(ssb_net_desc), _i32, _i32, P(_i64), _cp, _sz]),
    "ssb_shard_group": (C.c_int, [P(ssb_net_desc), _i32, _i32, _i32, _i32, _i32, P(_i32), P(_i32),
                                  P(_i32), P(_i64), P(_f32), P(_i32), P(_i64), _i64, _cp, _sz]),
    "ssb_comm_unique_id": (C.c_int, [P(_u8), _cp, _sz]),
    "ssb_comm_selftest": (C.c_int, [_i32, _cp, _sz]),
    "ssb_mem_sparse_elements": (_u64, [_u64, _u64]),
    "ssb_mem_dense_elements": (_u64, [_u64, _u64]),
    "ssb_propagate_dense": (C.c_int, [P(_f32), _i32, _i32, P(_i32), _i64, P(_f32), _i64, _cp, _sz]),
    "ssb_propagate_crs": (C.c_int, [P(_f32), P(_i32), P(_i64), _i32, _i32, P(_i32), _i64, P(_f32),
                                    _i64, _cp, _sz]),
    "ssb_propagate_dense_dev": (C.c_int, [_vp, _i32, _i32, _vp, _i32, _vp, _vp]),
    "ssb_crs_segments_dev": (C.c_int, [_vp, _vp, _i32, _i32, _i32, _vp, _vp]),
    "ssb_propagate_crs_dev": (C.c_int, [_vp, _vp, _vp, _i32, _i32, _i32, _vp, _i32, _vp, _vp]),
    "ssb_crs_slices": (C.c_int, [_vp, _vp, _vp, _i32, _i32, _vp, _vp, _vp, _i64, _vp, C.c_char_p,
                                 C.c_size_t]),
    "ssb_propagate_crs_sliced_dev": (C.c_int, [_vp, _vp, _vp, _i32, _i32, _vp, _i32, _vp, _vp]),
    "ssb_detect_nans": (C.c_int, [_i32, P(_f32), P(_f32), P(_f32), P(_f32), P(_u8), _i64, P(_i64),
                                  P(_i64), _cp, _sz]),
    "ssb_create": (C.c_int, [P(ssb_net_desc), _i32, P(ssb_engine_opts), P(_vp), _cp, _sz]),
    "ssb_destroy": (None, [_vp]),
    "ssb_last_error": (_cp, [_vp]),
    "ssb_step": (C.c_int, [_vp, _i64]),
    "ssb_steps_total": (_i64, [_vp]),
    "ssb_world": (_i32, [_vp]),
    "ssb_shard_range": (C.c_int, [_vp, _i32, P(_i64), P(_i64), P(_i64)]),
    "ssb_steps_done": (_i64, [_vp]),
    "ssb_sync": (C.c_int, [_vp]),
    "ssb_pull_state": (C.c_int, [_vp, _i32, _i32, _vp, _i64]),
    "ssb_push_state": (C.c_int, [_vp, _i32, _i32, _vp, _i64]),
    "ssb_group_info": (C.c_int, [_vp, _i32, P(_i32), P(_i32), P(_i32), P(_i64)]),
    "ssb_group_dense": (C.c_int, [_vp, _i32, P(_f32), _i64]),
    "ssb_group_weights": (C.c_int, [_vp, _i32, P(_f32), _i64]),
    "ssb_group_sparse": (C.c_int, [_vp, _i32, P(_f32), P(_i32), P(_i64)]),
    "ssb_finish": (C.c_int, [_vp, P(ssb_run_summary)]),
    "ssb_result_rates": (C.c_int, [_vp, P(_dbl), _i32]),
    "ssb_result_n_events": (_i64, [_vp]),
    "ssb_result_raster": (C.c_int, [_vp, P(_i64), P(_i32), P(_i32), _i64]),
    "ssb_result_counts": (C.c_int, [_vp, P(_i32), _i64]),
    "ssb_result_neurons": (C.c_int, [_vp, P(_i32), _i64]),
    "ssb_spike_counts": (C.c_int, [_vp, P(_i64), _i32]),
    "ssb_raster_discard": (C.c_int, [_vp]),
    "ssb_raster_drain": (C.c_int, [_vp, P(_i64)]),
    "ssb_raster_drain_async": (C.c_int, [_vp]),
    "ssb_stream": (_vp, [_vp]),
    "ssb_window": (_i32, [_vp]),
    "ssb_block_size": (_i32, [_vp, _i32]),
    "ssb_grid_size": (_i32, [_vp, _i32]),
    "ssb_n_kernel_stats": (_i32, [_vp]),
    "ssb_kernel_stats": (C.c_int, [_vp, P(ssb_kernel_stat), _i32]),
    "ssb_kernel_stats_reset": (C.c_int, [_vp]),
    "ssb_device_bytes": (_i64, [_vp]),
    "ssb_kernel_launches": (_i64, [_vp]),
    "ssb_device_preset": (C.c_int, [_cp, P(ssb_device_spec), _cp, _sz]),
    "ssb_device_preset_names": (_cp, []),
    "ssb_device_query": (C.c_int, [_i32, P(ssb_device_spec), _cp, _sz]),
    "ssb_occupancy": (C.c_int, [P(ssb_device_spec), _i64, _i64, _i64, P(ssb_occupancy_result), _cp,
                                _sz]),
    "ssb_recommend_block_size": (C.c_int, [P(ssb_device_spec), _i64, _i64, P(_i64),
                                           P(ssb_occupancy_result), _cp, _sz]),
    "ssb_kernel_attributes": (C.c_int, [_cp, P(_i32), P(_i32), P(_i32)]),
}

EXPORTED = tuple(_SIGNATURES)


def _load() -> C.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build the CUDA library first "
            "(python -c 'import __graft_entry__ as g; g.build()'); there is no CPU fallback")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in _SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()
