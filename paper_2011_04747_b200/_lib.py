"""ctypes binding of libcwgpu.so (include/cwgpu.h, include/cwgpu_setup.h).

The product path: every call goes to the sm_100a kernels in libcwgpu.so.
There is no CPU fallback -- if the library is missing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CWG_LIB_PATH") or os.path.join(HERE, "libcwgpu.so")  # override: experiments only

CWG_OK, CWG_EVALIDATION, CWG_EINSTABILITY, CWG_EIO, CWG_ECUDA = 0, 2, 3, 4, 5
OP_AUTO, OP_CSR, OP_STENCIL2D, OP_STRUCT3D, OP_SHEET2D = 0, 1, 2, 3, 4


class cwg_error(C.Structure):
    _fields_ = [("code", C.c_int), ("node", C.c_int64), ("t_ms", C.c_double), ("phase", C.c_int),
                ("msg", C.c_char * 256)]


class cwg_struct3d(C.Structure):
    _fields_ = [("nx", C.c_int64), ("ny", C.c_int64), ("nz", C.c_int64), ("h", C.c_double),
                ("d_long", C.c_double), ("rho", C.c_double), ("fiber_angle_of_layer", C.POINTER(C.c_double))]


_dp = C.POINTER(C.c_double)
_lp = C.POINTER(C.c_int64)
_ip = C.POINTER(C.c_int)
_i32p = C.POINTER(C.c_int32)
_u8p = C.POINTER(C.c_uint8)


class cwg_sheet2d(C.Structure):
    _fields_ = [("nx", C.c_int64), ("ny", C.c_int64), ("h", C.c_double), ("fiber_angle", C.c_double),
                ("d0_myocyte", C.c_double), ("d0_fibrotic", C.c_double), ("rho", C.c_double),
                ("node_tags", _i32p), ("elem_scale", _dp)]


class cwg_problem(C.Structure):
    _fields_ = [
        ("n", C.c_int64), ("row_ptr", _lp), ("col", _lp), ("val", _dp), ("lumped_mass", _dp), ("dt_s", C.c_double),
        ("op_kind", C.c_int), ("grid_nx1", C.c_int64), ("grid_ny1", C.c_int64), ("s3d", C.POINTER(cwg_struct3d)),
        ("n_models", C.c_int), ("model_kind", _ip), ("model_of_node", _u8p), ("gkr_scale", _dp),
        ("n_stim", C.c_int), ("stim_t_start", _dp), ("stim_duration", _dp), ("stim_amplitude", _dp),
        ("stim_period", _dp), ("stim_node_ptr", _i32p), ("stim_ids", _i32p),
        ("n_probes", C.c_int), ("probes", _lp), ("lat_threshold_mv", C.c_double), ("map_interval_ms", C.c_double),
        ("scheme", C.c_int), ("dt_ms", C.c_double), ("t_end_ms", C.c_double), ("k0_up", C.c_int), ("k0_down", C.c_int),
        ("strict_substeps", C.c_int), ("record_interval_ms", C.c_double),
        ("device", C.c_int), ("rank", C.c_int), ("world", C.c_int), ("nccl_id", C.POINTER(C.c_ubyte)),
        ("sheet2d", C.POINTER(cwg_sheet2d)),
    ]


class cwg_threshold_options(C.Structure):
    _fields_ = [("duration_ms", C.c_double), ("upper_factor", C.c_double), ("initial_guess", C.c_double),
                ("rel_tol", C.c_double), ("window_ms", C.c_double), ("dt_ms", C.c_double)]


class cwg_info(C.Structure):
    _fields_ = [("dt_effective", C.c_double), ("dt_s", C.c_double), ("dt_ad", C.c_double), ("l", C.c_int),
                ("k_max_global", C.c_int), ("n_steps", C.c_int64), ("steps_per_record", C.c_int64),
                ("steps_per_map", C.c_int64), ("n_samples", C.c_int64), ("n_local", C.c_int64),
                ("node_begin", C.c_int64), ("op_kind", C.c_int)]


_SIGS = {
    "cwg_version": (C.c_char_p, []),
    "cwg_last_error": (C.c_char_p, []),
    "cwg_create": (C.c_int, [C.POINTER(cwg_problem), C.POINTER(C.c_void_p), C.POINTER(cwg_error)]),
    "cwg_destroy": (None, [C.c_void_p]),
    "cwg_set_stream": (C.c_int, [C.c_void_p, C.c_void_p]),
    "cwg_stream": (C.c_void_p, [C.c_void_p]),
    "cwg_upload_state": (C.c_int, [C.c_void_p, _dp, _dp, C.c_int, _dp]),
    "cwg_download_state": (C.c_int, [C.c_void_p, _dp, _dp, C.c_int, _dp]),
    "cwg_init_rest_state": (C.c_int, [C.c_void_p]),
    "cwg_struct3d_tables": (C.c_double, [C.POINTER(cwg_struct3d), _dp, _dp]),
    "cwg_pinned_buffers": (C.c_int, [C.c_void_p, C.POINTER(_dp), C.POINTER(_dp), C.POINTER(_dp)]),
    "cwg_advance": (C.c_int, [C.c_void_p, C.c_double, C.c_int64, C.c_int64, C.POINTER(cwg_error)]),
    "cwg_run_begin": (C.c_int, [C.c_void_p]),
    "cwg_run_steps": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64]),
    "cwg_run_sync": (C.c_int, [C.c_void_p, C.POINTER(cwg_error)]),
    "cwg_run": (C.c_int, [C.c_void_p, C.POINTER(cwg_error)]),
    "cwg_get_info": (C.c_int, [C.c_void_p, C.POINTER(cwg_info)]),
    "cwg_get_khist": (C.c_int, [C.c_void_p, _lp, C.c_int]),
    "cwg_get_traces": (C.c_int, [C.c_void_p, _dp, _dp]),
    "cwg_get_maps": (C.c_int, [C.c_void_p, _dp, _u8p, _dp, _u8p]),
    "cwg_trim_pool": (None, []),
    "cwg_gather_result": (C.c_int, [C.c_void_p, _dp, _dp, C.c_int, _dp, _dp, _u8p, _dp, _u8p]),
    "cwg_get_timing": (C.c_int, [C.c_void_p, _dp, _dp, _dp]),
    "cwg_launch_count": (C.c_int64, [C.c_void_p]),
    "cwg_bench_steps": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_int, _dp, _dp, _dp]),
    "cwg_reaction_evals": (C.c_int64, [C.c_void_p]),
    "cwg_react_trace": (C.c_int, [C.c_void_p, C.c_int]),
    "cwg_fp64_peak_tflops": (C.c_double, [C.c_int, C.c_double]),
    "cwg_diastolic_threshold": (C.c_int, [C.POINTER(cwg_problem), _dp, _lp, C.c_int64,
                                          C.POINTER(cwg_threshold_options), _dp, _lp, C.POINTER(cwg_error)]),
    "cwg_diffusion_substep": (C.c_int, [C.c_int64, _lp, _lp, _dp, _dp, _dp, C.c_double, _dp, C.c_int,
                                        C.POINTER(cwg_error)]),
    "cwg_rates": (C.c_int, [C.c_int, C.c_int64, _dp, _dp, _dp, _dp, _dp, C.c_int, C.POINTER(cwg_error)]),
    "cwg_set_scheme": (C.c_int, [C.c_void_p, C.c_int, C.c_double, C.c_double, C.c_int, C.c_int, C.c_int,
                                 C.POINTER(cwg_error)]),
    "cwg_loopback_steps": (C.c_int, [C.POINTER(C.c_void_p), C.c_int, C.c_int64, C.c_int64]),
    "cwg_loopback_link": (C.c_int, [C.POINTER(C.c_void_p), C.c_int]),
    "cwg_snapshot_begin": (C.c_int, [C.c_void_p, _dp]),
    "cwg_snapshot_wait": (C.c_int, [C.c_void_p, C.POINTER(cwg_error)]),
    "cwg_host_register": (C.c_int, [C.c_void_p, C.c_size_t]),
    "cwg_host_unregister": (C.c_int, [C.c_void_p]),
    "cwg_pace_cells": (C.c_int, [C.c_int, C.c_int64, _dp, _dp, _dp, C.c_int, _dp, _dp, _dp, C.POINTER(C.c_int), _dp,
                                 C.c_int, C.POINTER(cwg_error)]),
    "cwg_model_state_count": (C.c_int, [C.c_int]),
    "cwg_model_stable_step": (C.c_double, [C.c_int]),
    "cwg_model_rest_state": (C.c_int, [C.c_int, _dp]),
    "cwg_model_kind_from_name": (C.c_int, [C.c_char_p]),
    "cwg_reaction_substeps": (C.c_int, [C.c_double, C.c_int, C.c_int, C.c_int, C.c_int]),
    "cwg_diffusion_substeps": (C.c_int, [C.c_double, C.c_double, C.c_int, C.c_int, _ip, _dp]),
    "cwg_k_max_for": (C.c_int, [C.c_double, C.c_int]),
    "cwg_slab_plan": (C.c_int, [C.c_int64, C.c_int, C.c_int, _lp, _lp]),
    "cwg_sheet2d_nnz": (C.c_int64, [C.POINTER(cwg_sheet2d)]),
    "cwg_sheet2d_assemble": (C.c_int, [C.POINTER(cwg_sheet2d), C.c_int, _lp, _lp, _dp, _dp, _dp,
                                       C.POINTER(cwg_error)]),
    # setup (cwgpu_setup.h)
    "cwg_sheet_build": (C.c_int, [C.c_double, C.c_double, C.c_double, C.c_double, C.c_double, C.c_double,
                                  C.c_double, C.c_double, C.c_uint64, _dp, C.POINTER(C.c_void_p),
                                  C.POINTER(cwg_error)]),
    "cwg_sheet_free": (None, [C.c_void_p]),
    "cwg_sheet_mesh": (C.c_int, [C.c_double, C.c_double, C.c_double, C.c_double, C.c_uint64, C.POINTER(C.c_void_p),
                                 C.POINTER(cwg_error)]),
    "cwg_sheet_nodes": (C.c_int64, [C.c_void_p]),
    "cwg_sheet_elements": (C.c_int64, [C.c_void_p]),
    "cwg_sheet_nnz": (C.c_int64, [C.c_void_p]),
    "cwg_sheet_nx1": (C.c_int64, [C.c_void_p]),
    "cwg_sheet_ny1": (C.c_int64, [C.c_void_p]),
    "cwg_sheet_dt_s": (C.c_double, [C.c_void_p]),
    "cwg_sheet_row_ptr": (_lp, [C.c_void_p]),
    "cwg_sheet_col": (_lp, [C.c_void_p]),
    "cwg_sheet_val": (_dp, [C.c_void_p]),
    "cwg_sheet_mass": (_dp, [C.c_void_p]),
    "cwg_sheet_coords": (_dp, [C.c_void_p]),
    "cwg_sheet_tags": (_i32p, [C.c_void_p]),
    "cwg_sheet_select": (C.c_int64, [C.c_void_p, C.c_int, _dp, _lp, C.c_int64, _lp, C.c_int64]),
    "cwg_sheet_nearest": (C.c_int64, [C.c_void_p, C.c_double, C.c_double]),
    "cwg_uniform_mt64": (None, [C.c_uint64, C.c_int64, C.c_double, C.c_double, _dp]),
}

EXPORTED = tuple(_SIGS)

_lib = None


def lib():
    """Load libcwgpu.so. Raises (never falls back) when the extension is missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() (nvcc, sm_100a)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def dp(a):
    return a.ctypes.data_as(_dp)


def lp(a):
    return a.ctypes.data_as(_lp)
