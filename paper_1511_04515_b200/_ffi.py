"""ctypes bindings of the C ABI (include/exg.h, include/exg_host.h).

The shared library ``libexg.so`` is built in-tree (``__graft_entry__.build()``)
next to this file.  There is no fallback: if the library is missing, importing
the package raises ``ImportError`` with the build command.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("EXG_LIB", _HERE / "libexg.so"))

# ---- status codes (exg.h) ---------------------------------------------------
EXG_OK = 0
EXG_E_CONTRACT = 1
EXG_E_NONFINITE = 2
EXG_E_SINGULAR = 3
EXG_E_ZERO_START = 4
EXG_E_NO_CONVERGENCE = 5
EXG_E_SINGULAR_REDUCED = 6
EXG_E_NO_DC = 7
EXG_E_STEP_FAILURE = 8
EXG_E_CUDA = 100
EXG_E_NOMEM = 101

EXG_MAT_C, EXG_MAT_G, EXG_MAT_B = 0, 1, 2
EXG_PTR_HOST, EXG_PTR_DEVICE = 0, 1
EXG_TRSV_EXACT, EXG_TRSV_FAST = 0, 1
EXG_WEIGHT_APPLY, EXG_WEIGHT_GSPMV = 0, 1
EXG_LOOP_GRAPH, EXG_LOOP_EAGER = 0, 1
EXG_METHOD_ER, EXG_METHOD_ERC = 1, 2

EXG_EL_R, EXG_EL_C, EXG_EL_L, EXG_EL_V, EXG_EL_I, EXG_EL_M = range(6)
EXG_SRC_DC, EXG_SRC_PWL, EXG_SRC_PULSE = range(3)


class exg_element(C.Structure):
    _fields_ = [("kind", C.c_int32), ("nodes", C.c_int32 * 4), ("aux", C.c_int32),
                ("value", C.c_double)]


class exg_source(C.Structure):
    _fields_ = [("kind", C.c_int32), ("pwl_off", C.c_int32), ("pwl_len", C.c_int32),
                ("pad", C.c_int32), ("dc", C.c_double), ("v1", C.c_double), ("v2", C.c_double),
                ("delay", C.c_double), ("rise", C.c_double), ("fall", C.c_double),
                ("width", C.c_double), ("period", C.c_double)]


class exg_mos_model(C.Structure):
    _fields_ = [("vth", C.c_double), ("kp", C.c_double), ("lam", C.c_double), ("w", C.c_double),
                ("l", C.c_double), ("cgs0", C.c_double), ("cgd0", C.c_double),
                ("pmos", C.c_int32), ("pad", C.c_int32)]


class exg_options(C.Structure):
    _fields_ = [("err_budget", C.c_double), ("krylov_eps", C.c_double), ("gmin", C.c_double),
                ("m_max", C.c_int32), ("has_tran", C.c_int32), ("hmin", C.c_double),
                ("hmax", C.c_double), ("tran_step", C.c_double), ("tran_stop", C.c_double)]


class exg_gen_params(C.Structure):
    _fields_ = [("config", C.c_int32), ("width", C.c_int32), ("height", C.c_int32),
                ("n", C.c_int32), ("seed", C.c_uint64), ("chains", C.c_int32),
                ("stages", C.c_int32)]


class exg_step_control(C.Structure):
    _fields_ = [("err_budget", C.c_double), ("alpha", C.c_double), ("beta", C.c_double),
                ("grow_threshold", C.c_int32), ("grow_only_on_clean", C.c_int32),
                ("eps", C.c_double), ("m_max", C.c_int32), ("max_rejects", C.c_int32),
                ("h_init", C.c_double), ("hmin", C.c_double), ("hmax", C.c_double),
                ("fixed_step", C.c_int32), ("method", C.c_int32), ("gamma", C.c_double),
                ("refactor_threshold", C.c_double)]


class exg_mevp_cfg(C.Structure):
    _fields_ = [("eps", C.c_double), ("m_max", C.c_int32), ("check_stride", C.c_int32),
                ("breakdown_tol", C.c_double)]


class exg_mevp_info(C.Structure):
    _fields_ = [("m", C.c_int32), ("happy", C.c_int32), ("beta", C.c_double),
                ("h_next", C.c_double), ("h_sub", C.c_double), ("last_residual", C.c_double)]


class exg_options_dev(C.Structure):
    _fields_ = [("trsv_mode", C.c_int32), ("weight_mode", C.c_int32), ("loop_mode", C.c_int32)]


class exg_counters(C.Structure):
    _fields_ = [("kernel_launches", C.c_int64), ("arnoldi_iters", C.c_int64),
                ("mevp_calls", C.c_int64), ("trsv_calls", C.c_int64), ("l_levels", C.c_int32),
                ("u_levels", C.c_int32), ("nnz_l", C.c_int64), ("nnz_u", C.c_int64),
                ("graph_launches", C.c_int64), ("graph_builds", C.c_int64),
                ("l_schedule", C.c_int32), ("u_schedule", C.c_int32), ("mgs_passes", C.c_int64),
                ("reorths", C.c_int64),
                ("fast_levels_l", C.c_int32), ("fast_levels_u", C.c_int32),
                ("fast_tasks_l", C.c_int64), ("fast_tasks_u", C.c_int64),
                ("fast_bytes_l", C.c_int64), ("fast_bytes_u", C.c_int64)]


class exg_kernel_times(C.Structure):
    _fields_ = [("ms", C.c_double * 7), ("count", C.c_int64 * 7)]


KERNEL_CLASSES = ["trsv_l", "trsv_u", "spmv", "mgs", "dense", "weight", "other"]

P = C.c_void_p
I = C.c_int
D = C.c_double
PI = C.POINTER(C.c_int)
PD = C.POINTER(C.c_double)

_HOST_PROTOS = {
    "exg_host_error_message": (C.c_char_p, []),
    "exg_system_generate": (I, [C.POINTER(exg_gen_params), C.POINTER(P)]),
    "exg_system_build": (I, [I, C.POINTER(exg_element), I, C.POINTER(exg_source), I, PD, PD, I,
                             C.POINTER(exg_mos_model), C.POINTER(exg_options), C.POINTER(P)]),
    "exg_system_free": (None, [P]),
    "exg_system_n": (I, [P]),
    "exg_system_n_nodes": (I, [P]),
    "exg_system_n_inputs": (I, [P]),
    "exg_system_n_mos": (I, [P]),
    "exg_system_csr": (I, [P, I, PI, PI, PI, C.POINTER(PI), C.POINTER(PI), C.POINTER(PD)]),
    "exg_system_elements": (I, [P, PI, C.POINTER(C.POINTER(exg_element)), PI,
                                C.POINTER(C.POINTER(exg_source)), PI, C.POINTER(PD),
                                C.POINTER(PD), PI, C.POINTER(C.POINTER(exg_mos_model))]),
    "exg_system_options": (I, [P, C.POINTER(exg_options)]),
    "exg_system_unknown_of_label": (I, [P, I]),
    "exg_sources_eval": (I, [P, D, PD]),
    "exg_breakpoints": (I, [P, D, D, PD, I]),
    "exg_dc_solve": (I, [P, PD]),
    "exg_linearize": (I, [P, PD, I, PI, PI, PI, PD, PD]),
    "exg_residual_F_host": (I, [P, PD, PD, PD]),
    "exg_lu_factor": (I, [I, PI, PI, PD, D, C.POINTER(P)]),
    "exg_factor_free": (None, [P]),
    "exg_aug_plan_solve": (I, [I, I, PI, PI, PD, PD, PI, PI, PD, PD, C.POINTER(C.c_longlong)]),
    "exg_stream_plan_solve": (I, [I, I, PI, PI, PD, PD, PI, PI, PI, I, PD, PD, PD, D, PD,
                                  C.POINTER(C.c_longlong)]),
    "exg_factor_get": (I, [P, PI, C.POINTER(PI), C.POINTER(PI), C.POINTER(PD), C.POINTER(PI),
                           C.POINTER(PI), C.POINTER(PD), C.POINTER(PI), C.POINTER(PI)]),
    "exg_factor_timing": (I, [P, PD, PD]),
    "exg_step_control_from": (I, [P, C.POINTER(exg_step_control)]),
}

_DEV_PROTOS = {
    "exg_create": (I, [I, C.POINTER(P)]),
    "exg_destroy": (None, [P]),
    "exg_last_error": (I, [P, C.c_char_p, C.c_size_t]),
    "exg_set_options": (I, [P, C.POINTER(exg_options_dev)]),
    "exg_set_csr": (I, [P, I, I, I, I, PI, PI, PD]),
    "exg_update_values": (I, [P, I, PD]),
    "exg_set_factors": (I, [P, I, PI, PI, PD, PI, PI, PD, PI, PI]),
    "exg_spmv": (I, [P, I, P, P, I]),
    "exg_solve": (I, [P, P, P, I]),
    "exg_apply": (I, [P, P, P, I]),
    "exg_mevp_iks": (I, [P, P, D, C.POINTER(exg_mevp_cfg), P, C.POINTER(exg_mevp_info), I]),
    "exg_basis_residual": (I, [P, D, PD]),
    "exg_basis_eval": (I, [P, D, P, I]),
    "exg_er_begin": (I, [P, P, P, P, D, I]),
    "exg_er_eval": (I, [P, D, C.POINTER(exg_mevp_cfg), P, PI, C.POINTER(exg_mevp_info), I]),
    "exg_er_step": (I, [P, P, P, P, D, C.POINTER(exg_mevp_cfg), P, PI, I]),
    "exg_gather": (I, [P, PI, I, PD]),
    "exg_set_devices": (I, [P, I, PI, PD]),
    "exg_set_oppoints": (I, [P, PD]),
    "exg_residual_F": (I, [P, P, P, I]),
    "exg_er_nonlinear": (I, [P, D, C.POINTER(exg_mevp_cfg), I, D, PD, PI, PI]),
    "exg_counters_get": (I, [P, C.POINTER(exg_counters)]),
    "exg_counters_reset": (I, [P]),
    "exg_profile_enable": (I, [P, I]),
    "exg_debug_trace_solve": (I, [P, PD, C.POINTER(C.c_uint64)]),
    "exg_debug_dense_expm": (I, [P, I, PD, PD]),
    "exg_debug_spmv_fast": (I, [P, PD, PD]),
    "exg_debug_orthogonalize": (I, [P, I, I, PD, PD, D, PD, PD, PI]),
    "exg_debug_trace_stream": (I, [P, PD, C.POINTER(C.c_uint64), C.POINTER(C.c_longlong)]),
    "exg_profile_get": (I, [P, C.POINTER(exg_kernel_times)]),
    "exg_synchronize": (I, [P]),
    "exg_device_alloc": (I, [P, C.c_size_t, C.POINTER(P)]),
    "exg_device_free": (I, [P, P]),
    "exg_memcpy": (I, [P, P, P, C.c_size_t, I]),
    "exg_stream": (P, [P]),
    "exg_transient": (I, [P, P, C.POINTER(exg_step_control), D, PI, I, C.POINTER(P)]),
    "exg_tran_result_free": (None, [P]),
    "exg_tran_n_times": (I, [P]),
    "exg_tran_n_rec": (I, [P]),
    "exg_tran_times": (PD, [P]),
    "exg_tran_samples": (PD, [P]),
    "exg_tran_n_steps": (I, [P]),
    "exg_tran_records": (I, [P, PD, PD, PI, PI, PD, PI]),
    "exg_tran_n_dims": (I, [P]),
    "exg_tran_dims": (PI, [P]),
    "exg_tran_timing": (I, [P, PD, PD, PD]),
    "exg_tran_write_csv": (I, [P, C.c_char_p, C.POINTER(C.c_char_p), I]),
    "exg_write_waveform_csv": (I, [C.c_char_p, I, I, PD, PD, C.POINTER(C.c_char_p), I]),
}


def _load():
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is missing: build the CUDA extension first "
            "(python -c 'import __graft_entry__ as g; g.build()')")
    lib = C.CDLL(str(LIB_PATH))
    for name, (res, args) in {**_HOST_PROTOS, **_DEV_PROTOS}.items():
        fn = getattr(lib, name, None)
        if fn is None:
            if name in _DEV_PROTOS and os.environ.get("EXG_HOST_ONLY"):
                continue
            raise ImportError(f"{LIB_PATH} does not export {name}")
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


def declared_symbols():
    """Every symbol include/exg.h and include/exg_host.h declare."""
    return sorted(set(_HOST_PROTOS) - {"exg_host_error_message"} | set(_DEV_PROTOS))


def as_ptr(a: np.ndarray, ctype):
    return a.ctypes.data_as(C.POINTER(ctype))


def i32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int32)


def f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)
