"""Python mirror of the device hot path (include/exg.h).

``Context`` owns one device context (own stream, device memory) and exposes
the reference's hot-path functions under their reference names:

=====================  =====================================================
``spmv``               exsim::spmv (sparse_matrix.cpp:69-82)
``solve`` / ``apply``  exsim::Factorization::solve / apply (sparse_lu.cpp:255-304)
``mevp_iks``           exsim::mevp_iks (krylov.cpp:177-182, :103-173)
``mevp_residual``      exsim::mevp_residual (krylov.cpp:191-205), cached basis
``eval_at_scaled_h``   exsim::eval_at_scaled_h (krylov.cpp:207-215), cached basis
``er_step``            exsim::er_step (integrate.cpp:302-316), linear part
``transient``          exsim::transient ER branch (integrate.cpp:368-480)
=====================  =====================================================

All arithmetic runs in libexg.so on the GPU; there is no host fallback.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _ffi as F
from .errors import raise_for
from .host import Csr, Factorization, System


@dataclass
class MevpInfo:
    m: int
    happy: bool
    beta: float
    h_next: float
    h_sub: float
    last_residual: float


@dataclass
class TransientResult:
    times: np.ndarray
    samples: np.ndarray          # n_times x n_rec
    t: np.ndarray                # per-step StepRecord fields
    h: np.ndarray
    lu_count: np.ndarray
    rejects: np.ndarray
    err_norm: np.ndarray
    krylov_dims: list            # per step list of Krylov dimensions
    lu_s: float
    dc_s: float
    loop_s: float


class Context:
    def __init__(self, device: int = 0, trsv_mode: int = F.EXG_TRSV_EXACT,
                 weight_mode: int = F.EXG_WEIGHT_APPLY, loop_mode: int = F.EXG_LOOP_GRAPH):
        h = C.c_void_p()
        st = F.lib.exg_create(device, C.byref(h))
        if st != F.EXG_OK:
            raise_for(st, f"exg_create(device={device}) failed (is an sm_100 GPU visible?)")
        self._h = h
        self.n = 0
        self.set_options(trsv_mode, weight_mode, loop_mode)

    def close(self):
        if getattr(self, "_h", None):
            F.lib.exg_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    @property
    def handle(self):
        return self._h

    def _check(self, st: int, value: float | None = None):
        if st != F.EXG_OK:
            buf = C.create_string_buffer(512)
            F.lib.exg_last_error(self._h, buf, 512)
            raise_for(st, buf.value.decode(), value)

    def set_options(self, trsv_mode: int = F.EXG_TRSV_EXACT, weight_mode: int = F.EXG_WEIGHT_APPLY,
                    loop_mode: int = F.EXG_LOOP_GRAPH):
        o = F.exg_options_dev(trsv_mode, weight_mode, loop_mode)
        self._check(F.lib.exg_set_options(self._h, C.byref(o)))

    # ---- device store
    def set_csr(self, which: int, A: Csr):
        rp, ci, va = F.i32(A.rowptr), F.i32(A.col), F.f64(A.val)
        self._check(F.lib.exg_set_csr(self._h, which, A.n_rows, A.n_cols, A.nnz,
                                      F.as_ptr(rp, C.c_int), F.as_ptr(ci, C.c_int),
                                      F.as_ptr(va, C.c_double)))

    def set_system(self, sys: System):
        for w in (F.EXG_MAT_C, F.EXG_MAT_G, F.EXG_MAT_B):
            self.set_csr(w, sys.csr(w))

    def set_factors(self, f: Factorization):
        arrs = [F.i32(f.L.rowptr), F.i32(f.L.col), F.f64(f.L.val), F.i32(f.U.rowptr),
                F.i32(f.U.col), F.f64(f.U.val), F.i32(f.row_perm), F.i32(f.col_perm)]
        ts = [C.c_int, C.c_int, C.c_double, C.c_int, C.c_int, C.c_double, C.c_int, C.c_int]
        self._check(F.lib.exg_set_factors(self._h, f.n, *[F.as_ptr(a, t) for a, t in zip(arrs, ts)]))
        self.n = f.n

    # ---- hot path (host buffers)
    def spmv(self, which: int, x: np.ndarray, n_rows: int) -> np.ndarray:
        x = F.f64(x)
        y = np.zeros(n_rows)
        self._check(F.lib.exg_spmv(self._h, which, x.ctypes.data, y.ctypes.data, F.EXG_PTR_HOST))
        return y

    def solve(self, b: np.ndarray) -> np.ndarray:
        b = F.f64(b)
        x = np.zeros_like(b)
        self._check(F.lib.exg_solve(self._h, b.ctypes.data, x.ctypes.data, F.EXG_PTR_HOST))
        return x

    def apply(self, x: np.ndarray) -> np.ndarray:
        x = F.f64(x)
        y = np.zeros_like(x)
        self._check(F.lib.exg_apply(self._h, x.ctypes.data, y.ctypes.data, F.EXG_PTR_HOST))
        return y

    def mevp_iks(self, v: np.ndarray, h: float, eps: float = 1e-7, m_max: int = 100,
                 check_stride: int = 1, breakdown_tol: float = 1e-12):
        v = F.f64(v)
        out = np.zeros_like(v)
        cfg = F.exg_mevp_cfg(eps, m_max, check_stride, breakdown_tol)
        info = F.exg_mevp_info()
        st = F.lib.exg_mevp_iks(self._h, v.ctypes.data, h, C.byref(cfg), out.ctypes.data,
                                C.byref(info), F.EXG_PTR_HOST)
        self._check(st, info.last_residual)
        return out, MevpInfo(info.m, bool(info.happy), info.beta, info.h_next, info.h_sub,
                             info.last_residual)

    def mevp_residual(self, h: float) -> float:
        r = C.c_double()
        self._check(F.lib.exg_basis_residual(self._h, h, C.byref(r)))
        return r.value

    def eval_at_scaled_h(self, h: float) -> np.ndarray:
        out = np.zeros(self.n)
        self._check(F.lib.exg_basis_eval(self._h, h, out.ctypes.data, F.EXG_PTR_HOST))
        return out

    def er_step(self, x_k, u_k, u_k1, h: float, eps: float = 1e-7, m_max: int = 100):
        x_k, u_k, u_k1 = F.f64(x_k), F.f64(u_k), F.f64(u_k1)
        xn = np.zeros_like(x_k)
        m = C.c_int(-1)
        cfg = F.exg_mevp_cfg(eps, m_max, 1, 1e-12)
        self._check(F.lib.exg_er_step(self._h, x_k.ctypes.data, u_k.ctypes.data, u_k1.ctypes.data,
                                      h, C.byref(cfg), xn.ctypes.data, C.byref(m), F.EXG_PTR_HOST))
        return xn, m.value

    # ---- nonlinear devices (config 4)
    def set_devices(self, sys: System):
        """MOSFET table of `sys` (devices.cpp:122-167 device data) onto the device."""
        elems, _, _, _, models = sys.elements()
        nodes, par = [], []
        for e in elems:
            if e.kind != F.EXG_EL_M:
                continue
            m = models[e.aux]
            nodes.append([sys.unknown_of_label(e.nodes[j]) if e.nodes[j] >= 0 else -1 for j in range(4)])
            par.append([m.vth, m.kp, m.lam, m.w, m.l, float(m.pmos)])
        nodes = np.ascontiguousarray(nodes, np.int32).reshape(-1, 4)
        par = np.ascontiguousarray(par, np.float64).reshape(-1, 6)
        self._check(F.lib.exg_set_devices(self._h, nodes.shape[0], F.as_ptr(nodes, C.c_int),
                                          F.as_ptr(par, C.c_double)))

    def set_oppoints(self, op):
        op = F.f64(op)
        self._check(F.lib.exg_set_oppoints(self._h, F.as_ptr(op, C.c_double)))

    def residual_F(self, x) -> np.ndarray:
        x = F.f64(x)
        out = np.zeros(self.n)
        self._check(F.lib.exg_residual_F(self._h, x.ctypes.data, out.ctypes.data, F.EXG_PTR_HOST))
        return out

    def counters(self) -> F.exg_counters:
        c = F.exg_counters()
        self._check(F.lib.exg_counters_get(self._h, C.byref(c)))
        return c

    def reset_counters(self):
        self._check(F.lib.exg_counters_reset(self._h))

    def synchronize(self):
        self._check(F.lib.exg_synchronize(self._h))

    # ---- whole transient
    def transient(self, sys: System, ctl: F.exg_step_control, t_stop: float, rec_idx, csv_path=None,
                  csv_columns=None) -> TransientResult:
        """exg_transient; csv_path: also write the recorded waveform as the reference CLI's CSV
        (exg_tran_write_csv; csv_columns default to the record indices)."""
        ri = F.i32(rec_idx)
        rh = C.c_void_p()
        self._check(F.lib.exg_transient(self._h, sys._h, C.byref(ctl), t_stop,
                                        F.as_ptr(ri, C.c_int), ri.size, C.byref(rh)))
        L = F.lib
        try:
            nt, nr, ns = L.exg_tran_n_times(rh), L.exg_tran_n_rec(rh), L.exg_tran_n_steps(rh)
            if csv_path is not None:
                cols = csv_columns if csv_columns is not None else [f"x{i}" for i in (ri if ri.size else range(nr))]
                names = (C.c_char_p * max(nr, 1))(*[str(c).encode() for c in cols])
                self._check(L.exg_tran_write_csv(rh, str(csv_path).encode(), names, 0))
            times = np.ctypeslib.as_array(L.exg_tran_times(rh), (nt,)).copy()
            samples = np.ctypeslib.as_array(L.exg_tran_samples(rh), (nt * nr,)).copy().reshape(nt, nr) \
                if nt * nr else np.zeros((nt, nr))
            t, h, err = np.zeros(ns), np.zeros(ns), np.zeros(ns)
            lu, rej, off = np.zeros(ns, np.int32), np.zeros(ns, np.int32), np.zeros(ns + 1, np.int32)
            L.exg_tran_records(rh, F.as_ptr(t, C.c_double), F.as_ptr(h, C.c_double),
                               F.as_ptr(lu, C.c_int), F.as_ptr(rej, C.c_int),
                               F.as_ptr(err, C.c_double), F.as_ptr(off, C.c_int))
            nd = L.exg_tran_n_dims(rh)
            dims = np.ctypeslib.as_array(L.exg_tran_dims(rh), (nd,)).copy() if nd else np.zeros(0, np.int32)
            a, b, c = C.c_double(), C.c_double(), C.c_double()
            L.exg_tran_timing(rh, C.byref(a), C.byref(b), C.byref(c))
            kd = [dims[off[i]:off[i + 1]].tolist() for i in range(ns)]
            return TransientResult(times, samples, t, h, lu, rej, err, kd, a.value, b.value, c.value)
        finally:
            L.exg_tran_result_free(rh)
