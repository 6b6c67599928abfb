"""Host-side Python mirror of the reference front end (include/exg_host.h).

Names follow the reference: ``System`` ~ ``exsim::MnaSystem`` (mna.hpp:44-58),
``lu_factor`` ~ ``exsim::lu_factor`` (sparse_lu.hpp:56), ``Factorization`` ~
``exsim::Factorization`` (sparse_lu.hpp:16-42), ``StepControl`` ~
``exsim::StepControl`` (integrate.hpp:27-46).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _ffi as F
from .errors import raise_for


@dataclass
class Csr:
    n_rows: int
    n_cols: int
    rowptr: np.ndarray
    col: np.ndarray
    val: np.ndarray

    @property
    def nnz(self) -> int:
        return int(self.val.size)

    def to_dense(self) -> np.ndarray:
        d = np.zeros((self.n_rows, self.n_cols))
        for r in range(self.n_rows):
            s, e = self.rowptr[r], self.rowptr[r + 1]
            d[r, self.col[s:e]] = self.val[s:e]
        return d


def _check(st: int) -> None:
    if st != F.EXG_OK:
        raise_for(st, F.lib.exg_host_error_message().decode())


class System:
    """MNA system: C, G, B (CSR), sources, options."""

    def __init__(self, handle):
        self._h = handle

    @classmethod
    def generate(cls, config: int, width: int = 0, height: int = 0, n: int = 0, seed: int = 0,
                 chains: int = 0, stages: int = 0) -> "System":
        p = F.exg_gen_params(config, width, height, n, seed, chains, stages)
        h = C.c_void_p()
        _check(F.lib.exg_system_generate(C.byref(p), C.byref(h)))
        sys_ = cls(h)
        sys_.config = config
        return sys_

    @classmethod
    def build(cls, elems, sources, pwl_t, pwl_v, models, opts) -> "System":
        h = C.c_void_p()
        pt = F.f64(pwl_t)
        pv = F.f64(pwl_v)
        _check(F.lib.exg_system_build(len(elems), elems, len(sources), sources, pt.size,
                                      F.as_ptr(pt, C.c_double), F.as_ptr(pv, C.c_double),
                                      len(models), models, C.byref(opts), C.byref(h)))
        return cls(h)

    def __del__(self):
        if getattr(self, "_h", None):
            F.lib.exg_system_free(self._h)
            self._h = None

    @property
    def n(self) -> int:
        return F.lib.exg_system_n(self._h)

    @property
    def n_nodes(self) -> int:
        return F.lib.exg_system_n_nodes(self._h)

    @property
    def n_inputs(self) -> int:
        return F.lib.exg_system_n_inputs(self._h)

    def csr(self, which: int) -> Csr:
        nr, nc, nnz = C.c_int(), C.c_int(), C.c_int()
        rp, ci = C.POINTER(C.c_int)(), C.POINTER(C.c_int)()
        va = C.POINTER(C.c_double)()
        _check(F.lib.exg_system_csr(self._h, which, C.byref(nr), C.byref(nc), C.byref(nnz),
                                    C.byref(rp), C.byref(ci), C.byref(va)))
        nnz = nnz.value
        return Csr(nr.value, nc.value,
                   np.ctypeslib.as_array(rp, (nr.value + 1,)).copy(),
                   np.ctypeslib.as_array(ci, (max(nnz, 1),))[:nnz].copy() if nnz else np.zeros(0, np.int32),
                   np.ctypeslib.as_array(va, (max(nnz, 1),))[:nnz].copy() if nnz else np.zeros(0))

    @property
    def C(self) -> Csr:
        return self.csr(F.EXG_MAT_C)

    @property
    def G(self) -> Csr:
        return self.csr(F.EXG_MAT_G)

    @property
    def B(self) -> Csr:
        return self.csr(F.EXG_MAT_B)

    def elements(self):
        ne, ns, npwl, nm = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        pe = C.POINTER(F.exg_element)()
        ps = C.POINTER(F.exg_source)()
        pt, pv = C.POINTER(C.c_double)(), C.POINTER(C.c_double)()
        pm = C.POINTER(F.exg_mos_model)()
        _check(F.lib.exg_system_elements(self._h, C.byref(ne), C.byref(pe), C.byref(ns),
                                         C.byref(ps), C.byref(npwl), C.byref(pt), C.byref(pv),
                                         C.byref(nm), C.byref(pm)))
        elems = (F.exg_element * ne.value).from_address(C.addressof(pe.contents)) if ne.value else (F.exg_element * 0)()
        srcs = (F.exg_source * ns.value).from_address(C.addressof(ps.contents)) if ns.value else (F.exg_source * 0)()
        models = (F.exg_mos_model * nm.value).from_address(C.addressof(pm.contents)) if nm.value else (F.exg_mos_model * 0)()
        pwl_t = np.ctypeslib.as_array(pt, (npwl.value,)).copy() if npwl.value else np.zeros(0)
        pwl_v = np.ctypeslib.as_array(pv, (npwl.value,)).copy() if npwl.value else np.zeros(0)
        return elems, srcs, pwl_t, pwl_v, models

    def options(self) -> F.exg_options:
        o = F.exg_options()
        _check(F.lib.exg_system_options(self._h, C.byref(o)))
        return o

    def unknown_of_label(self, label: int) -> int:
        return F.lib.exg_system_unknown_of_label(self._h, label)

    def eval_sources(self, t: float) -> np.ndarray:
        u = np.zeros(self.n_inputs)
        _check(F.lib.exg_sources_eval(self._h, t, F.as_ptr(u, C.c_double)))
        return u

    def breakpoints(self, t0: float, t1: float) -> np.ndarray:
        cnt = F.lib.exg_breakpoints(self._h, t0, t1, None, 0)
        out = np.zeros(max(cnt, 1))
        F.lib.exg_breakpoints(self._h, t0, t1, F.as_ptr(out, C.c_double), cnt)
        return out[:cnt]

    @property
    def n_mos(self) -> int:
        return F.lib.exg_system_n_mos(self._h)

    def dc_solve(self) -> np.ndarray:
        """exsim::dc_solve (integrate.cpp:92-115), bit-identical."""
        x = np.zeros(self.n)
        _check(F.lib.exg_dc_solve(self._h, F.as_ptr(x, C.c_double)))
        return x

    def linearize(self, x):
        """exsim::evaluate (devices.cpp:122-200): (C_k, G_k, op[n_mos, 5])."""
        x = F.f64(x)
        out = []
        for which in (F.EXG_MAT_C, F.EXG_MAT_G):
            nnz = C.c_int()
            _check(F.lib.exg_linearize(self._h, F.as_ptr(x, C.c_double), which, C.byref(nnz),
                                       None, None, None, None))
            rp = np.zeros(self.n + 1, np.int32)
            ci = np.zeros(nnz.value, np.int32)
            va = np.zeros(nnz.value)
            op = np.zeros((self.n_mos, 5))
            _check(F.lib.exg_linearize(self._h, F.as_ptr(x, C.c_double), which, C.byref(nnz),
                                       F.as_ptr(rp, C.c_int), F.as_ptr(ci, C.c_int),
                                       F.as_ptr(va, C.c_double), F.as_ptr(op, C.c_double)))
            out.append((Csr(self.n, self.n, rp, ci, va), op))
        return out[0][0], out[1][0], out[1][1]

    def residual_F(self, x_ref, x) -> np.ndarray:
        """exsim::residual_F(evaluate(x_ref), x) (devices.cpp:202-233)."""
        x_ref, x = F.f64(x_ref), F.f64(x)
        out = np.zeros(self.n)
        _check(F.lib.exg_residual_F_host(self._h, F.as_ptr(x_ref, C.c_double), F.as_ptr(x, C.c_double),
                                         F.as_ptr(out, C.c_double)))
        return out

    def step_control(self) -> F.exg_step_control:
        c = F.exg_step_control()
        _check(F.lib.exg_step_control_from(self._h, C.byref(c)))
        return c


@dataclass
class Factorization:
    n: int
    L: Csr
    U: Csr
    row_perm: np.ndarray
    col_perm: np.ndarray
    order_s: float = 0.0
    numeric_s: float = 0.0

    @property
    def fill_nnz(self) -> int:
        return self.L.nnz + self.U.nnz


def lu_factor(A: Csr, pivot_tol: float = 0.1) -> Factorization:
    """Bit-identical restatement of exsim::lu_factor (sparse_lu.cpp:134-253)."""
    h = C.c_void_p()
    rp, ci, va = F.i32(A.rowptr), F.i32(A.col), F.f64(A.val)
    _check(F.lib.exg_lu_factor(A.n_rows, F.as_ptr(rp, C.c_int), F.as_ptr(ci, C.c_int),
                               F.as_ptr(va, C.c_double), pivot_tol, C.byref(h)))
    try:
        n = C.c_int()
        ptrs = [C.POINTER(C.c_int)() if k in (0, 1, 3, 4, 6, 7) else C.POINTER(C.c_double)()
                for k in range(8)]
        _check(F.lib.exg_factor_get(h, C.byref(n), *[C.byref(p) for p in ptrs]))
        n = n.value
        Lp = np.ctypeslib.as_array(ptrs[0], (n + 1,)).copy()
        Up = np.ctypeslib.as_array(ptrs[3], (n + 1,)).copy()
        L = Csr(n, n, Lp, np.ctypeslib.as_array(ptrs[1], (Lp[n],)).copy(),
                np.ctypeslib.as_array(ptrs[2], (Lp[n],)).copy())
        U = Csr(n, n, Up, np.ctypeslib.as_array(ptrs[4], (Up[n],)).copy(),
                np.ctypeslib.as_array(ptrs[5], (Up[n],)).copy())
        rperm = np.ctypeslib.as_array(ptrs[6], (n,)).copy()
        cperm = np.ctypeslib.as_array(ptrs[7], (n,)).copy()
        o, nu = C.c_double(), C.c_double()
        F.lib.exg_factor_timing(h, C.byref(o), C.byref(nu))
        return Factorization(n, L, U, rperm, cperm, o.value, nu.value)
    finally:
        F.lib.exg_factor_free(h)


def write_waveform_csv(path, times, samples, columns, threads: int = 0) -> None:
    """The reference CLI's waveform CSV (write_waveform_csv, proj/tools/common.hpp:35-46), byte for
    byte, formatted by several host threads.  samples: n_times x n_cols."""
    times = F.f64(times)
    samples = np.ascontiguousarray(np.asarray(samples, dtype=np.float64).reshape(len(times), len(columns)))
    names = (C.c_char_p * max(len(columns), 1))(*[c.encode() for c in columns])
    rc = F.lib.exg_write_waveform_csv(str(path).encode(), len(times), len(columns), F.as_ptr(times, C.c_double),
                                      F.as_ptr(samples, C.c_double), names, threads)
    if rc != F.EXG_OK:
        raise_for(rc, F.lib.exg_host_error_message().decode())
