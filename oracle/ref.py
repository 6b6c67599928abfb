"""ORACLE / TEST INFRASTRUCTURE — ctypes access to the reference and the C restatement.

* ``Ref`` wraps ``oracle/_ref/libexsim_ref.so``: the unmodified reference
  core (proj/core/src) + ``ref_shim.cpp``.
* ``Orc`` wraps ``oracle/_build/liboracle.so``: the plain-C restatement.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU legs import this.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REF_LIB = HERE / "_ref" / "libexsim_ref.so"
ORC_LIB = HERE / "_build" / "liboracle.so"

P, I, D = C.c_void_p, C.c_int, C.c_double
PI, PD = C.POINTER(C.c_int), C.POINTER(C.c_double)


def _ptr(a, t):
    return a.ctypes.data_as(C.POINTER(t))


def _i(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def _d(a):
    return np.ascontiguousarray(a, dtype=np.float64)


class RefError(RuntimeError):
    def __init__(self, status, msg, value):
        super().__init__(f"reference status {status}: {msg}")
        self.status = status
        self.value = value


class Ref:
    """The reference library (exsim_core) through ref_shim.cpp."""

    def __init__(self, path: Path = REF_LIB):
        if not path.exists():
            raise FileNotFoundError(f"{path} missing: run `make -C oracle` where /root/reference exists")
        self.lib = L = C.CDLL(str(path))
        L.ref_last_error.restype = C.c_char_p
        L.ref_last_error.argtypes = [PD]
        L.ref_system_free.argtypes = [P]
        L.ref_system_n.argtypes = [P]
        L.ref_system_n_inputs.argtypes = [P]
        L.ref_factor_free.argtypes = [P]
        L.ref_basis_free.argtypes = [P]
        L.ref_tran_free.argtypes = [P]
        L.ref_system_unknown_of_label.argtypes = [P, I]
        L.ref_lu_count.restype = C.c_ulonglong

    def _check(self, st):
        if st != 0:
            v = C.c_double()
            msg = self.lib.ref_last_error(C.byref(v)).decode()
            raise RefError(st, msg, v.value)

    # ---- systems
    def system_from_elements(self, elems, srcs, pwl_t, pwl_v, models, opts):
        h = C.c_void_p()
        pt, pv = _d(pwl_t), _d(pwl_v)
        self._check(self.lib.ref_system_from_elements(
            len(elems), elems, len(srcs), srcs, _ptr(pt, C.c_double), _ptr(pv, C.c_double),
            models, C.byref(opts), C.byref(h)))
        return h

    def system_from_csr(self, n, G, Cm, B, srcs, pwl_t, pwl_v, opts):
        h = C.c_void_p()
        pt, pv = _d(pwl_t), _d(pwl_v)
        args = []
        for m in (G, Cm):
            args += [_ptr(_i(m.rowptr), C.c_int), _ptr(_i(m.col), C.c_int), _ptr(_d(m.val), C.c_double), m.nnz]
        keep = [_i(B.rowptr), _i(B.col), _d(B.val)]
        self._check(self.lib.ref_system_from_csr(
            n, *args, B.n_cols, _ptr(keep[0], C.c_int), _ptr(keep[1], C.c_int),
            _ptr(keep[2], C.c_double), B.nnz, srcs, _ptr(pt, C.c_double), _ptr(pv, C.c_double),
            C.byref(opts), C.byref(h)))
        return h

    def system_free(self, h):
        self.lib.ref_system_free(h)

    def system_csr(self, h, which):
        nnz, nc = C.c_int(), C.c_int()
        self.lib.ref_system_csr(h, which, C.byref(nnz), C.byref(nc), None, None, None)
        n = self.lib.ref_system_n(h)
        rp = np.zeros(n + 1, np.int32)
        ci = np.zeros(max(nnz.value, 1), np.int32)
        va = np.zeros(max(nnz.value, 1))
        self.lib.ref_system_csr(h, which, C.byref(nnz), C.byref(nc), _ptr(rp, C.c_int),
                                _ptr(ci, C.c_int), _ptr(va, C.c_double))
        return n, nc.value, rp, ci[: nnz.value], va[: nnz.value]

    def unknown_of_label(self, h, label):
        return self.lib.ref_system_unknown_of_label(h, label)

    def eval_sources(self, h, t):
        u = np.zeros(self.lib.ref_system_n_inputs(h))
        self._check(self.lib.ref_eval_sources(h, D(t), _ptr(u, C.c_double)))
        return u

    def dc_solve(self, h):
        x = np.zeros(self.lib.ref_system_n(h))
        self._check(self.lib.ref_dc_solve(h, _ptr(x, C.c_double)))
        return x

    def evaluate(self, h, x, n_mos):
        """exsim::evaluate -> (C_k, G_k) as (rowptr, col, val) and op[n_mos, 5]."""
        n = self.lib.ref_system_n(h)
        x = _d(x)
        out = []
        op = np.zeros((n_mos, 5))
        for which in (0, 1):
            nnz = C.c_int()
            self._check(self.lib.ref_evaluate(h, _ptr(x, C.c_double), which, C.byref(nnz),
                                              None, None, None, None))
            rp, ci, va = np.zeros(n + 1, np.int32), np.zeros(nnz.value, np.int32), np.zeros(nnz.value)
            self._check(self.lib.ref_evaluate(h, _ptr(x, C.c_double), which, C.byref(nnz),
                                              _ptr(rp, C.c_int), _ptr(ci, C.c_int),
                                              _ptr(va, C.c_double), _ptr(op, C.c_double)))
            out.append((rp, ci, va))
        return out[0], out[1], op

    def residual_F(self, h, x_ref, x):
        n = self.lib.ref_system_n(h)
        F_ = np.zeros(n)
        self._check(self.lib.ref_residual_F(h, _ptr(_d(x_ref), C.c_double), _ptr(_d(x), C.c_double),
                                            _ptr(F_, C.c_double)))
        return F_

    # ---- LU
    def lu_factor(self, A, pivot_tol=0.1):
        h = C.c_void_p()
        rp, ci, va = _i(A.rowptr), _i(A.col), _d(A.val)
        self._check(self.lib.ref_lu_factor(A.n_rows, _ptr(rp, C.c_int), _ptr(ci, C.c_int),
                                           _ptr(va, C.c_double), A.nnz, D(pivot_tol), C.byref(h)))
        return h

    def factor_from(self, f):
        h = C.c_void_p()
        arrs = [_i(f.L.rowptr), _i(f.L.col), _d(f.L.val), _i(f.U.rowptr), _i(f.U.col),
                _d(f.U.val), _i(f.row_perm), _i(f.col_perm)]
        types = [C.c_int, C.c_int, C.c_double, C.c_int, C.c_int, C.c_double, C.c_int, C.c_int]
        self._check(self.lib.ref_factor_from_arrays(f.n, *[_ptr(a, t) for a, t in zip(arrs, types)],
                                                    C.byref(h)))
        return h

    def factor_free(self, h):
        self.lib.ref_factor_free(h)

    def factor_export(self, h):
        nl, nu = C.c_int(), C.c_int()
        n = self.lib.ref_factor_nnz(h, C.byref(nl), C.byref(nu))
        out = dict(Lp=np.zeros(n + 1, np.int32), Li=np.zeros(nl.value, np.int32),
                   Lx=np.zeros(nl.value), Up=np.zeros(n + 1, np.int32),
                   Ui=np.zeros(nu.value, np.int32), Ux=np.zeros(nu.value),
                   row_perm=np.zeros(n, np.int32), col_perm=np.zeros(n, np.int32))
        ts = [C.c_int, C.c_int, C.c_double, C.c_int, C.c_int, C.c_double, C.c_int, C.c_int]
        self.lib.ref_factor_export(h, *[_ptr(a, t) for a, t in zip(out.values(), ts)])
        out["n"] = n
        return out

    def solve(self, fh, b):
        b = _d(b)
        x = np.zeros_like(b)
        self._check(self.lib.ref_solve(fh, _ptr(b, C.c_double), _ptr(x, C.c_double)))
        return x

    def apply(self, fh, x):
        x = _d(x)
        y = np.zeros_like(x)
        self._check(self.lib.ref_apply(fh, _ptr(x, C.c_double), _ptr(y, C.c_double)))
        return y

    def spmv(self, A, x):
        x = _d(x)
        y = np.zeros(A.n_rows)
        rp, ci, va = _i(A.rowptr), _i(A.col), _d(A.val)
        self._check(self.lib.ref_spmv(A.n_rows, A.n_cols, A.nnz, _ptr(rp, C.c_int), _ptr(ci, C.c_int),
                                      _ptr(va, C.c_double), _ptr(x, C.c_double), _ptr(y, C.c_double)))
        return y

    def mevp_iks(self, fh, Cm, v, h, eps=1e-7, m_max=100, keep_basis=False):
        v = _d(v)
        out = np.zeros_like(v)
        m, happy = C.c_int(), C.c_int()
        beta, hn = C.c_double(), C.c_double()
        bh = C.c_void_p()
        rp, ci, va = _i(Cm.rowptr), _i(Cm.col), _d(Cm.val)
        self._check(self.lib.ref_mevp_iks(
            fh, Cm.n_rows, Cm.nnz, _ptr(rp, C.c_int), _ptr(ci, C.c_int), _ptr(va, C.c_double),
            _ptr(v, C.c_double), D(h), D(eps), m_max, _ptr(out, C.c_double), C.byref(m),
            C.byref(happy), C.byref(beta), C.byref(hn), C.byref(bh) if keep_basis else None))
        info = dict(m=m.value, happy=happy.value, beta=beta.value, h_next=hn.value)
        if keep_basis:
            info["basis"] = bh
        return out, info

    def basis_residual(self, bh, G, h):
        r = C.c_double()
        rp, ci, va = _i(G.rowptr), _i(G.col), _d(G.val)
        self._check(self.lib.ref_basis_residual(bh, G.n_rows, G.nnz, _ptr(rp, C.c_int),
                                                _ptr(ci, C.c_int), _ptr(va, C.c_double), D(h),
                                                C.byref(r)))
        return r.value

    def basis_eval(self, bh, h, n):
        out = np.zeros(n)
        self._check(self.lib.ref_basis_eval(bh, D(h), _ptr(out, C.c_double)))
        return out

    def basis_free(self, bh):
        self.lib.ref_basis_free(bh)

    def write_waveform_csv(self, path, times, samples, columns):
        """The reference CLI's writer (proj/tools/common.hpp:35-46), unmodified."""
        times, samples = _d(times), _d(samples)
        names = (C.c_char_p * len(columns))(*[c.encode() for c in columns])
        self.lib.ref_write_waveform_csv.argtypes = [C.c_char_p, C.c_int, C.c_int, C.POINTER(C.c_double),
                                                    C.POINTER(C.c_double), C.POINTER(C.c_char_p)]
        self._check(self.lib.ref_write_waveform_csv(str(path).encode(), len(times), len(columns),
                                                    _ptr(times, C.c_double), _ptr(samples, C.c_double), names))

    def dense_expm(self, a):
        a = _d(a)
        n = a.shape[0]
        out = np.zeros_like(a)
        self._check(self.lib.ref_dense_expm(n, _ptr(a, C.c_double), _ptr(out, C.c_double)))
        return out

    def dense_inverse(self, a):
        a = _d(a)
        out = np.zeros_like(a)
        cond = C.c_double()
        self._check(self.lib.ref_dense_inverse(a.shape[0], _ptr(a, C.c_double),
                                               _ptr(out, C.c_double), C.byref(cond)))
        return out, cond.value

    # ---- transient
    def _tran(self, rh):
        nt, nr, ns, nd = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        self.lib.ref_tran_sizes(rh, C.byref(nt), C.byref(nr), C.byref(ns), C.byref(nd))
        r = dict(times=np.zeros(nt.value), samples=np.zeros(nt.value * nr.value),
                 t=np.zeros(ns.value), h=np.zeros(ns.value), lu=np.zeros(ns.value, np.int32),
                 rejects=np.zeros(ns.value, np.int32), err=np.zeros(ns.value),
                 dims_off=np.zeros(ns.value + 1, np.int32), dims=np.zeros(max(nd.value, 1), np.int32))
        ts = [C.c_double, C.c_double, C.c_double, C.c_double, C.c_int, C.c_int, C.c_double,
              C.c_int, C.c_int]
        self.lib.ref_tran_get(rh, *[_ptr(a, t) for a, t in zip(r.values(), ts)])
        nw = self.lib.ref_tran_wall(rh, None)
        r["wall"] = np.zeros(nw)
        if nw:
            self.lib.ref_tran_wall(rh, _ptr(r["wall"], C.c_double))
        r["dims"] = r["dims"][: nd.value]
        r["samples"] = r["samples"].reshape(nt.value, nr.value)
        self.lib.ref_tran_free(rh)
        return r

    def transient(self, sh, ctl, t_stop, rec_idx, method=1):
        rh = C.c_void_p()
        ri = _i(rec_idx)
        self._check(self.lib.ref_transient(sh, method, C.byref(ctl), D(t_stop), _ptr(ri, C.c_int),
                                           ri.size, C.byref(rh)))
        return self._tran(rh)

    def transient_cached(self, sh, fh, ctl, t_stop, rec_idx, method=1, max_steps=0, x0=None):
        rh = C.c_void_p()
        ri = _i(rec_idx)
        xp = None if x0 is None else _ptr(_d(x0), C.c_double)
        self._check(self.lib.ref_transient_cached(sh, fh, method, C.byref(ctl), D(t_stop),
                                                  _ptr(ri, C.c_int), ri.size,
                                                  C.c_long(max_steps), xp, C.byref(rh)))
        return self._tran(rh)

    def transient_policy(self, sh, ctl, t_stop, rec_idx, method=1, threshold=0.1, max_steps=0):
        """Restated loop with the refactor policy of exg_step_control.refactor_threshold:
        the Linearization and lu_factor(G_k) are renewed only when a device conductance
        moved by more than `threshold` (0: every step, bit-identical to transient())."""
        import copy
        c2 = copy.copy(ctl)
        c2.refactor_threshold = threshold
        return self.transient_cached(sh, None, c2, t_stop, rec_idx, method=method, max_steps=max_steps)


class Orc:
    """The plain-C restatement (oracle/exsim_oracle.c)."""

    class Csr(C.Structure):
        _fields_ = [("n_rows", C.c_int), ("n_cols", C.c_int), ("rowptr", PI), ("col", PI),
                    ("val", PD)]

    class Factor(C.Structure):
        pass

    class Cfg(C.Structure):
        _fields_ = [("eps", C.c_double), ("m_max", C.c_int), ("check_stride", C.c_int),
                    ("breakdown_tol", C.c_double)]

    class Basis(C.Structure):
        _fields_ = [("n", C.c_int), ("m", C.c_int), ("happy", C.c_int), ("m_max", C.c_int),
                    ("beta", C.c_double), ("h_next", C.c_double), ("h_sub", C.c_double),
                    ("last_residual", C.c_double), ("V", PD), ("hbar", PD), ("h_inv", PD),
                    ("work", PD)]

    Factor._fields_ = [("n", C.c_int), ("L", Csr), ("U", Csr), ("row_perm", PI), ("col_perm", PI)]

    def __init__(self, path: Path = ORC_LIB):
        if not path.exists():
            raise FileNotFoundError(f"{path} missing: run `make -C oracle oracle`")
        self.lib = C.CDLL(str(path))
        self._keep = []

    def csr(self, A):
        rp, ci, va = _i(A.rowptr), _i(A.col), _d(A.val)
        self._keep += [rp, ci, va]
        return Orc.Csr(A.n_rows, A.n_cols, _ptr(rp, C.c_int), _ptr(ci, C.c_int), _ptr(va, C.c_double))

    def factor(self, f):
        rperm, cperm = _i(f.row_perm), _i(f.col_perm)
        self._keep += [rperm, cperm]
        return Orc.Factor(f.n, self.csr(f.L), self.csr(f.U), _ptr(rperm, C.c_int),
                          _ptr(cperm, C.c_int))

    def spmv(self, A, x):
        x = _d(x)
        y = np.zeros(A.n_rows)
        self.lib.orc_spmv(C.byref(self.csr(A)), _ptr(x, C.c_double), _ptr(y, C.c_double))
        return y

    def solve(self, f, b):
        b = _d(b)
        x = np.zeros_like(b)
        w = np.zeros_like(b)
        self.lib.orc_solve(C.byref(self.factor(f)), _ptr(b, C.c_double), _ptr(x, C.c_double),
                           _ptr(w, C.c_double))
        return x

    def apply(self, f, x):
        x = _d(x)
        y = np.zeros_like(x)
        w = np.zeros(3 * x.size)
        self.lib.orc_apply(C.byref(self.factor(f)), _ptr(x, C.c_double), _ptr(y, C.c_double),
                           _ptr(w, C.c_double))
        return y

    def dense_expm(self, a):
        a = _d(a)
        out = np.zeros_like(a)
        st = self.lib.orc_dense_expm(a.shape[0], _ptr(a, C.c_double), _ptr(out, C.c_double), None)
        if st:
            raise RuntimeError(f"orc_dense_expm status {st}")
        return out

    def _basis(self, n, m_max):
        V = np.zeros(n * (m_max + 1))
        hb = np.zeros((m_max + 1) * (m_max + 2))
        hi = np.zeros(m_max * m_max)
        self._keep += [V, hb, hi]
        b = Orc.Basis()
        b.V, b.hbar, b.h_inv = _ptr(V, C.c_double), _ptr(hb, C.c_double), _ptr(hi, C.c_double)
        return b, V

    def mevp_iks(self, f, Cm, v, h, eps=1e-7, m_max=100):
        v = _d(v)
        out = np.zeros_like(v)
        b, V = self._basis(v.size, m_max)
        cfg = Orc.Cfg(eps, m_max, 1, 1e-12)
        st = self.lib.orc_mevp_iks(C.byref(self.factor(f)), C.byref(self.csr(Cm)),
                                   _ptr(v, C.c_double), C.byref(cfg), D(h), _ptr(out, C.c_double),
                                   C.byref(b))
        if st:
            raise RuntimeError(f"orc_mevp_iks status {st}")
        return out, dict(m=b.m, happy=b.happy, beta=b.beta, h_next=b.h_next,
                         last_residual=b.last_residual, V=V.reshape(m_max + 1, v.size))

    def er_step(self, f, Cm, Bm, x_k, u_k, u_k1, h, eps=1e-7, m_max=100):
        x_k, u_k, u_k1 = _d(x_k), _d(u_k), _d(u_k1)
        xn = np.zeros_like(x_k)
        m = C.c_int()
        b, _ = self._basis(x_k.size, m_max)
        cfg = Orc.Cfg(eps, m_max, 1, 1e-12)
        st = self.lib.orc_er_step(C.byref(self.factor(f)), C.byref(self.csr(Cm)),
                                  C.byref(self.csr(Bm)), _ptr(x_k, C.c_double),
                                  _ptr(u_k, C.c_double), _ptr(u_k1, C.c_double), D(h),
                                  C.byref(cfg), _ptr(xn, C.c_double), C.byref(m), C.byref(b))
        if st:
            raise RuntimeError(f"orc_er_step status {st}")
        self._keep.clear()
        return xn, m.value
