"""Shared test helpers: systems on both sides, factor conversion, comparisons."""
import numpy as np

import paper_1511_04515_b200 as ex


def bits(a):
    a = np.ascontiguousarray(a, dtype=np.float64)
    # +0.0 and -0.0 compare equal in the reference's (value) semantics
    a = np.where(a == 0.0, 0.0, a)
    return a.view(np.int64)


def bit_equal(a, b):
    return a.shape == b.shape and np.array_equal(bits(a), bits(b))


def ref_system(ref, s):
    """The reference's own MnaSystem for a generated system."""
    el, src, pt, pv, mo = s.elements()
    if len(el):
        return ref.system_from_elements(el, src, pt, pv, mo, s.options())
    return ref.system_from_csr(s.n, s.G, s.C, s.B, src, pt, pv, s.options())


def full_scale_err(a, b):
    """max over nodes of max_t |a-b| / max_t |b| (the parity metric)."""
    scale = np.maximum(np.abs(b).max(axis=0), 1e-300)
    return float((np.abs(a - b).max(axis=0) / scale).max())


def random_rc_pair(n, seed):
    """Sparse SPD-dominant tridiagonal pair like test_krylov.cpp:37-56
    (numpy RNG; values differ from the reference test's, structure is the same)."""
    rng = np.random.default_rng(seed)
    Cd = np.zeros((n, n))
    Gd = np.zeros((n, n))
    for i in range(n):
        Cd[i, i] = rng.uniform(0.5, 2.0)
        Gd[i, i] = 2.0 + rng.uniform(0.5, 2.0)
        if i + 1 < n:
            gc = -0.5 * rng.uniform()
            Gd[i, i + 1] = Gd[i + 1, i] = gc
            cc = 0.2 * rng.uniform()
            Cd[i, i + 1] = Cd[i + 1, i] = cc
    return dense_to_csr(Cd), dense_to_csr(Gd)


def dense_to_csr(D):
    n_rows, n_cols = D.shape
    rowptr = [0]
    col, val = [], []
    for r in range(n_rows):
        nz = np.nonzero(D[r])[0]
        col += nz.tolist()
        val += D[r, nz].tolist()
        rowptr.append(len(col))
    return ex.Csr(n_rows, n_cols, np.array(rowptr, np.int32), np.array(col, np.int32), np.array(val))
