"""ORACLE / TEST INFRASTRUCTURE — build the reference's MnaSystem for a generated system.

Small systems go through the reference's own build_mna (element list);
large ones (config 1 at 1M nodes) are handed over as CSR (C, G, B) plus the
per-column source list — tests/test_host.py proves the two assemblies are
bit-identical on the cuts.
"""
import numpy as np

import paper_1511_04515_b200 as ex
from paper_1511_04515_b200 import _ffi as F


def column_sources(s):
    """One exg_source per B column, in build_mna's card order (mna.cpp:102-114)."""
    el, src, pt, pv, mo = s.elements()
    if not len(el):
        return src, pt, pv
    arr = np.ctypeslib.as_array(el)
    kinds = arr["kind"]
    aux = arr["aux"][(kinds == F.EXG_EL_V) | (kinds == F.EXG_EL_I)]
    cols = (F.exg_source * max(len(aux), 1))(*[src[int(a)] for a in aux])
    return cols, pt, pv


def ref_system_for(ref, s, max_elements_n=300_000):
    if s.n <= max_elements_n:
        el, src, pt, pv, mo = s.elements()
        if len(el):
            return ref.system_from_elements(el, src, pt, pv, mo, s.options())
    cols, pt, pv = column_sources(s)
    return ref.system_from_csr(s.n, s.G, s.C, s.B, cols, pt, pv, s.options())
