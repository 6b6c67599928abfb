"""CPU tests of the host mirror (generators, MNA, setup LU) and the C ABI surface."""
import ctypes as C
import re
from pathlib import Path

import numpy as np
import pytest

import paper_1511_04515_b200 as ex
from paper_1511_04515_b200 import _ffi as F

from helpers import bit_equal, ref_system

ROOT = Path(__file__).resolve().parents[1]


def test_library_exports_every_declared_symbol():
    """include/*.h declarations == exported symbols of the in-tree libexg.so."""
    declared = set()
    for h in (ROOT / "include").glob("*.h"):
        declared |= set(re.findall(r"^\s*(?:[\w\*]+\s+)+\**(exg_\w+)\s*\(", h.read_text(), re.M))
    assert declared, "no declarations parsed"
    lib = C.CDLL(str(F.LIB_PATH))
    missing = [s for s in sorted(declared) if not hasattr(lib, s)]
    assert not missing, missing
    assert set(F.declared_symbols()) <= declared | {"exg_host_error_message"}


@pytest.mark.parametrize("cfg,kw", [(0, {}), (1, dict(width=64)), (2, dict(width=12)),
                                    (4, dict(width=12, chains=4, stages=4))])
def test_mna_identical_to_reference_build_mna(ref, cfg, kw):
    s = ex.System.generate(cfg, **kw)
    rh = ref_system(ref, s)
    try:
        for w in (F.EXG_MAT_C, F.EXG_MAT_G, F.EXG_MAT_B):
            n, nc, rp, ci, va = ref.system_csr(rh, w)
            m = s.csr(w)
            assert (n, nc) == (m.n_rows, m.n_cols)
            assert np.array_equal(rp, m.rowptr) and np.array_equal(ci, m.col)
            assert bit_equal(va, m.val)
        for t in (0.0, 3e-12, 17.5e-12, 1.05e-10, 9.99e-10):
            assert bit_equal(s.eval_sources(t), ref.eval_sources(rh, t))
    finally:
        ref.system_free(rh)


@pytest.mark.parametrize("cfg,kw", [(0, {}), (1, dict(width=100)), (2, dict(width=16)),
                                    (3, dict(n=2000)), (4, dict(width=10, chains=4, stages=4))])
def test_lu_bit_identical_to_reference(ref, cfg, kw):
    s = ex.System.generate(cfg, **kw)
    f = ex.lu_factor(s.G)
    fh = ref.lu_factor(s.G)
    try:
        e = ref.factor_export(fh)
    finally:
        ref.factor_free(fh)
    assert np.array_equal(e["col_perm"], f.col_perm)
    assert np.array_equal(e["row_perm"], f.row_perm)
    assert np.array_equal(e["Lp"], f.L.rowptr) and np.array_equal(e["Li"], f.L.col)
    assert np.array_equal(e["Up"], f.U.rowptr) and np.array_equal(e["Ui"], f.U.col)
    assert bit_equal(e["Lx"], f.L.val) and bit_equal(e["Ux"], f.U.val)


def _assert_factor_equals_reference(ref, A, f):
    fh = ref.lu_factor(A)
    try:
        e = ref.factor_export(fh)
    finally:
        ref.factor_free(fh)
    assert np.array_equal(e["col_perm"], f.col_perm) and np.array_equal(e["row_perm"], f.row_perm)
    assert np.array_equal(e["Li"], f.L.col) and np.array_equal(e["Ui"], f.U.col)
    assert bit_equal(e["Lx"], f.L.val) and bit_equal(e["Ux"], f.U.val)


def test_lu_ordering_reuse_across_patterns(ref):
    """lu_factor reuses the ordering while the pattern is unchanged (a nonlinear
    transient's refactorisations): same pattern with new values, a different
    pattern in between, then the first pattern again -- all bit-identical to
    the reference's lu_factor."""
    a = ex.System.generate(4, width=10, chains=4, stages=4).G
    b = ex.System.generate(0).G
    rng = np.random.default_rng(7)
    a2 = ex.Csr(a.n_rows, a.n_cols, a.rowptr, a.col, a.val * (1.0 + 0.25 * rng.random(a.val.size)))
    for A in (a, a2, b, a, a2):
        _assert_factor_equals_reference(ref, A, ex.lu_factor(A))


def test_lu_singular_raises():
    """test_sparse.cpp:104-110."""
    A = ex.Csr(2, 2, np.array([0, 2, 4], np.int32), np.array([0, 1, 0, 1], np.int32), np.ones(4))
    with pytest.raises(ex.SingularMatrixError):
        ex.lu_factor(A)


def test_breakpoints_sorted_unique():
    s = ex.System.generate(1, width=64)
    b = s.breakpoints(0.0, 2e-9)
    assert np.all(np.diff(b) > 0) and b.min() > 0 and b.max() < 2e-9


def test_generators_deterministic():
    a, b = ex.System.generate(1, width=40), ex.System.generate(1, width=40)
    assert bit_equal(a.C.val, b.C.val) and np.array_equal(a.G.col, b.G.col)


@pytest.mark.parametrize("kw", [dict(width=12, chains=4, stages=4), dict(width=20, chains=16, stages=8)],
                         ids=["12x12-4x4", "20x20-16x8"])
def test_nonlinear_host_mirror_bit_identical(ref, kw):
    """dc_solve (integrate.cpp:92-115), evaluate (devices.cpp:122-200) and
    residual_F (devices.cpp:202-233) of the host mirror against exsim."""
    s = ex.System.generate(4, **kw)
    rh = ref_system(ref, s)
    try:
        x = s.dc_solve()
        assert np.array_equal(x, ref.dc_solve(rh))
        Cr, Gr, opr = ref.evaluate(rh, x, s.n_mos)
        Ck, Gk, op = s.linearize(x)
        for mine, theirs in ((Ck, Cr), (Gk, Gr)):
            assert np.array_equal(mine.rowptr, theirs[0])
            assert np.array_equal(mine.col, theirs[1])
            assert np.array_equal(mine.val, theirs[2])
        assert np.array_equal(op, opr)
        x2 = x + np.random.default_rng(3).normal(0.0, 0.05, s.n)
        assert np.array_equal(s.residual_F(x, x2), ref.residual_F(rh, x, x2))
    finally:
        ref.system_free(rh)


# ---- waveform CSV: the reference CLI's writer, byte for byte --------------------
@pytest.mark.parametrize("n_times,n_cols,threads", [(0, 3, 0), (1, 0, 1), (7, 1, 3), (4001, 16, 0), (20000, 5, 8)])
def test_waveform_csv_matches_reference_writer(ref, tmp_path, n_times, n_cols, threads):
    """exg_write_waveform_csv against write_waveform_csv of proj/tools/common.hpp:35-46 (unmodified,
    through oracle/_ref): identical bytes, whatever the thread count; values include zeros of both
    signs, denormals, huge and non-finite numbers (the reference prints them with %.17g too)."""
    from paper_1511_04515_b200.host import write_waveform_csv
    rng = np.random.default_rng(n_times + n_cols)
    times = np.cumsum(rng.uniform(1e-13, 2e-11, n_times))
    samples = rng.normal(0.0, 1.0, (n_times, n_cols)) * 10.0 ** rng.integers(-12, 3, (n_times, n_cols))
    if samples.size >= 8:
        samples.flat[:8] = [0.0, -0.0, 5e-324, -2.2250738585072014e-308, 1.7976931348623157e308, np.inf, -np.inf, np.nan]
    cols = [f"v(n{c}_{c * 7})" for c in range(n_cols)]
    a, b = tmp_path / "ours.csv", tmp_path / "ref.csv"
    write_waveform_csv(a, times, samples, cols, threads)
    ref.write_waveform_csv(b, times, samples.reshape(n_times, n_cols), cols)
    assert a.read_bytes() == b.read_bytes()


def test_waveform_csv_unwritable_path_is_a_contract_error(tmp_path):
    from paper_1511_04515_b200.host import write_waveform_csv
    with pytest.raises(ex.ContractError):
        write_waveform_csv(tmp_path / "no_such_dir" / "w.csv", [0.0], [[1.0]], ["a"])
