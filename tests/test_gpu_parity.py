"""GPU parity tests: every kernel through the C ABI against the reference
library (oracle/_ref) and the C restatement, on the same seeded inputs.

Bars:
* SpMV, factor apply, EXACT triangular solves: bit-identical (row-sequential
  accumulation in the reference's order, no FMA contraction).
* FAST triangular solves: <= 1e-13 relative (reordered U sums).
* MEVP: identical Krylov dimension, value within 1e-12 relative (only the
  dot-product summation order differs).
* Transient: identical step times and per-step Krylov dimensions, waveforms
  within 1e-8 of each node's full scale (north_star tolerance).
"""
import ctypes as C

import numpy as np
import pytest

import paper_1511_04515_b200 as ex
from paper_1511_04515_b200 import _ffi as F
from paper_1511_04515_b200.device import Context

from helpers import bit_equal, full_scale_err, random_rc_pair, ref_system

pytestmark = pytest.mark.gpu

CASES = [
    (0, {}),                        # config 0: 32x32 RC grid
    (1, dict(width=64)),            # config 1 cut: 64x64 power grid, VDD pads
    (2, dict(width=12)),            # config 2 cut: RLC with branch currents
    (3, dict(n=3000)),              # config 3 cut: banded post-extraction system
]


@pytest.fixture(scope="module", params=CASES, ids=lambda c: f"c{c[0]}")
def case(request, ref):
    cfg, kw = request.param
    s = ex.System.generate(cfg, **kw)
    f = ex.lu_factor(s.G)
    fh = ref.factor_from(f)
    yield cfg, s, f, fh
    ref.factor_free(fh)


def _ctx(s, f, mode=F.EXG_TRSV_EXACT):
    c = Context(0, trsv_mode=mode)
    c.set_system(s)
    c.set_factors(f)
    return c


def test_spmv_bit_identical(case, ref):
    _, s, f, _ = case
    rng = np.random.default_rng(1)
    with _ctx(s, f) as c:
        for w, A in ((F.EXG_MAT_C, s.C), (F.EXG_MAT_G, s.G), (F.EXG_MAT_B, s.B)):
            x = rng.uniform(-1, 1, A.n_cols)
            assert bit_equal(c.spmv(w, x, A.n_rows), ref.spmv(A, x))


def test_solve_exact_bit_identical(case, ref, orc):
    _, s, f, fh = case
    rng = np.random.default_rng(2)
    with _ctx(s, f) as c:
        for _ in range(3):
            b = rng.uniform(-1, 1, s.n)
            got = c.solve(b)
            assert bit_equal(got, ref.solve(fh, b))
            assert bit_equal(got, orc.solve(f, b))
        cn = c.counters()
        assert cn.l_levels > 0 and cn.u_levels > 0


def test_solve_fast_close(case, ref):
    _, s, f, fh = case
    b = np.random.default_rng(3).uniform(-1, 1, s.n)
    with _ctx(s, f, F.EXG_TRSV_FAST) as c:
        got = c.solve(b)
    want = ref.solve(fh, b)
    assert np.max(np.abs(got - want)) <= 1e-13 * np.max(np.abs(want))


@pytest.mark.parametrize("budget", [0, 16, 256, 4096])
@pytest.mark.parametrize("cfg,kw", [(1, dict(width=64)), (1, dict(width=160)), (2, dict(width=24)),
                                    (3, dict(n=3000))], ids=["c1-64", "c1-160", "c2-24", "c3-3000"])
def test_solve_fast_subtree_budgets(ref, monkeypatch, cfg, kw, budget):
    """FAST plan with the subtree phase of k_trsv_sub at several component
    budgets (EXG_SUB_ROWS; 0 disables it): the mixed plans (components +
    wide runs + chain) stay within the FAST bar, in both triangles."""
    monkeypatch.setenv("EXG_SUB_ROWS", str(budget))
    s = ex.System.generate(cfg, **kw)
    f = ex.lu_factor(s.G)
    fh = ref.factor_from(f)
    try:
        rng = np.random.default_rng(11)
        with _ctx(s, f, F.EXG_TRSV_FAST) as c:
            for _ in range(2):
                b = rng.uniform(-1, 1, s.n)
                got = c.solve(b)
                want = ref.solve(fh, b)
                assert np.max(np.abs(got - want)) <= 1e-13 * np.max(np.abs(want))
    finally:
        ref.factor_free(fh)


def test_apply_bit_identical(case, ref):
    _, s, f, fh = case
    x = np.random.default_rng(4).uniform(-1, 1, s.n)
    with _ctx(s, f) as c:
        assert bit_equal(c.apply(x), ref.apply(fh, x))


def test_solve_residual_contract(case):
    """test_sparse.cpp:112-131: ||A x - b||_inf <= 1e-10 (1 + ||b||_inf)."""
    _, s, f, _ = case
    b = np.random.default_rng(5).uniform(-1, 1, s.n)
    with _ctx(s, f) as c:
        x = c.solve(b)
        r = c.spmv(F.EXG_MAT_G, x, s.n) - b
    assert np.max(np.abs(r)) <= 1e-10 * (1 + np.max(np.abs(b)))


def test_mevp_matches_reference(case, ref):
    cfg, s, f, fh = case
    rng = np.random.default_rng(6)
    v = rng.uniform(-1, 1, s.n)
    opts = s.options()
    h = 1e-12 if cfg != 3 else 1e-12
    from ref import RefError
    with _ctx(s, f) as c:
        for eps in (1e-7, 1e-10):
            try:
                want, winfo = ref.mevp_iks(fh, s.C, v, h, eps=eps, m_max=opts.m_max)
            except RefError as e:
                # the reference fails on this input: the device must fail the same way
                with pytest.raises(ex.Error) as ei:
                    c.mevp_iks(v, h, eps=eps, m_max=opts.m_max)
                assert {5: ex.NoConvergenceError, 2: ex.NonFiniteError,
                        3: ex.SingularMatrixError}[e.status] is type(ei.value)
                continue
            got, info = c.mevp_iks(v, h, eps=eps, m_max=opts.m_max)
            assert info.m == winfo["m"]
            assert info.happy == bool(winfo["happy"])
            assert np.max(np.abs(got - want)) <= 1e-12 * np.max(np.abs(want))


def test_mevp_cached_basis(case, ref):
    cfg, s, f, fh = case
    if cfg == 2:
        pytest.skip("random start vectors do not converge on the RLC cut (the reference fails too)")
    v = np.random.default_rng(7).uniform(-1, 1, s.n)
    h = 2e-12
    with _ctx(s, f) as c:
        got, info = c.mevp_iks(v, h, eps=1e-9, m_max=60)
        want, winfo = ref.mevp_iks(fh, s.C, v, h, eps=1e-9, m_max=60, keep_basis=True)
        bh = winfo["basis"]
        try:
            for fr in (1.0, 0.75, 0.5):
                r_got = c.mevp_residual(fr * h)
                r_want = ref.basis_residual(bh, s.G, fr * h)
                assert abs(r_got - r_want) <= 1e-9 * abs(r_want) + 1e-300
                e_got = c.eval_at_scaled_h(fr * h)
                e_want = ref.basis_eval(bh, fr * h, s.n)
                assert np.max(np.abs(e_got - e_want)) <= 1e-12 * np.max(np.abs(e_want))
        finally:
            ref.basis_free(bh)


def test_er_step_matches_oracle(case, ref, orc):
    cfg, s, f, fh = case
    opts = s.options()
    x0 = ref_dc = None
    rh = ref_system(ref, s)
    try:
        x0 = ref.dc_solve(rh)
        u0 = s.eval_sources(0.0)
        h = 1e-12
        u1 = s.eval_sources(h)
        with _ctx(s, f) as c:
            got, m = c.er_step(x0, u0, u1, h, eps=opts.krylov_eps, m_max=opts.m_max)
        want, m_want = orc.er_step(f, s.C, s.B, x0, u0, u1, h, eps=opts.krylov_eps, m_max=opts.m_max)
        assert m == m_want
        scale = max(np.max(np.abs(want)), 1e-300)
        assert np.max(np.abs(got - want)) <= 1e-12 * scale
    finally:
        ref.system_free(rh)


# ---- reference-test known answers, on the device ----------------------------

def test_happy_breakdown_known_answer():
    """test_krylov.cpp:65-78: C = I, G = diag(1,2,3), v = e1 -> m = 1, e^{-h}."""
    Cm = ex.Csr(3, 3, np.array([0, 1, 2, 3], np.int32), np.array([0, 1, 2], np.int32), np.ones(3))
    G = ex.Csr(3, 3, np.array([0, 1, 2, 3], np.int32), np.array([0, 1, 2], np.int32),
               np.array([1.0, 2.0, 3.0]))
    f = ex.lu_factor(G)
    with Context(0) as c:
        c.set_csr(F.EXG_MAT_C, Cm)
        c.set_csr(F.EXG_MAT_G, G)
        c.set_factors(f)
        out, info = c.mevp_iks(np.array([1.0, 0, 0]), 0.7)
        assert info.m == 1 and info.happy
        assert out[0] == pytest.approx(np.exp(-0.7), rel=1e-13)
        assert out[1] == 0.0 and out[2] == 0.0
        assert c.mevp_residual(0.7) == 0.0


def test_zero_start_and_no_convergence():
    """test_krylov.cpp:93-97 and :115-125."""
    Cm, G = random_rc_pair(30, 23)
    f = ex.lu_factor(G)
    with Context(0) as c:
        c.set_csr(F.EXG_MAT_C, Cm)
        c.set_csr(F.EXG_MAT_G, G)
        c.set_factors(f)
        with pytest.raises(ex.ZeroStartVectorError):
            c.mevp_iks(np.zeros(30), 1.0)
        v = np.random.default_rng(23).uniform(-1, 1, 30)
        with pytest.raises(ex.NoConvergenceError):
            c.mevp_iks(v, 0.05, eps=1e-14, m_max=2)


def test_mevp_dense_oracle_20():
    """test_krylov.cpp:99-113: 20x20 RC pair vs dense e^{-hC^-1G} v."""
    from scipy.linalg import expm
    Cm, G = random_rc_pair(20, 17)
    f = ex.lu_factor(G)
    v = np.random.default_rng(17).uniform(-1, 1, 20)
    with Context(0) as c:
        c.set_csr(F.EXG_MAT_C, Cm)
        c.set_csr(F.EXG_MAT_G, G)
        c.set_factors(f)
        got, info = c.mevp_iks(v, 1.0, eps=1e-7, m_max=40)
    J = -np.linalg.solve(Cm.to_dense(), G.to_dense())
    want = expm(J) @ v
    assert np.linalg.norm(got - want) <= 10 * 1e-7 * np.linalg.norm(v)


@pytest.mark.parametrize("kw", [dict(width=12, chains=4, stages=4), dict(width=20, chains=16, stages=8)],
                         ids=["12x12-4x4", "20x20-16x8"])
def test_residual_F_bit_identical(ref, kw):
    """Device MOSFET re-evaluation + per-node gather (devices.cpp:202-233)
    against exsim::residual_F: bit-identical."""
    s = ex.System.generate(4, **kw)
    rh = ref_system(ref, s)
    try:
        x_ref = ref.dc_solve(rh)
        rng = np.random.default_rng(5)
        xs = [x_ref + rng.normal(0.0, sc, s.n) for sc in (1e-3, 0.1, 0.5)]
        wants = [ref.residual_F(rh, x_ref, x) for x in xs]
    finally:
        ref.system_free(rh)
    Ck, Gk, op = s.linearize(x_ref)
    f = ex.lu_factor(Gk)
    with Context(0) as c:
        c.set_csr(F.EXG_MAT_C, Ck)
        c.set_csr(F.EXG_MAT_G, Gk)
        c.set_csr(F.EXG_MAT_B, s.B)
        c.set_factors(f)
        c.set_devices(s)
        c.set_oppoints(op)
        for x, want in zip(xs, wants):
            got = c.residual_F(x)
            assert bit_equal(got, want)
            assert np.abs(want).max() > 0.0


@pytest.mark.parametrize("trsv", [F.EXG_TRSV_EXACT, F.EXG_TRSV_FAST], ids=["exact", "fast"])
@pytest.mark.parametrize("weight", [F.EXG_WEIGHT_APPLY, F.EXG_WEIGHT_GSPMV], ids=["apply", "gspmv"])
def test_graph_loop_equals_eager(case, trsv, weight):
    """The Arnoldi loop as one CUDA graph (WHILE node) runs the same kernels as
    the eager loop: bit-identical values, identical m, one graph launch per
    MEVP, and the graph is reused across MEVPs."""
    _, s, f, _ = case
    opts = s.options()
    rng = np.random.default_rng(11)
    vs = [rng.uniform(-1, 1, s.n) for _ in range(3)]
    res = {}
    for loop in (F.EXG_LOOP_EAGER, F.EXG_LOOP_GRAPH):
        with Context(0, trsv_mode=trsv, weight_mode=weight, loop_mode=loop) as c:
            c.set_system(s)
            c.set_factors(f)
            out = []
            for v in vs:
                try:
                    out.append(c.mevp_iks(v, 1e-12, eps=1e-8, m_max=opts.m_max))
                except ex.NoConvergenceError as e:  # the same failure in both modes
                    out.append((None, ("no-convergence", e.last_residual)))
            cn = c.counters()
            res[loop] = (out, cn.graph_launches, cn.graph_builds, cn.arnoldi_iters)
    (eo, eg, _, ei), (go, gg, gb, gi) = res[F.EXG_LOOP_EAGER], res[F.EXG_LOOP_GRAPH]
    assert eg == 0 and gg == len(vs) and gb == 1
    assert ei == gi
    for (a, ia), (b, ib) in zip(eo, go):
        if a is None or b is None:
            assert ia == ib
            continue
        assert ia.m == ib.m and ia.happy == ib.happy
        assert bit_equal(a, b)


# ---- dense block in isolation: k_dense against dense_expm --------------------------
@pytest.mark.parametrize("m", [1, 2, 7, 13, 32, 33, 41, 64, 100])
@pytest.mark.parametrize("norm", [1e-3, 0.2, 0.9, 2.0, 5.0, 40.0, 3000.0],
                         ids=["pade3", "pade5", "pade7", "pade9", "pade13", "squarings3", "squarings10"])
def test_dense_expm_bit_identical(ref, m, norm):
    """dense_expm (dense_matrix.cpp:185-225) through the dense-block kernel: every Padé degree, the
    scaling-and-squaring branch, the shared-memory scratch (m <= 32) and the global scratch above it
    (m up to MMAX = 100, config 2) — the same bits as the reference."""
    rng = np.random.default_rng(1000 * m + int(norm * 10))
    a = rng.standard_normal((m, m))
    a *= norm / np.abs(a).sum(axis=0).max()
    with Context(0) as c:
        e = np.empty((m, m))
        c._check(F.lib.exg_debug_dense_expm(c.handle, m, F.as_ptr(np.ascontiguousarray(a), C.c_double),
                                             F.as_ptr(e, C.c_double)))
    want = ref.dense_expm(a)
    assert np.array_equal(e.view(np.int64), np.asarray(want).view(np.int64))


def test_dense_expm_rejects_non_finite():
    a = np.eye(3)
    a[1, 2] = np.inf
    with Context(0) as c:
        e = np.empty((3, 3))
        with pytest.raises(ex.NonFiniteError):
            c._check(F.lib.exg_debug_dense_expm(c.handle, 3, F.as_ptr(a, C.c_double), F.as_ptr(e, C.c_double)))


# ---- the FAST-mode SpMV in isolation: k_spmv_v4 (small) and k_spmv_v4t (col/val through a shared-memory ring) ----
@pytest.mark.parametrize("cfg,kw", [(1, dict(width=64)), (1, dict(width=300)), (1, dict(width=420)),
                                    (2, dict(width=200)), (3, dict(n=3000))],
                         ids=["c1-4k", "c1-90k", "c1-176k", "c2-250k", "c3-3k"])
def test_fast_spmv_matches_reference(ref, cfg, kw):
    """sparse_matrix.cpp:69-82 with the row's products summed by four lanes: <= a few ulp of sum |c_ik x_k|.
    Systems above 64k rows take k_spmv_v4t (col/val through the shared-memory ring)."""
    s = ex.System.generate(cfg, **kw)
    x = np.random.default_rng(cfg).uniform(-1, 1, s.n)
    with Context(0, trsv_mode=F.EXG_TRSV_FAST) as c:
        c.set_system(s)
        y = np.zeros(s.n)
        c._check(F.lib.exg_debug_spmv_fast(c.handle, F.as_ptr(x, C.c_double), F.as_ptr(y, C.c_double)))
        y2 = np.zeros(s.n)
        c._check(F.lib.exg_debug_spmv_fast(c.handle, F.as_ptr(x, C.c_double), F.as_ptr(y2, C.c_double)))
    want = np.asarray(ref.spmv(s.C, x))
    rp = np.asarray(s.C.rowptr)
    rows = np.repeat(np.arange(s.n), np.diff(rp))
    mag = np.bincount(rows, np.abs(np.asarray(s.C.val) * x[np.asarray(s.C.col)]), minlength=s.n)
    assert np.all(np.abs(y - want) <= 8 * np.finfo(float).eps * mag)
    assert bit_equal(y, y2)


# ---- orthogonalize in isolation: k_mgs / k_mgs2 against krylov.cpp:46-78 --------
def _orthogonalize_ref(V, w, tol):
    """The reference's modified Gram-Schmidt with one conditional re-orthogonalisation."""
    w = w.copy()
    j = V.shape[1] - 1
    pre = np.sqrt(np.dot(w, w))
    h = np.zeros(j + 2)
    for i in range(j + 1):
        h[i] = np.dot(w, V[:, i])
        w -= h[i] * V[:, i]
    post = np.sqrt(np.dot(w, w))
    re = post < 0.70710678118654752 * pre
    if re:
        for i in range(j + 1):
            s = np.dot(w, V[:, i])
            w -= s * V[:, i]
            h[i] += s
        post = np.sqrt(np.dot(w, w))
    h[j + 1] = post
    happy = post <= tol * pre
    return h, (None if happy else w / post), happy, re


@pytest.mark.parametrize("mode", [F.EXG_TRSV_EXACT, F.EXG_TRSV_FAST], ids=["k_mgs", "k_mgs2"])
@pytest.mark.parametrize("n,j", [(1024, 0), (1024, 5), (11417, 12), (44640, 7), (300000, 3), (300000, 17),
                                 (1000800, 9)])
@pytest.mark.parametrize("kind", ["generic", "reorth", "happy"])
def test_orthogonalize_matches_reference(mode, n, j, kind):
    """One Arnoldi orthogonalisation step: Hessenberg column, next basis vector, the
    re-orthogonalisation trigger and the happy-breakdown flag, for one-CTA, few-CTA and full-grid
    shapes (k_mgs2's groups of 1..4 columns and its tile ring)."""
    rng = np.random.default_rng(n + 31 * j)
    V, _ = np.linalg.qr(rng.standard_normal((n, j + 1)))
    if kind == "generic":
        w = rng.standard_normal(n)
    elif kind == "reorth":  # mostly inside span(V): the norm drops by far more than 1/sqrt(2)
        w = V @ rng.standard_normal(j + 1) + 1e-3 * rng.standard_normal(n)
    else:  # inside span(V) to rounding: happy breakdown
        w = V @ rng.standard_normal(j + 1)
    tol = 1e-9 if kind == "happy" else 1e-12
    h_want, v_want, happy_want, re_want = _orthogonalize_ref(V, w, tol)
    with Context(0, trsv_mode=mode) as c:
        h = np.zeros(j + 2)
        v = np.zeros(n)
        info = np.zeros(2, np.int32)
        Vf = np.asfortranarray(V)
        c._check(F.lib.exg_debug_orthogonalize(c.handle, n, j, F.as_ptr(Vf, C.c_double), F.as_ptr(w, C.c_double), tol,
                                                F.as_ptr(h, C.c_double), F.as_ptr(v, C.c_double),
                                                F.as_ptr(info, C.c_int)))
    assert bool(info[0]) == happy_want
    assert bool(info[1]) == re_want
    scale = np.linalg.norm(w)
    assert np.max(np.abs(h[: j + 1] - h_want[: j + 1])) <= 1e-12 * scale
    if not happy_want:
        assert abs(h[j + 1] - h_want[j + 1]) <= 1e-9 * max(h_want[j + 1], 1e-300) + 1e-13 * scale
        assert np.max(np.abs(v - v_want)) <= 1e-8
        assert np.max(np.abs(V.T @ v)) <= 1e-10


# ---- run-to-run determinism of the polling / mbarrier kernels (compute-sanitizer is not available on
# the GPU pool: a data race or a read of a not-yet-published value would show up here as differing bits)
@pytest.mark.parametrize("cfg,kw", [(1, dict(width=64)), (1, dict(width=600)), (3, dict(n=3000))],
                         ids=["c1-64-levelruns", "c1-600-streams", "c3-3000"])
def test_fast_path_bits_repeat(cfg, kw):
    s = ex.System.generate(cfg, **kw)
    f = ex.lu_factor(s.G)
    rng = np.random.default_rng(3)
    b = rng.uniform(-1, 1, s.n)
    v = rng.uniform(-1, 1, s.n)
    outs, mevps = [], []
    for rep in range(3):
        with _ctx(s, f, F.EXG_TRSV_FAST) as c:
            c.set_options(trsv_mode=F.EXG_TRSV_FAST, weight_mode=F.EXG_WEIGHT_GSPMV,
                          loop_mode=F.EXG_LOOP_GRAPH if rep != 1 else F.EXG_LOOP_EAGER)
            xs = [c.solve(b) for _ in range(4)]
            for x in xs[1:]:
                assert np.array_equal(x.view(np.int64), xs[0].view(np.int64)), "FAST solve bits differ run to run"
            outs.append(xs[0])
            val, info = c.mevp_iks(v, 2e-12, eps=1e-9, m_max=40)
            mevps.append((val, info.m))
    for x in outs[1:]:
        assert np.array_equal(x.view(np.int64), outs[0].view(np.int64)), "FAST solve bits differ between contexts"
    for val, m in mevps[1:]:
        assert m == mevps[0][1]
        assert np.array_equal(val.view(np.int64), mevps[0][0].view(np.int64)), "MEVP bits differ between runs / loop modes"
