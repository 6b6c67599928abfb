"""CPU tests: pin the oracle before trusting it.

1. The C restatement (oracle/exsim_oracle.c) is bit-identical to the
   reference library (oracle/_ref) on spmv, solve, apply, dense_expm,
   mevp_iks and er_step.
2. The restated cached-LU ER loop (ref_transient_cached) is bit-identical to
   exsim::transient() as shipped.
3. Both reproduce the reference tests' known-answer values
   (tests/golden/known_answers.json, from proj/tests/*.cpp).
"""
import json
from pathlib import Path

import numpy as np
import pytest

import paper_1511_04515_b200 as ex
from paper_1511_04515_b200 import _ffi as F

from helpers import bit_equal, random_rc_pair, ref_system

GOLDEN = json.loads((Path(__file__).parent / "golden" / "known_answers.json").read_text())


@pytest.fixture(scope="module")
def sys0():
    return ex.System.generate(0)


def test_restatement_matches_reference_kernels(ref, orc, sys0):
    s = sys0
    f = ex.lu_factor(s.G)
    fh = ref.factor_from(f)
    rng = np.random.default_rng(0)
    try:
        x = rng.uniform(-1, 1, s.n)
        assert bit_equal(orc.spmv(s.C, x), ref.spmv(s.C, x))
        assert bit_equal(orc.solve(f, x), ref.solve(fh, x))
        assert bit_equal(orc.apply(f, x), ref.apply(fh, x))
        for eps in (1e-7, 1e-12):
            got, gi = orc.mevp_iks(f, s.C, x, 1e-12, eps=eps, m_max=30)
            want, wi = ref.mevp_iks(fh, s.C, x, 1e-12, eps=eps, m_max=30)
            assert gi["m"] == wi["m"]
            assert bit_equal(got, want)
    finally:
        ref.factor_free(fh)


@pytest.mark.parametrize("n,scale", [(3, 0.01), (6, 0.2), (9, 0.9), (12, 2.0), (15, 40.0), (30, 300.0)])
def test_restatement_dense_expm(ref, orc, n, scale):
    a = np.random.default_rng(n).uniform(-1, 1, (n, n)) * scale / n
    assert bit_equal(orc.dense_expm(a), ref.dense_expm(a))


def test_restatement_er_step(ref, orc, sys0):
    s = sys0
    f = ex.lu_factor(s.G)
    rh = ref_system(ref, s)
    try:
        x0 = ref.dc_solve(rh)
        u0, u1 = s.eval_sources(0.0), s.eval_sources(1e-12)
        xn, m = orc.er_step(f, s.C, s.B, x0, u0, u1, 1e-12, eps=1e-7, m_max=30)
        ctl = s.step_control()
        ctl.fixed_step = 1
        ctl.h_init = 1e-12
        fh = ref.factor_from(f)
        r = ref.transient_cached(rh, fh, ctl, 1e-9, np.arange(s.n), max_steps=1)
        ref.factor_free(fh)
        assert bit_equal(xn, r["samples"][1])
        assert [m] == r["dims"].tolist()
    finally:
        ref.system_free(rh)


def test_cached_loop_equals_transient_as_shipped(ref):
    """The cached-LU restatement is the reference's transient() bit for bit."""
    s = ex.System.generate(0, width=16)
    ctl = s.step_control()
    rec = np.arange(0, s.n, 7, dtype=np.int32)
    for fixed in (1, 0):
        ctl.fixed_step = fixed
        ctl.h_init = 1e-12 if fixed else 0.0
        rh = ref_system(ref, s)
        try:
            a = ref.transient(rh, ctl, 3e-10, rec)
            f = ex.lu_factor(s.G)
            fh = ref.factor_from(f)
            b = ref.transient_cached(rh, fh, ctl, 3e-10, rec)
            ref.factor_free(fh)
            c = ref.transient_cached(rh, None, ctl, 3e-10, rec)  # refactor every step
        finally:
            ref.system_free(rh)
        for r in (b, c):
            assert np.array_equal(a["times"], r["times"])
            assert bit_equal(a["samples"], r["samples"])
            assert np.array_equal(a["dims"], r["dims"])
            assert np.array_equal(a["dims_off"], r["dims_off"])


def test_known_answers_dense(ref, orc):
    g = GOLDEN["dense_expm_diag"]  # test_dense.cpp:66-74
    a = np.diag(g["diag"])
    for impl in (ref.dense_expm, orc.dense_expm):
        e = impl(a)
        assert e[0, 0] == pytest.approx(g["want"][0], rel=1e-14)
        assert e[1, 1] == pytest.approx(g["want"][1], rel=1e-14)
        assert abs(e[0, 1]) < 1e-16
    nil = np.array([[0.0, 1.0], [0.0, 0.0]])  # test_dense.cpp:57-64
    for impl in (ref.dense_expm, orc.dense_expm):
        e = impl(nil)
        assert e[0, 1] == pytest.approx(1.0, rel=1e-15) and e[1, 0] == 0.0


def test_known_answers_krylov(ref, orc):
    g = GOLDEN["mevp_happy"]  # test_krylov.cpp:65-78
    Cm = ex.Csr(3, 3, np.array([0, 1, 2, 3], np.int32), np.array([0, 1, 2], np.int32), np.ones(3))
    G = ex.Csr(3, 3, np.array([0, 1, 2, 3], np.int32), np.array([0, 1, 2], np.int32),
               np.array(g["g_diag"]))
    f = ex.lu_factor(G)
    fh = ref.factor_from(f)
    try:
        for got, info in (orc.mevp_iks(f, Cm, np.array([1.0, 0, 0]), g["h"]),
                          ref.mevp_iks(fh, Cm, np.array([1.0, 0, 0]), g["h"])):
            assert info["m"] == 1 and info["happy"]
            assert got[0] == pytest.approx(g["want"], rel=1e-13)
    finally:
        ref.factor_free(fh)


def _rc_cell(elements, gmin=0.0, tran=None):
    """Tiny netlist-equivalent systems of proj/tests/test_integrate.cpp."""
    els = (F.exg_element * len(elements))()
    srcs = []
    pwl_t, pwl_v = [], []
    for i, (kind, a, b, val, src) in enumerate(elements):
        els[i].kind = kind
        els[i].nodes[0], els[i].nodes[1], els[i].nodes[2], els[i].nodes[3] = a, b, -2, -2
        els[i].value = val
        els[i].aux = -1
        if src is not None:
            s = F.exg_source()
            if src[0] == "pwl":
                s.kind = F.EXG_SRC_PWL
                s.pwl_off = len(pwl_t)
                s.pwl_len = len(src[1])
                for t, v in src[1]:
                    pwl_t.append(t)
                    pwl_v.append(v)
            else:
                s.kind = F.EXG_SRC_DC
                s.dc = src[1]
            els[i].aux = len(srcs)
            srcs.append(s)
    sarr = (F.exg_source * max(len(srcs), 1))(*srcs)
    o = F.exg_options()
    o.err_budget, o.krylov_eps, o.gmin, o.m_max = 1e-4, 1e-7, gmin, 100
    o.hmin = o.hmax = float("nan")
    if tran:
        o.has_tran, o.tran_step, o.tran_stop = 1, tran[0], tran[1]
    return ex.System.build(els, sarr if srcs else (F.exg_source * 0)(), pwl_t, pwl_v,
                           (F.exg_mos_model * 0)(), o)


def test_known_answer_rc_decay(ref, orc):
    """test_integrate.cpp:101-111: R=C=1, x0=1, h=1 -> e^{-1} (1e-12)."""
    s = _rc_cell([(F.EXG_EL_R, 0, -1, 1.0, None), (F.EXG_EL_C, 0, -1, 1.0, None)])
    f = ex.lu_factor(s.G)
    xn, m = orc.er_step(f, s.C, s.B, np.array([1.0]), np.zeros(0), np.zeros(0), 1.0, eps=1e-9)
    assert xn[0] == pytest.approx(GOLDEN["er_rc_decay"]["want"], rel=1e-12)


def test_known_answer_ramp(ref, orc):
    """test_integrate.cpp:122-134: unit ramp into RC -> t - 1 + e^{-t} at t=1."""
    s = _rc_cell([(F.EXG_EL_V, 1, -1, 0.0, ("pwl", [(0.0, 0.0), (1.0, 1.0)])),
                  (F.EXG_EL_R, 1, 0, 1.0, None), (F.EXG_EL_C, 0, -1, 1.0, None)])
    f = ex.lu_factor(s.G)
    n1 = s.unknown_of_label(0)
    x0 = np.zeros(s.n)
    xn, m = orc.er_step(f, s.C, s.B, x0, s.eval_sources(0.0), s.eval_sources(1.0), 1.0, eps=1e-10)
    assert xn[n1] == pytest.approx(GOLDEN["er_ramp"]["want"], rel=1e-11)


def test_known_answer_transient_rc(ref):
    """test_integrate.cpp:255-291 via the reference: piecewise-exact oracle 1e-6."""
    s = _rc_cell([(F.EXG_EL_V, 1, -1, 0.0, ("pwl", [(0.0, 1.0), (1e-6, 0.0)])),
                  (F.EXG_EL_R, 1, 0, 1.0, None), (F.EXG_EL_C, 0, -1, 1.0, None)],
                 tran=(0.05, 5.0))
    ctl = s.step_control()
    ctl.eps = 1e-9
    ctl.err_budget = 1e-6
    n1 = s.unknown_of_label(0)
    rh = ref_system(ref, s)
    try:
        r = ref.transient(rh, ctl, 5.0, [n1])
    finally:
        ref.system_free(rh)
    v_ref, t_prev, max_err = 1.0, 0.0, 0.0
    u_of = lambda t: 0.0 if t >= 1e-6 else 1.0 - t / 1e-6
    for t, v in zip(r["times"], r["samples"][:, 0]):
        dt = t - t_prev
        if dt > 0:
            a0, a1 = u_of(t_prev), u_of(t)
            b = (a1 - a0) / dt
            k0 = v_ref - (a0 - b)
            v_ref = (a0 - b) + b * dt + k0 * np.exp(-dt)
        max_err = max(max_err, abs(v - v_ref))
        t_prev = t
    assert max_err <= GOLDEN["transient_rc"]["tol"]


def test_refactor_policy_oracle_pins(ref):
    """The restated loop with the refactor policy (exg_step_control.refactor_threshold):
    threshold 0 is transient() as shipped bit for bit (nonlinear circuit, a factorization per
    step); threshold 0.1 freezes the Linearization between refactorizations: fewer lu_factor
    calls, same physics to the policy's accuracy."""
    s = ex.System.generate(4, width=12, chains=4, stages=4)
    ctl = s.step_control()
    rec = np.arange(0, s.n_nodes, 5, dtype=np.int32)
    t_stop = s.options().tran_stop
    rh = ref_system(ref, s)
    try:
        a = ref.transient(rh, ctl, t_stop, rec)
        b = ref.transient_policy(rh, ctl, t_stop, rec, threshold=0.0)
        c = ref.transient_policy(rh, ctl, t_stop, rec, threshold=0.1)
    finally:
        ref.system_free(rh)
    assert np.array_equal(a["times"], b["times"]) and bit_equal(a["samples"], b["samples"])
    assert np.array_equal(a["dims"], b["dims"]) and np.array_equal(a["rejects"], b["rejects"])
    assert np.all(b["lu"] == 1)
    assert 0 < int(np.sum(c["lu"])) < int(np.sum(b["lu"])), "the policy skipped no factorization"
    assert c["lu"][0] == 1
    assert c["times"][-1] == a["times"][-1]
    scale = np.max(np.abs(a["samples"]))
    assert np.max(np.abs(c["samples"][-1] - a["samples"][-1])) <= 2e-2 * scale
