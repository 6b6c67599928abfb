"""CPU tests of the FAST-solve plan (csrc/trsv_plan.cpp, exg_aug_plan_solve).

The blocked augmented system replaces every dense diagonal block of a factor
by y = b - (external part), x = inv(block) y, and cuts long rows into partial
sums.  Evaluated in plan order on the CPU it must solve the same triangular
system as Factorization::solve's sweeps (sparse_lu.cpp:255-291), to rounding
(the block inverse reorders the arithmetic: FAST mode's <= 1e-13 contract),
with far fewer dependency levels.  The reference solve here is the oracle's
Factorization::solve restated in oracle/exsim_oracle.c (pinned to the
reference by tests/test_oracle.py), run on the same factor.
"""
import ctypes as C

import numpy as np
import pytest

import paper_1511_04515_b200 as ex
from paper_1511_04515_b200 import _ffi as F


def strict_parts(f):
    """L strictly lower, U strictly upper + diagonal, in pivot coordinates."""
    n = f.n
    out = []
    for upper, M in ((False, f.L), (True, f.U)):
        ptr, col, val, diag = [0], [], [], np.ones(n)
        for r in range(n):
            s, e = M.rowptr[r], M.rowptr[r + 1]
            for k in range(s, e):
                c = M.col[k]
                if c == r:
                    if upper:
                        diag[r] = M.val[k]
                elif (c > r) == upper:
                    col.append(c)
                    val.append(M.val[k])
            ptr.append(len(col))
        out.append((np.array(ptr, np.int32), np.array(col, np.int32), np.array(val), diag))
    return out


def aug_solve(upper, n, part, in_index, b, params=None):
    ptr, col, val, diag = part
    x = np.zeros(n)
    st = (C.c_longlong * 8)()
    prm = (C.c_int * 5)(*params) if params else None
    rc = F.lib.exg_aug_plan_solve(int(upper), n, F.as_ptr(ptr, C.c_int), F.as_ptr(col, C.c_int),
                                  F.as_ptr(val, C.c_double), F.as_ptr(diag, C.c_double),
                                  F.as_ptr(in_index, C.c_int), prm, F.as_ptr(b, C.c_double),
                                  F.as_ptr(x, C.c_double), st)
    assert rc == F.EXG_OK, F.lib.exg_host_error_message().decode()
    return x, dict(zip(["orig_levels", "levels", "blocks", "block_rows", "max_block", "partials",
                        "n_aug", "tasks"], list(st)))


CASES = [(0, {}), (1, dict(width=64)), (2, dict(width=12)), (3, dict(n=3000)),
         (4, dict(width=10, chains=4, stages=4))]


@pytest.mark.parametrize("cfg,kw", CASES, ids=[f"c{c}" for c, _ in CASES])
@pytest.mark.parametrize("params", [None, (2, 16, 40, 8, 16)], ids=["default", "small-blocks-chunked"])
def test_aug_plan_solves_the_factor(orc, cfg, kw, params):
    s = ex.System.generate(cfg, **kw)
    f = ex.lu_factor(s.G)
    n = f.n
    lpart, upart = strict_parts(f)
    b = np.random.default_rng(cfg).uniform(-1, 1, n)
    # L sweep reads b through row_perm; U sweep reads the L result in place
    y, sl = aug_solve(False, n, lpart, np.asarray(f.row_perm, np.int32), b, params)
    z, su = aug_solve(True, n, upart, np.arange(n, dtype=np.int32), y, params)
    x = np.empty(n)
    x[np.asarray(f.col_perm)] = z
    want = orc.solve(f, b)
    err = np.max(np.abs(x - want)) / np.max(np.abs(want))
    assert err <= 1e-13, err
    for st in (sl, su):
        assert st["levels"] <= st["orig_levels"] + 1
        assert st["n_aug"] == n + st["block_rows"] + st["partials"]
    if params:  # tiny blocks and chunks exercise every row kind
        assert sl["blocks"] + su["blocks"] > 0
        assert sl["partials"] + su["partials"] > 0 or max(np.diff(lpart[0]).max(), np.diff(upart[0]).max()) <= 40


def test_aug_plan_dense_triangle_is_one_block():
    """A dense unit-lower triangle becomes one block: two levels, exact to rounding."""
    n = 50
    rng = np.random.default_rng(3)
    ptr, col, val = [0], [], []
    for r in range(n):
        col += list(range(r))
        val += list(rng.uniform(-0.1, 0.1, r))
        ptr.append(len(col))
    part = (np.array(ptr, np.int32), np.array(col, np.int32), np.array(val), np.ones(n))
    b = rng.uniform(-1, 1, n)
    x, st = aug_solve(False, n, part, np.arange(n, dtype=np.int32), b, (8, 4096, 10000, 128, 256))
    assert st["orig_levels"] == n and st["levels"] == 2 and st["blocks"] == 1 and st["max_block"] == n
    Ld = np.eye(n)
    for r in range(n):
        Ld[r, :r] = val[ptr[r]:ptr[r + 1]]
    assert np.allclose(x, np.linalg.solve(Ld, b), rtol=0, atol=1e-13)


def test_aug_plan_rejects_bad_parameters():
    z = np.zeros(2, np.int32)
    d = np.ones(1)
    rc = F.lib.exg_aug_plan_solve(0, 1, F.as_ptr(z, C.c_int), F.as_ptr(z, C.c_int), F.as_ptr(d, C.c_double),
                                  F.as_ptr(d, C.c_double), F.as_ptr(z, C.c_int), (C.c_int * 5)(8, 0, 1, 1, 1),
                                  None, None, None)
    assert rc == F.EXG_E_CONTRACT


# ---- per-warp record streams (k_trsv4's input format, trsv_plan.hpp) ---------------------------
def stream_solve(upper, n, part, in_index, b, n_warps, out_index=None, coef=1.0, add=None, params=None):
    ptr, col, val, diag = part
    x = np.zeros(n)
    fin = np.full(n, np.nan) if out_index is not None else None
    st = (C.c_longlong * 10)()
    prm = (C.c_int * 2)(*params) if params else None
    rc = F.lib.exg_stream_plan_solve(
        int(upper), n, F.as_ptr(ptr, C.c_int), F.as_ptr(col, C.c_int), F.as_ptr(val, C.c_double),
        F.as_ptr(diag, C.c_double), F.as_ptr(in_index, C.c_int),
        F.as_ptr(out_index, C.c_int) if out_index is not None else None, prm, n_warps,
        F.as_ptr(b, C.c_double), F.as_ptr(x, C.c_double),
        F.as_ptr(fin, C.c_double) if fin is not None else None, coef,
        F.as_ptr(add, C.c_double) if add is not None else None, st)
    assert rc == F.EXG_OK, F.lib.exg_host_error_message().decode()
    return x, fin, dict(zip(["orig_levels", "levels", "n_aug", "tasks", "rows", "entries", "slots", "bytes",
                             "max_record", "partials"], list(st)))


@pytest.mark.parametrize("cfg,kw", CASES, ids=[f"c{c}" for c, _ in CASES])
@pytest.mark.parametrize("n_warps", [8, 1000, 3552])
def test_stream_plan_solves_the_factor(orc, cfg, kw, n_warps):
    """The streams, evaluated warp-round-robin as the kernel's static schedule runs them, solve
    the factor to FAST mode's 1e-13, including the fused epilogue of the U sweep."""
    s = ex.System.generate(cfg, **kw)
    f = ex.lu_factor(s.G)
    n = f.n
    lpart, upart = strict_parts(f)
    rng = np.random.default_rng(cfg)
    b = rng.uniform(-1, 1, n)
    add = rng.uniform(-1, 1, n)
    y, _, sl = stream_solve(False, n, lpart, np.asarray(f.row_perm, np.int32), b, n_warps)
    z, fin, su = stream_solve(True, n, upart, np.arange(n, dtype=np.int32), y, n_warps,
                              out_index=np.asarray(f.col_perm, np.int32), coef=-2.0, add=add)
    x = np.empty(n)
    x[np.asarray(f.col_perm)] = z
    want = orc.solve(f, b)
    scale = np.max(np.abs(want))
    assert np.max(np.abs(x - want)) / scale <= 1e-13
    assert np.max(np.abs(fin - (add - 2.0 * want))) / max(scale, 1.0) <= 1e-12
    for st in (sl, su):
        assert st["levels"] <= st["orig_levels"] + 2
        assert st["rows"] == st["n_aug"] and st["entries"] <= st["slots"]
        assert st["max_record"] <= 2048 and st["max_record"] % 16 == 0  # one record per ring slot (TMA granularity)
        assert st["bytes"] % 16 == 0


def test_stream_plan_long_rows_become_partials():
    """A dense triangle of 700 rows: rows of up to 699 entries are cut into 128-entry partial sums
    (and the block inverse keeps the level count at a handful)."""
    n = 700
    rng = np.random.default_rng(5)
    ptr, col, val = [0], [], []
    for r in range(n):
        col += list(range(r))
        val += list(rng.uniform(-0.01, 0.01, r))
        ptr.append(len(col))
    part = (np.array(ptr, np.int32), np.array(col, np.int32), np.array(val), np.ones(n))
    b = rng.uniform(-1, 1, n)
    Ld = np.eye(n)
    for r in range(n):
        Ld[r, :r] = val[ptr[r]:ptr[r + 1]]
    want = np.linalg.solve(Ld, b)
    for params in (None, (100000, 4096)):  # with the block inverse / plain rows with partial sums only
        x, _, st = stream_solve(False, n, part, np.arange(n, dtype=np.int32), b, 64, params=params)
        assert st["partials"] > 0
        assert np.allclose(x, want, rtol=0, atol=1e-12)
    assert st["levels"] >= n  # no block rewrite: the dense triangle stays sequential


@pytest.mark.parametrize("cfg,kw", [(1, dict(width=64)), (1, dict(width=160)), (3, dict(n=3000))],
                         ids=["c1-4k", "c1-26k", "c3"])
def test_stream_plan_orders_and_bundles_agree_bit_for_bit(monkeypatch, cfg, kw):
    """A row's arithmetic depends on its own lanes only: level order (task t on warp t mod W), the
    list schedule, and the list schedule with bundles of rows sharing a column list (cont records,
    evaluated with the columns of the record before them) all give the same bits.  The dense
    triangle below makes sure bundles exist and shrink the streams (no column ids in a cont record)."""
    s = ex.System.generate(cfg, **kw)
    f = ex.lu_factor(s.G)
    n = f.n
    parts = strict_parts(f)
    b = np.random.default_rng(cfg).uniform(-1, 1, n)
    for upper, part, in_index in ((False, parts[0], np.asarray(f.row_perm, np.int32)),
                                  (True, parts[1], np.arange(n, dtype=np.int32))):
        got = []
        for sched, bundle in ((0, 1), (1, 1), (1, 3), (1, 16)):
            monkeypatch.setenv("EXG_STREAM_SCHED", str(sched))
            monkeypatch.setenv("EXG_STREAM_BUNDLE", str(bundle))
            x, _, st = stream_solve(upper, n, part, in_index, b, 256)
            got.append((x, st))
        for x, st in got[1:]:
            assert np.array_equal(x.view(np.int64), got[0][0].view(np.int64))
            assert st["tasks"] >= got[0][1]["tasks"] - 64 and st["entries"] == got[0][1]["entries"]
        assert got[3][1]["bytes"] <= got[2][1]["bytes"] <= got[1][1]["bytes"]


def test_stream_plan_bundles_shrink_a_dense_block(monkeypatch):
    """Rows of a 700-row block inverse over one 128-column chunk repeat a column list: bundled, they
    drop their column ids (512 bytes of a 1.5 KB record)."""
    n = 700
    rng = np.random.default_rng(7)
    ptr, col, val = [0], [], []
    for r in range(n):
        col += list(range(r))
        val += list(rng.uniform(-0.01, 0.01, r))
        ptr.append(len(col))
    part = (np.array(ptr, np.int32), np.array(col, np.int32), np.array(val), np.ones(n))
    b = rng.uniform(-1, 1, n)
    res = {}
    for bundle in (1, 3):
        monkeypatch.setenv("EXG_STREAM_BUNDLE", str(bundle))
        res[bundle] = stream_solve(False, n, part, np.arange(n, dtype=np.int32), b, 64)
    assert np.array_equal(res[1][0].view(np.int64), res[3][0].view(np.int64))
    assert res[3][2]["bytes"] < 0.9 * res[1][2]["bytes"]
