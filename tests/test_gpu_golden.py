"""Full-size parity against golden transients of the unmodified reference.

The fixtures under tests/golden/ were produced on the CPU by
tools/make_golden.py from oracle/_ref (exsim_core compiled from
/root/reference): configs 0 and 4 are ``exsim::transient()`` as shipped;
configs 1-3 the restated cached-factorization loop (pinned to transient() by
tests/test_oracle.py) with the factor whose sha256 the fixture records.
tools/make_lu_hash.py pins that factor against the reference's own
``lu_factor`` at full size (tests/golden/lu_hash_c*.json).

Each test replays the SAME transient through the drop-in driver
``exg_transient`` in the shipped performance mode (FAST triangular solves,
G-weight residual; config 4 runs EXACT) and requires:
identical step times, identical Krylov dimension of every MEVP, identical
rejection counts, and probed waveforms within 1e-8 of each node's full scale
(BASELINE.json north_star tolerance, full-scale form: SURVEY.md §0.7).
"""
import json
import sys
from pathlib import Path

import numpy as np
import pytest

import paper_1511_04515_b200 as ex
from paper_1511_04515_b200 import _ffi as F
from paper_1511_04515_b200.device import Context

from helpers import full_scale_err

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT / "tools"))
from make_golden import control, factor_sha  # noqa: E402

GOLDEN = ROOT / "tests" / "golden"
TOL = 1e-8

pytestmark = pytest.mark.gpu


def fixture(name):
    p = GOLDEN / name
    if not p.exists():
        pytest.skip(f"{name} not generated (tools/make_golden.py)")
    z = np.load(p)
    return {k: z[k] for k in z.files}


def compare(got, want):
    assert np.array_equal(got.times, want["times"]), "step times differ"
    want_dims = [want["dims"][want["dims_off"][i]:want["dims_off"][i + 1]].tolist()
                 for i in range(len(want["t"]))]
    assert got.krylov_dims == want_dims, "Krylov dimension sequence differs"
    assert np.array_equal(got.rejects, want["rejects"]), "rejection sequence differs"
    err = full_scale_err(got.samples, want["samples"])
    assert err <= TOL, f"waveform full-scale error {err:.3e}"
    return err


@pytest.mark.parametrize("cfg", [0, 1, 2, 3])
def test_linear_config_full_size(cfg):
    want = fixture(f"config{cfg}_full.npz")
    s = ex.System.generate(cfg)
    ctl = control(s, cfg, None)
    if want["lu_sha"].item():
        # the factor exg_transient builds is the one the oracle used ...
        f = ex.lu_factor(s.G)
        assert factor_sha(f) == want["lu_sha"].item()
        del f
        # ... and the reference's own lu_factor's, where that pin exists
        pin = GOLDEN / f"lu_hash_c{cfg}.json"
        if pin.exists():
            assert json.loads(pin.read_text())["sha256"] == want["lu_sha"].item()
    with Context(0, trsv_mode=F.EXG_TRSV_FAST, weight_mode=F.EXG_WEIGHT_GSPMV) as c:
        got = c.transient(s, ctl, s.options().tran_stop, want["rec"])
    compare(got, want)


@pytest.mark.parametrize("method", ["er"])
def test_config4_full_size(method):
    want = fixture(f"config4_{method}_full.npz")
    s = ex.System.generate(4)
    ctl = control(s, 4, F.EXG_METHOD_ERC if method == "erc" else F.EXG_METHOD_ER)
    with Context(0, trsv_mode=F.EXG_TRSV_EXACT, weight_mode=F.EXG_WEIGHT_APPLY) as c:
        got = c.transient(s, ctl, s.options().tran_stop, want["rec"])
    assert np.array_equal(got.t, want["t"]), "accepted step times differ"
    compare(got, want)


def test_config4_refactor_policy_full_size():
    """Config 4 as BASELINE.json states it (refactor when the Jacobian changed by more than 10%)
    against the golden transient of the restated loop with the same policy."""
    want = fixture("config4_er_th0.1_full.npz")
    s = ex.System.generate(4)
    ctl = control(s, 4, F.EXG_METHOD_ER)
    ctl.refactor_threshold = 0.1
    with Context(0, trsv_mode=F.EXG_TRSV_EXACT, weight_mode=F.EXG_WEIGHT_APPLY) as c:
        got = c.transient(s, ctl, s.options().tran_stop, want["rec"])
    assert np.array_equal(got.t, want["t"]), "accepted step times differ"
    assert int(np.sum(got.lu_count)) < len(got.t), "the policy skipped no factorization"
    compare(got, want)
