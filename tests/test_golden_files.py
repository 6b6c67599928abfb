"""CPU checks of the committed full-size golden fixtures (no GPU, no reference).

The fixtures are data; these tests check they are complete and mutually
consistent: every step has its Krylov dimensions, the waveform has one row per
accepted step plus t = 0, the probe list is the seeded one, and the factor
hash a linear fixture was computed with equals the hash of the reference's own
lu_factor where tools/make_lu_hash.py pinned it.
"""
import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT / "tools"))
from make_golden import probes  # noqa: E402

GOLDEN = ROOT / "tests" / "golden"
FILES = sorted(GOLDEN.glob("config*_full.npz"))


@pytest.mark.parametrize("path", FILES, ids=[p.stem for p in FILES])
def test_fixture_consistent(path):
    z = np.load(path)
    meta = json.loads(z["meta"].item())
    ns = len(z["t"])
    assert ns == meta["steps"] > 0
    assert z["samples"].shape == (ns + 1, len(z["rec"]))
    assert np.all(np.diff(z["times"]) > 0) and z["times"][0] == 0.0
    assert np.array_equal(z["times"][1:], z["t"])
    assert z["dims_off"][0] == 0 and z["dims_off"][-1] == len(z["dims"]) == meta["mevps"]
    assert np.all(np.diff(z["dims_off"]) >= 0)
    assert int(np.sum(z["rejects"])) == meta["rejects"]
    assert np.all(np.isfinite(z["samples"]))


@pytest.mark.parametrize("cfg", [1, 2])
def test_lu_pin_matches_fixture(cfg):
    pin, fx = GOLDEN / f"lu_hash_c{cfg}.json", GOLDEN / f"config{cfg}_full.npz"
    if not (pin.exists() and fx.exists()):
        pytest.skip("pin or fixture not generated")
    assert json.loads(pin.read_text())["sha256"] == np.load(fx)["lu_sha"].item()


def test_probes_are_seeded():
    a = probes(1_000_000)
    assert np.array_equal(a, probes(1_000_000)) and a.size == 16 and np.all(np.diff(a) > 0)
