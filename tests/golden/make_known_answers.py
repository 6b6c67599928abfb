"""Writes tests/golden/known_answers.json: the closed-form values the
reference's own tests assert (proj/tests/test_dense.cpp:66-74,
test_krylov.cpp:65-78, test_integrate.cpp:101-134, :255-291).  The values are
analytic (exp of the stated arguments), so they are recomputed here rather
than copied; run: python tests/golden/make_known_answers.py"""
import json
import math
from pathlib import Path

out = {
    "dense_expm_diag": {"src": "test_dense.cpp:66-74", "diag": [-1.0, -2.0],
                        "want": [math.exp(-1.0), math.exp(-2.0)]},
    "mevp_happy": {"src": "test_krylov.cpp:65-78", "g_diag": [1.0, 2.0, 3.0], "h": 0.7,
                   "want": math.exp(-0.7)},
    "er_rc_decay": {"src": "test_integrate.cpp:101-111", "want": math.exp(-1.0)},
    "er_ramp": {"src": "test_integrate.cpp:122-134", "want": 1.0 - 1.0 + math.exp(-1.0)},
    "transient_rc": {"src": "test_integrate.cpp:255-291", "tol": 1e-6},
}
Path(__file__).with_name("known_answers.json").write_text(json.dumps(out, indent=1) + "\n")
