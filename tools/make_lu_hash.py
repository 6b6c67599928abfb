"""ORACLE / TEST INFRASTRUCTURE — pin the repo's host LU to exsim::lu_factor at full size.

Runs the reference's OWN ``lu_factor`` (oracle/_ref, sparse_lu.cpp:134-253,
with its O(n^2) exact minimum-degree ordering: ~1 h at 1M unknowns on one
core) on config k's G at full size, hashes the factor arrays exactly as
tools/make_golden.py hashes the repo's factor, and writes
tests/golden/lu_hash_c{k}.json.  tests/test_gpu_golden.py asserts that the
repo's ``lu_factor`` (csrc/lu.cpp) produces the same sha256 — i.e. the
factors the GPU path and the oracle fixtures use are the reference's own,
bit for bit, at 1M.

    python tools/make_lu_hash.py --config 1
"""
from __future__ import annotations

import argparse
import hashlib
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
import paper_1511_04515_b200 as ex  # noqa: E402
from ref import Ref  # noqa: E402


def export_sha(e) -> str:
    h = hashlib.sha256()
    for k in ("Lp", "Li", "Lx", "Up", "Ui", "Ux", "row_perm", "col_perm"):
        a = np.ascontiguousarray(e[k])
        if a.dtype == np.float64:
            a = np.where(a == 0.0, 0.0, a)  # -0.0 == 0.0 in the reference's value semantics
        h.update(a.tobytes())
    return h.hexdigest()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, required=True)
    args = ap.parse_args()
    s = ex.System.generate(args.config)
    G = s.G
    ref = Ref()
    t0 = time.time()
    fh = ref.lu_factor(G)
    wall = time.time() - t0
    try:
        e = ref.factor_export(fh)
    finally:
        ref.factor_free(fh)
    out = {"config": args.config, "n": int(G.n_rows), "nnz_G": int(G.nnz),
           "nnz_L": int(e["Li"].size), "nnz_U": int(e["Ui"].size),
           "sha256": export_sha(e), "ref_lu_factor_s": round(wall, 1),
           "how": "exsim::lu_factor (unmodified reference, oracle/_ref) on this container's CPU, 1 thread"}
    p = ROOT / "tests" / "golden" / f"lu_hash_c{args.config}.json"
    p.write_text(json.dumps(out, indent=1) + "\n")
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
