"""Per-config throughput of the whole transient through the drop-in driver
(exg_transient = the reference's transient() loop over the device hot path),
for every BASELINE.json config, next to the reference CPU path on a bounded
sample of the same transient.  One JSON line per config; also written to
gpurun_out/configs.json.

    python tools/bench_configs.py [--configs 0,1,2,3,4] [--cpu-seconds 20]

GPU: FAST solves + G-weight (the bench modes), full transient from the DC
point, wall time of the step loop (host step control, H2D/D2H of sources and
probes included) -> steps/s and Arnoldi iterations/s.
CPU: the unmodified reference (oracle/_ref) restated ER loop with the cached
factorization, 1 thread, first K steps (K bounded by --cpu-seconds); config 4
(nonlinear, refactor per step as shipped) is not sampled at full size.
Parity: full-scale waveform error of the GPU run against the CPU sample on
the shared steps (linear configs)."""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
import paper_1511_04515_b200 as ex  # noqa: E402
from bench import CFG_FIXED_STEP  # noqa: E402
from paper_1511_04515_b200 import _ffi as F  # noqa: E402
from paper_1511_04515_b200.device import Context  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="0,1,2,3,4")
ap.add_argument("--cpu-seconds", type=float, default=20.0)
ap.add_argument("--threshold", type=float, default=0.1,
                help="config 4: refactor threshold (BASELINE.json names 0.1; 0 = every step, the reference)")
ap.add_argument("--exact4", action="store_true", help="config 4 in EXACT + APPLY mode (the parity modes)")
ap.add_argument("--out", default=str(ROOT / "gpurun_out" / "configs.json"))
args = ap.parse_args()

results = []
for cfg in [int(x) for x in args.configs.split(",")]:
    t0 = time.perf_counter()
    s = ex.System.generate(cfg)
    gen_s = time.perf_counter() - t0
    ctl = s.step_control()
    if CFG_FIXED_STEP(s):  # configs 0 and 3: fixed 1 ps steps (BASELINE.json)
        ctl.fixed_step = 1
        ctl.h_init = 1e-12
    t_stop = s.options().tran_stop
    n = s.n
    rng = np.random.default_rng(5)
    rec = np.sort(rng.choice(s.n_nodes, size=min(16, s.n_nodes), replace=False)).astype(np.int32)
    if cfg == 4:  # probe the unknowns the golden transient of the same policy recorded
        name = "config4_er_full.npz" if args.threshold == 0 else f"config4_er_th{args.threshold:g}_full.npz"
        if (ROOT / "tests" / "golden" / name).exists():
            rec = np.load(ROOT / "tests" / "golden" / name)["rec"].astype(np.int32)
    print(f"config {cfg}: n={n}, GPU transient to {t_stop:g} s ...", file=sys.stderr, flush=True)
    if cfg == 4:
        ctl.refactor_threshold = args.threshold
    exact = cfg == 4 and args.exact4
    with Context(0, trsv_mode=F.EXG_TRSV_EXACT if exact else F.EXG_TRSV_FAST,
                 weight_mode=F.EXG_WEIGHT_APPLY if exact else F.EXG_WEIGHT_GSPMV) as c:
        c.reset_counters()
        got = c.transient(s, ctl, t_stop, rec)
        cn = c.counters()
    print(f"config {cfg}: {len(got.t)} steps in {got.loop_s:.1f} s (LU {got.lu_s:.1f} s, DC {got.dc_s:.1f} s)",
          file=sys.stderr, flush=True)
    steps = len(got.t)
    iters = int(cn.arnoldi_iters)
    dims = [d for ds in got.krylov_dims for d in ds]
    r = {"config": cfg, "n": n, "nnz_C": s.C.nnz, "nnz_G": s.G.nnz, "steps": steps,
         "rejects": int(np.sum(got.rejects)), "mevps": len(dims), "arnoldi_iters": iters,
         "m_mean": round(float(np.mean(dims)), 2) if dims else 0, "m_max": int(max(dims)) if dims else 0,
         "loop_s": round(got.loop_s, 3), "steps_per_s": round(steps / got.loop_s, 2),
         "arnoldi_iters_per_s": round(iters / got.loop_s, 1), "lu_s": round(got.lu_s, 2),
         "dc_s": round(got.dc_s, 3), "gen_s": round(gen_s, 2), "l_levels": cn.l_levels,
         "u_levels": cn.u_levels, "gpu_launches": int(cn.kernel_launches),
         "graph_launches": int(cn.graph_launches)}
    if cfg == 4:
        # parity against the committed golden transient of the same policy (tools/make_golden.py:
        # the restated loop over the unmodified reference, full size)
        r["modes"] = "exact+apply" if exact else "fast+gspmv"
        r["refactor_threshold"] = args.threshold
        r["lu_count"] = int(np.sum(got.lu_count))
        name = "config4_er_full.npz" if args.threshold == 0 else f"config4_er_th{args.threshold:g}_full.npz"
        gp = ROOT / "tests" / "golden" / name
        if gp.exists():
            z = np.load(gp)
            m = min(len(z["times"]), len(got.times))
            same_t = bool(len(z["times"]) == len(got.times) and np.array_equal(z["times"], got.times))
            fs = np.max(np.abs(z["samples"]), axis=0)
            fs[fs == 0] = 1.0
            same_rec = bool(np.array_equal(z["rec"], rec))
            err = float(np.max(np.abs(got.samples[:m] - z["samples"][:m]) / fs)) if (m and same_rec) else None
            gd = [d for ds in got.krylov_dims for d in ds]
            r["parity"] = {"golden": name, "same_times": same_t, "same_rejects": bool(np.array_equal(z["rejects"], got.rejects)) if same_t else False,
                           "krylov_dims_equal": bool(np.array_equal(z["dims"], np.asarray(gd))), "full_scale_err": err,
                           "tol": 1e-8, "golden_wall_s": json.loads(str(z["meta"])).get("wall_s")}
            gw = json.loads(str(z["meta"])).get("wall_s")
            if gw:
                r["cpu_baseline"] = {"steps_per_s": round(len(z["t"]) / gw, 4), "cores": 1, "kind": "reference",
                                     "sample": "the whole golden transient (restated loop over the unmodified "
                                               "reference, same policy), wall time of tools/make_golden.py here"}
    # ---- CPU reference sample (linear configs)
    if s.n_mos == 0:
        from helpers_bench import ref_system_for
        from ref import Ref
        ref = Ref()
        rh = ref_system_for(ref, s)
        f = ex.lu_factor(s.G)
        fh = ref.factor_from(f)
        # the DC point with the (bit-identical) cached factorization, as the
        # reference's dc_solve computes it for a linear circuit
        # (integrate.cpp:92-115) -- without it the restated loop would run the
        # reference's own lu_factor (about an hour at 1M nodes)
        x0 = ref.solve(fh, ref.spmv(s.B, s.eval_sources(0.0)))
        try:
            # size the sample: time 2 steps, then extend to ~cpu_seconds
            w = ref.transient_cached(rh, fh, ctl, t_stop, rec, max_steps=2, x0=x0)
            per = float(w["wall"][-1]) / max(len(w["wall"]), 1)
            k = int(max(2, min(steps, args.cpu_seconds / max(per, 1e-6))))
            if k > len(w["wall"]):
                w = ref.transient_cached(rh, fh, ctl, t_stop, rec, max_steps=k, x0=x0)
        finally:
            ref.factor_free(fh)
            ref.system_free(rh)
        kk = len(w["wall"])
        cpu_sps = kk / float(w["wall"][-1])
        ts = np.asarray(w["times"])
        m = min(len(ts), len(got.times))
        same_t = bool(np.array_equal(ts[:m], got.times[:m]))
        fs = np.max(np.abs(w["samples"][:m]), axis=0)
        fs[fs == 0] = 1.0
        err = float(np.max(np.abs(got.samples[:m] - w["samples"][:m]) / fs)) if m else None
        r["cpu_baseline"] = {"steps_per_s": round(cpu_sps, 4), "cores": 1, "kind": "reference",
                             "sample": f"first {kk} steps, restated ER loop of the unmodified reference "
                                       f"with the cached factorization"}
        r["speedup_vs_cpu"] = round(r["steps_per_s"] / cpu_sps, 1)
        wd = [w["dims"][w["dims_off"][i]:w["dims_off"][i + 1]].tolist() for i in range(len(w["t"]))]
        r["parity"] = {"shared_samples": int(m), "same_times": same_t, "full_scale_err": err,
                       "tol": 1e-8, "krylov_dims_equal": [list(x) for x in got.krylov_dims[:kk]] == wd[:kk]}
    results.append(r)
    print(json.dumps(r), flush=True)
Path(args.out).parent.mkdir(parents=True, exist_ok=True)
Path(args.out).write_text(json.dumps(results, indent=1))
