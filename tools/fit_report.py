#!/usr/bin/env python
"""Fit GenModel on B200 measurements and report its prediction error on HELD-OUT rows
(the paper fits from CPS benchmarks and predicts other plans, P:530-532,
P:776).

    python tools/fit_report.py --cps cps_*.jsonl --val val_*.jsonl --tag nvlink \
        [--holdout-bytes 268435456] [--install]
    python tools/fit_report.py --shared --cps cps_emu.jsonl --val val_emu8.jsonl --tag emulated \
        [--holdout-n 8] [--install]

NVLink ranks (one per GPU): §3.4's fit — (α, k = 2β+γ, δ, ε, w_t) by the library's
`genmodel_fit` (NNLS per w_t) on the CPS rows — minus the held-out rows (--holdout-bytes: the
bench.py size is never fitted); prediction = `genmodel_predict_executed` (reading A6x, bit-
identical to oracle.genmodel.predict_executed) of the plan the library builds for the row.
Also reported: the (α,β,γ) model fitted on the same rows (P:876's comparison) and GenModel on
the paper's unfused step structure (`genmodel_predict`).

Emulated ranks (all on one GPU, --shared; reading A6e): T = A·α + C·γ + D·δ with the shared
coefficients (every rank's memory traffic through one HBM), (α, γ, δ) by NNLS on the CPS rows
of rank counts below --holdout-n; prediction = `genmodel_predict_executed_shared`.

Every validation row is a plan/size the fit never saw.  Error = |pred − meas| / meas (the
paper's definition).  Writes profiles/genmodel_fit_<tag>.json (+ the params file bench.py
reads with --install).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2409_04202_b200 as G  # noqa: E402
from tools.harness import doc  # noqa: E402


def load(paths, timing):
    rows = []
    for p in paths:
        for line in open(p):
            if line.startswith("{"):
                r = json.loads(line)
                if r.get("timing", timing) == timing and r.get("impl", "ours") == "ours":
                    rows.append(r)
    return rows


_plans = {}


def plan_for(kind, n, nbytes, dtype):
    key = (kind, n, nbytes, dtype)
    if key not in _plans:
        es = 4 if dtype == "f32" else 2
        _plans[key] = G.Plan.from_topology(doc(n), nbytes // es, dtype, None, None if kind == "gentree" else kind)
    return _plans[key]


def summarize(out_rows, key):
    es = [x[key] for x in out_rows]
    by = {}
    for x in out_rows:
        by.setdefault(x["plan"], []).append(x[key])
    return {"median": statistics.median(es) if es else None, "max": max(es) if es else None,
            "by_plan_max": {k: max(v) for k, v in sorted(by.items())},
            "by_plan_median": {k: statistics.median(v) for k, v in sorted(by.items())}}


def fit_nvlink(a, cps, val):
    hold = set(a.holdout_bytes or [])
    rows = [(r["n"], r["bytes"], r["t_mean"]) for r in cps if r["bytes"] >= a.min_bytes and r["bytes"] not in hold]
    nmax = max(n for n, _, _ in rows)
    wt_lo = a.wt_min or 2
    wt_hi = max(wt_lo, a.wt_max or max(2, nmax))
    fit, sse = G.genmodel_fit(rows, wt_lo, wt_hi)
    A = np.array([[2.0, (n - 1) * s / n] for n, s, _ in rows])
    t = np.array([x for _, _, x in rows])
    (alpha3, k3), *_ = np.linalg.lstsq(A, t, rcond=None)
    abc = G.params(max(alpha3, 0.0), 0.0, 0.0, 0.0, 0.0, 1 << 20, combined=max(k3, 0.0))
    out_rows = []
    fit_keys = {(n, s) for n, s, _ in rows}
    # executor-path rows: with --multistep, plans that run as several dependent
    # steps on the step-table kernel get their own (α, β, δ), fitted by NNLS on the A6x
    # coefficients of multi-step rows of rank counts below --holdout-n-nvlink (CPS-shaped
    # plans, e.g. Ring / RHD at N = 2, stay on the CPS row)
    st, st_info, st_keys = None, None, set()
    if a.multistep:
        from scipy.optimize import nnls
        ms = [r for r in load(a.multistep, a.timing) if r["plan"] not in ("cps", "gentree") and r["bytes"] >= a.min_bytes
              and r["n"] < a.holdout_n_nvlink
              and plan_for(r["plan"], r["n"], r["bytes"], r["dtype"]).report()[-1]["chosen"] != "cps"]
        X, tt = [], []
        for r in ms:
            plan = plan_for(r["plan"], r["n"], r["bytes"], r["dtype"])
            X.append([plan.predict_executed(G.params(*u, 0.0, 1 << 20))["total"]
                      for u in ((1.0, 0, 0, 0), (0, 1.0, 0, 0), (0, 0, 0, 1.0))])
            tt.append(r["t_mean"])
        xs, res_s = nnls(np.array(X), np.array(tt))
        st = G.params(xs[0], xs[1], 0.0, xs[2], 0.0, 1 << 20)
        st_keys = {(r["plan"], r["n"], r["bytes"]) for r in ms}
        st_info = {"alpha": xs[0], "beta": xs[1], "gamma": 0.0, "delta": xs[2], "epsilon": 0.0, "w_t": 1 << 20,
                   "fit_rows": len(ms), "fit_plans": sorted({r["plan"] for r in ms}),
                   "n_fit": sorted({r["n"] for r in ms}), "fit_residual": res_s}
    for r in val:
        if r["bytes"] < a.min_bytes:
            continue
        plan = plan_for(r["plan"], r["n"], r["bytes"], r["dtype"])
        on_st = st is not None and plan.report()[-1]["chosen"] != "cps"
        pg = plan.predict_executed(st if on_st else fit)["total"]
        pa = plan.predict_executed(abc)["total"]
        ps = plan.predict(fit)["total"]
        m = r["t_mean"]
        in_fit = r["plan"] in ("cps", "gentree") and (r["n"], r["bytes"]) in fit_keys
        out_rows.append({"plan": r["plan"], "executed": plan.report()[-1]["chosen"], "n": r["n"], "bytes": r["bytes"],
                         "dtype": r["dtype"], "measured_s": m, "genmodel_s": pg, "abc_s": pa,
                         "genmodel_paper_steps_s": ps,
                         "cps_point_in_fit": in_fit or (r["plan"], r["n"], r["bytes"]) in st_keys,
                         "path": "step_table" if on_st else "cps",
                         "err_genmodel": abs(pg - m) / m, "err_abc": abs(pa - m) / m,
                         "err_genmodel_paper_steps": abs(ps - m) / m})
    p = fit.as_dict()
    params = {"alpha": p["alpha"], "beta": p["combined"] / 2 if p["has_combined"] else p["beta"],
              "gamma": 0.0 if p["has_combined"] else p["gamma"], "delta": p["delta"], "epsilon": p["epsilon"],
              "w_t": p["w_t"], "n_max_fit": nmax}
    info = {"fit_rows": len(rows), "params_per_byte": p, "fit_sse": sse,
            "abc_params": {"alpha": abc.alpha, "combined": abc.combined}, "held_out_bytes": sorted(hold)}
    if st_info is not None:
        params["step_table_row"] = st_info
        info["step_table_row"] = st_info
    return params, info, out_rows


def _nnls_shared(rows, stat):
    """(α, γ, δ) by NNLS on T = A·α + C·γ + D·δ, the shared coefficients of each row's plan."""
    from scipy.optimize import nnls
    X, t = [], []
    for r in rows:
        plan = plan_for(r["plan"], r["n"], r["bytes"], r["dtype"])
        # the shared coefficients' A, C, D: read back through unit parameters (bit-exact
        # per-step sums of the library's A6e evaluation)
        ua = plan.predict_executed_shared(G.params(1.0, 0, 0, 0, 0, 1))["latency"]
        uc = plan.predict_executed_shared(G.params(0, 0, 1.0, 0, 0, 1))["compute"]
        ud = plan.predict_executed_shared(G.params(0, 0, 0, 1.0, 0, 1))["memory"]
        X.append([ua, uc, ud])
        t.append(r[stat])
    return nnls(np.array(X), np.array(t))


def fit_shared(a, cps, val):
    rows = [r for r in cps if r["bytes"] >= a.min_bytes and r["n"] < a.holdout_n]
    x, res = _nnls_shared(rows, a.stat)
    gp = G.params(x[0], 0.0, x[1], x[2], 0.0, 1 << 20)
    # executor-path rows (as over NVLink): CPS-shaped plans run on ar_flat_kernel,
    # every multi-step plan on the step-table kernel (static slices, flags between steps) —
    # with --multistep, that kernel gets its own (α, γ, δ), fitted on multi-step rows of rank
    # counts below --holdout-n (never the validated rank count)
    gs, xs, ms_rows = None, None, []
    if a.multistep:
        ms_rows = [r for r in load(a.multistep, a.timing) if r["plan"] not in ("cps", "gentree")
                   and r["bytes"] >= a.min_bytes and r["n"] < a.holdout_n]
        xs, res_s = _nnls_shared(ms_rows, a.stat)
        gs = G.params(xs[0], 0.0, xs[1], xs[2], 0.0, 1 << 20)
    out_rows = []
    for r in val:
        if r["bytes"] < a.min_bytes:
            continue
        plan = plan_for(r["plan"], r["n"], r["bytes"], r["dtype"])
        executed = plan.report()[-1]["chosen"]
        path = "flat" if executed == "cps" or gs is None else "step_table"
        pg = plan.predict_executed_shared(gp if path == "flat" else gs)["total"]
        m = r[a.stat]
        out_rows.append({"plan": r["plan"], "executed": executed, "path": path, "n": r["n"], "bytes": r["bytes"],
                         "dtype": r["dtype"], "measured_s": m, "genmodel_s": pg, "err_genmodel": abs(pg - m) / m})
    params = {"alpha": x[0], "beta": 0.0, "gamma": x[1], "delta": x[2], "epsilon": 0.0, "w_t": 1 << 20,
              "model": "shared (reading A6e)", "n_fit": sorted({r["n"] for r in rows})}
    info = {"fit_rows": len(rows), "params_per_byte": params, "fit_residual": res, "held_out_n": a.holdout_n,
            "stat": a.stat}
    if gs is not None:
        params["step_table_row"] = {"alpha": xs[0], "beta": 0.0, "gamma": xs[1], "delta": xs[2], "epsilon": 0.0,
                                    "w_t": 1 << 20, "fit_rows": len(ms_rows),
                                    "fit_plans": sorted({r["plan"] for r in ms_rows}),
                                    "n_fit": sorted({r["n"] for r in ms_rows}), "fit_residual": res_s}
        info["step_table_row"] = params["step_table_row"]
    return params, info, out_rows


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cps", nargs="+", required=True)
    ap.add_argument("--val", nargs="+", required=True)
    ap.add_argument("--tag", required=True)
    ap.add_argument("--timing", default="graph")
    ap.add_argument("--min-bytes", type=int, default=1 << 20)
    ap.add_argument("--install", action="store_true", help="write the params file bench.py reads")
    ap.add_argument("--fanin", default=None, help="harness fanin JSONL (C3-i, Eq. 6)")
    ap.add_argument("--shared", action="store_true", help="emulated ranks on one GPU (reading A6e)")
    ap.add_argument("--holdout-n", type=int, default=8, help="--shared: fit on rank counts below this")
    ap.add_argument("--multistep", nargs="*", default=None,
                    help="--shared: multi-step rows (e.g. Ring at 3..7 ranks) fitting the step-table kernel's row")
    ap.add_argument("--holdout-n-nvlink", type=int, default=4,
                    help="--multistep over NVLink: fit the step-table row on rank counts below this")
    ap.add_argument("--stat", choices=["t_mean", "t_med"], default="t_mean",
                    help="--shared: timing statistic fitted and compared")
    ap.add_argument("--holdout-bytes", type=int, nargs="*", default=None, help="CPS sizes never fitted")
    ap.add_argument("--wt-min", type=int, default=0, help="incast threshold lower bound (x-to-x probe)")
    ap.add_argument("--wt-max", type=int, default=0)
    a = ap.parse_args()
    eq6 = None
    if a.fanin:
        # Eq. 6: T(x)/(x-1) = a/(x-1) + b with C1 = a/2 = S*delta, C2 = b - a/2 = S*gamma
        fr = [json.loads(x) for x in open(a.fanin) if x.startswith("{")]
        xs = np.array([r["k"] for r in fr], dtype=float)
        ys = np.array([r["t_med"] / (r["k"] - 1) for r in fr])
        S = fr[0]["count"] * (4 if fr[0]["dtype"] == "f32" else 2)
        (aa, bb), *_ = np.linalg.lstsq(np.stack([1 / (xs - 1), np.ones_like(xs)], 1), ys, rcond=None)
        eq6 = {"a_s": aa, "b_s": bb, "C1_s": aa / 2, "C2_s": bb - aa / 2, "vector_bytes": S,
               "delta_per_byte": aa / 2 / S, "gamma_per_byte": (bb - aa / 2) / S,
               "points": [{"x": int(x), "t_per_add_s": float(y)} for x, y in zip(xs, ys)],
               "strictly_decreasing": bool(np.all(np.diff(ys) < 0))}
    cps = [r for r in load(a.cps, a.timing) if r["plan"] == "cps"]
    val = load(a.val, a.timing)
    if a.shared:
        params, info, out_rows = fit_shared(a, cps, val)
    else:
        params, info, out_rows = fit_nvlink(a, cps, val)
    held = [x for x in out_rows if not x.get("cps_point_in_fit")]
    summary = {"tag": a.tag, "timing": a.timing, "model": "shared" if a.shared else "executed", **info,
               "validation_rows": len(held),
               "genmodel_err": summarize(held, "err_genmodel"),
               "genmodel_err_ge_64MiB": summarize([x for x in held if x["bytes"] >= 64 << 20], "err_genmodel"),
               "eq6_local_fanin": eq6, "rows": out_rows}
    if not a.shared:
        summary["abc_err"] = summarize(held, "err_abc")
        summary["genmodel_paper_steps_err"] = summarize(held, "err_genmodel_paper_steps")
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", f"genmodel_fit_{a.tag}.json"), "w") as f:
        json.dump(summary, f, indent=1)
    if a.install:
        name = "genmodel_params_emulated.json" if a.shared else "genmodel_params.json"
        params.update({"source": f"genmodel_fit_{a.tag}.json",
                       "validation": {"rows": len(held), "median": summary["genmodel_err"]["median"],
                                      "max": summary["genmodel_err"]["max"],
                                      "by_plan_max": summary["genmodel_err"]["by_plan_max"],
                                      "ge_64MiB": {k: summary["genmodel_err_ge_64MiB"][k] for k in ("median", "max")}},
                       "note": ("per byte; top level = the CPS-shaped plans' row fitted on CPS rows, step_table_row = "
                                "the multi-step plans' (step-table kernel's) row fitted on multi-step rows of rank "
                                "counts below the validated one; validated on held-out plans/sizes/rank counts" if "step_table_row" in params
                                else "per byte; fitted on CPS rows only, validated on held-out plans/sizes")})
        with open(os.path.join(ROOT, "profiles", name), "w") as f:
            json.dump(params, f, indent=1)
    print(json.dumps({k: v for k, v in summary.items() if k != "rows"}, indent=1))


if __name__ == "__main__":
    main()
