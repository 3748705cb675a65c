"""Fit the NVLS plan row (reading NV1) from harness sweeps and check
GenModel's plan-vs-NVLS choice against the measured winner.

    python tools/fit_nvls.py profiles/round1/c2/sweep_n4_f32_nvls16.jsonl \
        profiles/round1/c2/sweep_n2_f32_nvls16.jsonl [--timing graph] [--min-bytes 2097152] [--install]

Writes profiles/genmodel_fit_nvls_<timing>.json (fit, per-row prediction errors, choice
accuracy); --install also writes profiles/genmodel_params_nvls.json for bench.py."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2409_04202_b200 as G  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("files", nargs="+")
    ap.add_argument("--timing", default="graph")
    ap.add_argument("--min-bytes", type=int, default=1 << 20)
    ap.add_argument("--install", action="store_true")
    a = ap.parse_args()
    rows = []
    for f in a.files:
        rows += [json.loads(l) for l in open(f) if l.startswith("{")]
    rows = [r for r in rows if r.get("timing") == a.timing]
    nv = [r for r in rows if r["plan"] == "nvls"]
    fit_rows = [(r["n"], r["bytes"], r["t_mean"]) for r in nv if r["bytes"] >= a.min_bytes]
    p, sse = G.genmodel_fit_nvls(fit_rows)
    errs = []
    for r in nv:
        pred = G.genmodel_closed_form("nvls", r["n"], r["bytes"], p)["total"]
        errs.append({"n": r["n"], "bytes": r["bytes"], "measured_s": r["t_mean"], "predicted_s": pred,
                     "rel_err": abs(pred - r["t_mean"]) / r["t_mean"]})
    fitted = [e for e in errs if e["bytes"] >= a.min_bytes]
    # plan-vs-NVLS choice: GenTree's plan (P2P params from the C3 fit) vs the NVLS row
    gp = json.load(open(os.path.join(ROOT, "profiles", "genmodel_params.json")))
    pp = G.params(alpha=gp["alpha"], beta=gp["beta"], gamma=gp["gamma"], delta=gp["delta"],
                  epsilon=gp["epsilon"], w_t=gp["w_t"])
    gt = {(r["n"], r["bytes"]): r["t_mean"] for r in rows if r["plan"] == "gentree"}
    choices = []
    for r in nv:
        key = (r["n"], r["bytes"])
        if key not in gt or r["bytes"] < a.min_bytes:   # below: the plan side runs the one-shot path
            continue
        dtype = r.get("dtype", "f32")
        es = 4 if dtype == "f32" else 2
        plan = G.Plan.single_switch(r["n"], r["bytes"] // es, dtype, pp)
        c = plan.choose_nvls(pp, p)
        measured_nvls = r["t_mean"] < gt[key]
        best = min(r["t_mean"], gt[key])
        picked = r["t_mean"] if c["use_nvls"] else gt[key]
        choices.append({"n": r["n"], "bytes": r["bytes"], "use_nvls": c["use_nvls"], "measured_nvls_faster": measured_nvls,
                        "correct": c["use_nvls"] == measured_nvls, "regret": picked / best - 1})
    med = sorted(e["rel_err"] for e in fitted)[len(fitted) // 2]
    out = {"timing": a.timing, "min_bytes": a.min_bytes, "fit_rows": len(fit_rows),
           "alpha": p.alpha, "beta": p.beta, "beta_gbs": 1 / p.beta / 1e9, "sse": sse,
           "pred_err_median": med, "pred_err_max": max(e["rel_err"] for e in fitted),
           "choice_correct": sum(c["correct"] for c in choices), "choice_total": len(choices),
           "choice_max_regret": max((c["regret"] for c in choices), default=0.0),
           "rows": errs, "choices": choices, "sources": a.files}
    path = os.path.join(ROOT, "profiles", f"genmodel_fit_nvls_{a.timing}.json")
    json.dump(out, open(path, "w"), indent=1)
    print(json.dumps({k: v for k, v in out.items() if k not in ("rows", "choices")}, indent=1))
    for c in choices:
        if not c["correct"]:
            print("wrong choice:", c)
    if a.install:
        json.dump({"alpha": p.alpha, "beta": p.beta, "source": os.path.basename(path),
                   "note": "NVLS row T = 2α + (n+1)s/n·β (reading NV1), per byte"},
                  open(os.path.join(ROOT, "profiles", "genmodel_params_nvls.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
