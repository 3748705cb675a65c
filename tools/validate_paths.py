"""GenModel along a sweep of every plan kind, each row predicted on the row of the executor path
that ran it: the one-shot row OS1 and the LL128 row for messages the flag-free
paths take (plans whose RS step is one all-rank reduce per block in one order — CPS, GenTree's
single-switch plan, RB, and Ring / RHD at N = 2 — inside ar_default_paths' ranges), else A6x
with the CPS row (CPS-shaped plans) or the multi-step row (`step_table_row`) — all from the
committed fits, none fitted on the sweep given.

    python tools/validate_paths.py profiles/round2/fit/final_val_n*.jsonl [--stat t_mean]
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2409_04202_b200 as G  # noqa: E402
from tools.fit_report import load, plan_for  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("files", nargs="+")
    ap.add_argument("--stat", choices=["t_mean", "t_med"], default="t_mean")
    ap.add_argument("--min-bytes", type=int, default=2 << 20)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    P = os.path.join(ROOT, "profiles")
    pj = json.load(open(os.path.join(P, "genmodel_params.json")))
    oj = json.load(open(os.path.join(P, "genmodel_fit_oneshot_graph.json")))
    lj = json.load(open(os.path.join(P, "genmodel_fit_ll128_graph.json")))
    gp = G.params(pj["alpha"], pj["beta"], pj["gamma"], pj["delta"], pj["epsilon"], int(pj["w_t"]))
    st = pj.get("step_table_row", pj)
    sp = G.params(st["alpha"], st["beta"], st["gamma"], st["delta"], st["epsilon"], int(st["w_t"]))
    op = G.params(alpha=oj["alpha"], beta=oj["beta"])
    out = []
    for r in load(a.files, "graph"):
        n, b = r["n"], r["bytes"]
        if b < a.min_bytes:
            continue
        paths = G.default_paths(n)
        nrow = lj.get("per_n", {}).get(str(n)) or lj
        lp = G.params(alpha=nrow["alpha"], beta=nrow["beta"])
        plan = plan_for(r["plan"], n, b, r["dtype"])
        flag_free = r["plan"] in ("cps", "gentree", "rb") or n == 2
        if flag_free and paths["ll128_min"] < b <= paths["ll128_max"]:
            t, path = G.genmodel_closed_form("ll128", n, b, lp)["total"], "ll128"
        elif flag_free and b <= paths["oneshot_max"]:
            t, path = G.genmodel_closed_form("oneshot", n, b, op)["total"], "oneshot"
        elif plan.report()[-1]["chosen"] == "cps" or (n == 2 and r["plan"] in ("ring", "rhd")):
            t, path = plan.predict_executed(gp)["total"], "a6x_cps"
        else:
            t, path = plan.predict_executed(sp)["total"], "a6x_steps"
        m = r[a.stat]
        out.append({"plan": r["plan"], "n": n, "bytes": b, "path": path, "measured_s": m, "predicted_s": t,
                    "err": t / m - 1})
    errs = [abs(x["err"]) for x in out]
    by = {}
    for x in out:
        by.setdefault(x["plan"], []).append(abs(x["err"]))
    summ = {"rows": len(out), "stat": a.stat, "median": statistics.median(errs), "max": max(errs),
            "by_plan_max": {k: max(v) for k, v in by.items()},
            "ge_64MiB_max": max(abs(x["err"]) for x in out if x["bytes"] >= 64 << 20),
            "over_10pct": [x for x in out if abs(x["err"]) > 0.10]}
    if a.out:
        json.dump({"summary": summ, "rows": out}, open(a.out, "w"), indent=1)
    print(json.dumps({k: v for k, v in summ.items() if k != "over_10pct"}, indent=1))
    for x in summ["over_10pct"]:
        print(f"  over 10 %: {x['plan']} N={x['n']} {x['bytes'] >> 20} MiB {x['path']} {x['err']:+.1%}")


if __name__ == "__main__":
    main()
