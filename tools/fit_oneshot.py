"""Fit the one-shot row (reading OS1) from the rows of harness sweeps that the executor ran
through its one-shot small-message path (GenTree plan, bytes <= 1.5 MiB/(N-1)), and report
its prediction error.

    python tools/fit_oneshot.py SWEEP.jsonl [...] [--timing graph]

Writes profiles/genmodel_fit_oneshot_<timing>.json."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2409_04202_b200 as G  # noqa: E402


def cutoff(n):
    """The one-shot cut-off in effect when the committed round-2 C2 data were measured (then the
    one-shot path took every message up to it; since round 2's cut-off sweep the LL128 path
    takes eligible messages from ar_default_paths' lower floor)."""
    return min(1536 * 1024, (3 << 19) // (n - 1)) // 256 * 256


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("files", nargs="+")
    ap.add_argument("--timing", default="graph")
    a = ap.parse_args()
    rows = []
    for f in a.files:
        rows += [json.loads(l) for l in open(f) if l.startswith("{")]
    ll = [r for r in rows if r.get("timing") == a.timing and r["plan"] == "gentree" and r.get("impl", "ours") == "ours"
          and r["bytes"] <= cutoff(r["n"])]
    fit_rows = [(r["n"], r["bytes"], r["t_mean"]) for r in ll]
    p, sse = G.genmodel_fit_row("oneshot", fit_rows)
    errs = []
    for r in ll:
        pred = G.genmodel_closed_form("oneshot", r["n"], r["bytes"], p)["total"]
        errs.append({"n": r["n"], "bytes": r["bytes"], "measured_s": r["t_mean"], "predicted_s": pred,
                     "rel_err": abs(pred - r["t_mean"]) / r["t_mean"]})
    e = sorted(x["rel_err"] for x in errs)
    out = {"timing": a.timing, "rows": len(errs), "alpha": p.alpha, "beta": p.beta,
           "line_gbs": 1 / p.beta / 1e9 if p.beta > 0 else None, "sse": sse,
           "pred_err_median": e[len(e) // 2], "pred_err_max": e[-1], "points": errs, "sources": a.files}
    json.dump(out, open(os.path.join(ROOT, "profiles", f"genmodel_fit_oneshot_{a.timing}.json"), "w"), indent=1)
    print(json.dumps({k: v for k, v in out.items() if k not in ("points", "sources")}, indent=1))


if __name__ == "__main__":
    main()
