"""Fit the LL128 row (the executor's mid-size two-shot path) from the rows of
harness sweeps that ran through it (GenTree plan, equal 16-byte-aligned blocks, one-shot
cut-off < bytes <= the LL128 maximum), and report its prediction error.

    python tools/fit_ll128.py SWEEP.jsonl [...] [--timing graph] [--max-bytes 16777216]

Writes profiles/genmodel_fit_ll128_<timing>.json."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2409_04202_b200 as G  # noqa: E402


def oneshot_cutoff(n):
    """The one-shot cut-off in effect when the committed round-2 C2 data were measured (then the
    one-shot path took every message up to it; since round 2's cut-off sweep the LL128 path
    takes eligible messages from ar_default_paths' lower floor)."""
    return min(1536 * 1024, (3 << 19) // (n - 1)) // 256 * 256


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("files", nargs="+")
    ap.add_argument("--timing", default="graph")
    ap.add_argument("--max-bytes", type=int, default=16 << 20)
    ap.add_argument("--stat", choices=["t_mean", "t_med"], default="t_mean",
                    help="timing statistic fitted and compared (the paper reports means, P:227; the "
                         "median is robust to a disturbed graph replay)")
    ap.add_argument("--paths", choices=["round2", "current"], default="round2",
                    help="which LL128 range the data were measured with: round2 = (one-shot cut-off, "
                         "--max-bytes]; current = ar_default_paths' (ll128_min, ll128_max]")
    a = ap.parse_args()
    rows = []
    for f in a.files:
        rows += [json.loads(l) for l in open(f) if l.startswith("{")]
    def in_range(n, b):
        if a.paths == "current":
            d = G.default_paths(n)
            return d["ll128_min"] < b <= d["ll128_max"]
        return oneshot_cutoff(n) < b <= a.max_bytes

    # round-2 data: only equal 16-byte-aligned blocks ran the LL128 path; since the kernel's own
    # partition (session 3) every count in range does
    sel = [r for r in rows if r.get("timing") == a.timing and r["plan"] == "gentree" and r.get("impl", "ours") == "ours"
           and in_range(r["n"], r["bytes"]) and (a.paths == "current" or r["bytes"] % (r["n"] * 16) == 0)]
    fit_rows = [(r["n"], r["bytes"], r[a.stat]) for r in sel]
    p, sse = G.genmodel_fit_row("ll128", fit_rows)
    errs = []
    for r in sel:
        pred = G.genmodel_closed_form("ll128", r["n"], r["bytes"], p)["total"]
        errs.append({"n": r["n"], "bytes": r["bytes"], "measured_s": r[a.stat], "predicted_s": pred,
                     "rel_err": abs(pred - r[a.stat]) / r[a.stat]})
    e = sorted(x["rel_err"] for x in errs)
    # held out across the rank count: fit on one N, predict the other
    cross = {}
    ns = sorted({r["n"] for r in sel})
    for fit_n in ns:
        rows_f = [(r["n"], r["bytes"], r[a.stat]) for r in sel if r["n"] == fit_n]
        if len({b for _, b, _ in rows_f}) < 2:
            continue
        pf, _ = G.genmodel_fit_row("ll128", rows_f)
        ev = [abs(G.genmodel_closed_form("ll128", r["n"], r["bytes"], pf)["total"] - r[a.stat]) / r[a.stat]
              for r in sel if r["n"] != fit_n]
        if ev:
            cross[f"fit_n{fit_n}"] = {"alpha": pf.alpha, "beta": pf.beta, "heldout_rows": len(ev),
                                      "heldout_err_median": sorted(ev)[len(ev) // 2], "heldout_err_max": max(ev)}
    # per rank count: the protocol's fixed cost grows with N (a rank waits for the lines of N − 1
    # peers), which one (α, β) pair over all N cannot express; consumers take the row of their N
    # when it was measured (tools/harness.py, tools/predict8.py fall back to the pooled row)
    per_n = {}
    for fn in ns:
        rows_f = [(r["n"], r["bytes"], r[a.stat]) for r in sel if r["n"] == fn]
        if len({b for _, b, _ in rows_f}) < 2:
            continue
        pf, _ = G.genmodel_fit_row("ll128", rows_f)
        ev = sorted(abs(G.genmodel_closed_form("ll128", n_, b_, pf)["total"] - t_) / t_ for n_, b_, t_ in rows_f)
        per_n[str(fn)] = {"alpha": pf.alpha, "beta": pf.beta, "rows": len(rows_f),
                          "err_median": ev[len(ev) // 2], "err_max": ev[-1]}
    out = {"timing": a.timing, "rows": len(errs), "alpha": p.alpha, "beta": p.beta, "per_n": per_n, "cross_n": cross,
           "line_gbs": 1 / p.beta / 1e9 if p.beta > 0 else None, "sse": sse, "max_bytes": a.max_bytes, "paths": a.paths, "stat": a.stat,
           "pred_err_median": e[len(e) // 2], "pred_err_max": e[-1], "points": errs, "sources": a.files}
    json.dump(out, open(os.path.join(ROOT, "profiles", f"genmodel_fit_ll128_{a.timing}.json"), "w"), indent=1)
    print(json.dumps({k: v for k, v in out.items() if k not in ("points", "sources")}, indent=1))


if __name__ == "__main__":
    main()
