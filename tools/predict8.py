"""GenModel's prediction for configuration C2 at 8 x B200 (the box size this pool cannot lease).

    python tools/predict8.py [--world 8] > profiles/genmodel_predict_n8.json

For every size of the C2 sweep (fp32, 64 KiB - 1 GiB) it asks the library's GenTree for the
plan (fitted NVLink parameters, profiles/genmodel_params.json), predicts the executed plan's time
(`genmodel_predict_executed`, reading A6x) — or the one-shot row (reading OS1) below the
executor's one-shot cut-off 1.5 MiB/(N-1) — and the NVLS row (reading NV1, fitted
profiles/genmodel_params_nvls.json), and converts both to busbw.  The parameters were fitted
on N = 2..4 (median executed-plan error 1.7 %); at N = 8 the numbers are a model prediction,
not a measurement, and say so in the output.  CPU only.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2409_04202_b200 as G  # noqa: E402

P = os.path.join(ROOT, "profiles")


def busbw(nbytes, n, t):
    return nbytes * 2 * (n - 1) / n / t / 1e9


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--world", type=int, default=8)
    a = ap.parse_args()
    n = a.world
    pj = json.load(open(os.path.join(P, "genmodel_params.json")))
    nj = json.load(open(os.path.join(P, "genmodel_params_nvls.json")))
    oj = json.load(open(os.path.join(P, "genmodel_fit_oneshot_graph.json")))
    lj = json.load(open(os.path.join(P, "genmodel_fit_ll128_graph.json")))
    per_n = lj.get("per_n", {})
    if per_n:   # the row fitted at n ranks, else at the largest measured rank count
        lj = dict(lj, **per_n.get(str(n), per_n[max(per_n, key=int)]))
    gp = G.params(pj["alpha"], pj["beta"], pj["gamma"], pj["delta"], pj["epsilon"], pj["w_t"])
    npar = G.params(alpha=nj["alpha"], beta=nj["beta"])
    paths = G.default_paths(n)   # the executor's default path cut-offs (ar_default_paths)
    rows = []
    for k in range(16, 31):
        nbytes = 1 << k
        count = nbytes // 4
        plan = G.Plan.single_switch(n, count, "f32", gp)
        kind = plan.report()[-1]["chosen"]
        op = G.params(alpha=oj["alpha"], beta=oj["beta"])
        lp = G.params(alpha=lj["alpha"], beta=lj["beta"])
        if paths["ll128_min"] < nbytes <= paths["ll128_max"]:
            t_plan = G.genmodel_closed_form("ll128", n, nbytes, lp)["total"]
            path = "LL128 two-shot"
        elif nbytes <= paths["oneshot_max"]:
            t_plan = G.genmodel_closed_form("oneshot", n, nbytes, op)["total"]
            path = "one-shot"
        else:
            t_plan = plan.predict_executed(gp)["total"]
            path = f"{kind} (executed steps)"
        c = plan.choose_nvls(gp, npar)
        doc = json.dumps({"nodes": [{"id": "sw", "kind": "switch", "parent": None, "uplink": None}] + [
            {"id": f"s{i}", "kind": "server", "parent": "sw",
             "uplink": {"alpha": 0, "beta": 1, "epsilon": 0, "w_t": 1}, "compute": {"gamma": 0, "delta": 0}}
            for i in range(n)]})
        pick = G.Plan.from_topology_nvls(doc, count, "f32", gp, npar, op, paths["oneshot_max"], lp,
                                         paths["ll128_max"], paths["ll128_min"])
        t_pick = c["t_nvls"] if pick.switch_reduce else t_plan
        rows.append({"bytes": nbytes, "gentree_plan": kind, "path": path, "t_pred_s": t_plan,
                     "busbw_pred": round(busbw(nbytes, n, t_plan), 1), "t_nvls_pred_s": c["t_nvls"],
                     "nvls_busbw_pred": round(busbw(nbytes, n, c["t_nvls"]), 1),
                     "gentree_incl_nvls_pick": "nvls" if pick.switch_reduce else kind,
                     "pick_busbw_pred": round(busbw(nbytes, n, t_pick), 1)})
    out = {"tool": "predict8", "world": n, "dtype": "f32", "kind": "GenModel prediction, not a measurement",
           "params": pj["source"], "nvls_params": nj["source"], "oneshot_params": "genmodel_fit_oneshot_graph.json",
           "ll128_params": "genmodel_fit_ll128_graph.json (the row of the largest measured rank count)",
           "paths": paths,
           "fit_range": "parameters fitted on CPS rows at N = 2..4 (w_t >= 4, eps = 0: no incast seen up to the 4-GPU lease)",
           "context": "NCCL 8-rank all-reduce busbw 725 GB/s at 1 GiB on B200 (B200_PROFILING.md)",
           "rows": rows}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
