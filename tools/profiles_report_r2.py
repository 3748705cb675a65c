"""Regenerate profiles/round2/README.md from the round-2 evidence files under profiles/round2/.

    python tools/profiles_report_r2.py > profiles/round2/README.md

Every number comes from a file committed next to it (bench lines, harness JSONL sweeps, fit
reports, ncu summaries)."""
import glob
import json
import os
import sys
import statistics

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
P = os.path.join(ROOT, "profiles", "round2")


def jl(path):
    if not os.path.exists(path):
        return []
    with open(path) as f:
        return [json.loads(l) for l in f if l.startswith("{")]


def jload(path):
    rows = jl(path)
    return rows[0] if rows else None


def size(b):
    for shift, unit in ((30, "GiB"), (20, "MiB"), (10, "KiB")):
        if b >= 1 << shift:
            return f"{b / (1 << shift):g} {unit}"
    return f"{b} B"


def bench_section(out):
    out.append("## 1. bench.py lines\n")
    out.append("| file | GPUs | dtype | plan | kernel | busbw GB/s | roofline | NCCL default / Ring / NVLS-off | ours ÷ NCCL (default, Ring, NVLS-off) | NVLS kind | GenModel pred. err (held out) |")
    out.append("|---|---|---|---|---|---|---|---|---|---|---|")
    for f in sorted(glob.glob(os.path.join(P, "bench_*.json"))):
        d = jload(f)
        if not d or "value" not in d or d.get("impl") == "reference":
            continue
        rf = d["roofline"]
        nc = d.get("nccl") or {}
        ncs = " / ".join(str(nc.get(k, {}).get("busbw", "-")) for k in ("default", "ring", "nvls_off")) if nc else "-"
        vs = d.get("vs_nccl") or {}
        vss = ", ".join(f"{vs[k]:.3f}" for k in ("default", "ring", "nvls_off") if k in vs) or "-"
        roof = f"{rf['bound']} {rf['achieved']} / {rf['peak']} = {rf['frac']}"
        if "frac_wire_ceiling" in rf:
            roof += f"; {rf['frac_wire_ceiling']} of the {rf['wire_user_ceiling']} wire ceiling"
        nv = (d.get("nvls") or {}).get("busbw", "-")
        out.append(f"| `{os.path.basename(f)}` | {d['n_gpus']} | {d['dtype']} | {d['config']['plan']} | "
                   f"`{rf.get('kernel')}` | {d['value']} | {roof} | {ncs} | {vss} | {nv} | "
                   f"{d.get('genmodel', {}).get('pred_err', '-')} |")
    out.append("")


def nccl_algo_section(out):
    logs = sorted(glob.glob(os.path.join(P, "nccl", "nccl_tuning*.log")))
    if not logs:
        return
    out.append("## 2b. NCCL's algorithm choice (NCCL_DEBUG_SUBSYS=TUNING, default env, 4 GPUs, fp32)\n")
    seen = {}
    for f in logs[:1]:
        for line in open(f):
            if "Algo" in line and "Bytes" in line:
                try:
                    tail = line.split("AllReduce:")[1].strip()
                except IndexError:
                    continue
                nb = int(tail.split()[0])
                seen.setdefault(nb, tail)
    out.append("| bytes | NCCL's line |")
    out.append("|---|---|")
    for nb in sorted(seen):
        out.append(f"| {size(nb)} | `{seen[nb][:110]}` |")
    out.append("")


def final_c2(n, dt):
    """The latest C2 run of the final executor: `r3_c2_*` (session 3's final build: re-tuned path
    cut-offs, LL128 for any count; `r3a_c2_*` is the same sweep on the build before the ragged
    LL128 change, which the LL128 row was fitted on), else `final_c2_*`."""
    return (jl(os.path.join(P, "c2", f"r3_c2_n{n}_{dt}.jsonl")) or
            jl(os.path.join(P, "c2", f"final_c2_n{n}_{dt}.jsonl")))


def c2_section(out):
    out.append("## 2. C2: fp32 busbw vs size — GenTree, GenTree incl. NVLS (path-aware min-GenModel pick), NCCL default / Ring / NVLS-off\n")
    out.append("Our columns and NCCL default: the final executor (`r3_c2_*`: LL128 two-shot (CPS-shaped plans; equal"
               " 16-byte-aligned blocks when measured, any count since) from 768 KiB/(N−1) (≤ 384 KiB) to 64 MiB/N, one-shot otherwise up to 1.5 MiB/(N−1), step-table"
               " kernel above — §12); NCCL Ring / NVLS-off: separate processes with the variable set"
               " (`c2_*_ncclring`, `c2_*_ncclnvlsoff`).  Earlier runs: `final_c2_*` (LL128 only above the one-shot"
               " cut-off, to 16 MiB), `c2_n*_f32.jsonl` (before the LL128 path).\n")
    for n in (4, 3, 2):
        ours = final_c2(n, "f32") or jl(os.path.join(P, "c2", f"c2_n{n}_f32.jsonl"))
        if not ours:
            continue
        ring = jl(os.path.join(P, "c2", f"c2_n{n}_f32_ncclring.jsonl"))
        off = jl(os.path.join(P, "c2", f"c2_n{n}_f32_ncclnvlsoff.jsonl"))
        for timing in ("graph", "eager"):
            def get(rows, impl, plan):
                return {r["bytes"]: r for r in rows if r.get("timing") == timing and r["impl"] == impl
                        and r["plan"] == plan}
            g = get(ours, "ours", "gentree")
            gn = get(ours, "ours", "gentree+nvls")
            nv = get(ours, "ours", "nvls")
            nd = get(ours, "nccl", "default")
            nr = get(ring, "nccl", "Ring")
            no = get(off, "nccl", "nvls_off")
            if not g:
                continue
            out.append(f"**{n} × B200, fp32, {timing} timing** (busbw GB/s, median)\n")
            out.append("| size | GenTree | GenTree incl. NVLS (pick) | NVLS | NCCL default | NCCL Ring | NCCL NVLS-off | GenTree ÷ NCCL Ring | pick ÷ best NCCL |")
            out.append("|---|---|---|---|---|---|---|---|---|")
            for b in sorted(g):
                def v(d):
                    return d[b]["busbw_med"] if b in d else float("nan")
                pick = f"{v(gn):.1f} ({gn[b]['chosen']})" if b in gn else "-"
                best = max(x for x in (v(nd), v(nr), v(no)) if x == x) if any(b in d for d in (nd, nr, no)) else float("nan")
                f1 = lambda x: f"{x:.1f}" if x == x else "-"
                f2 = lambda x: f"{x:.2f}" if x == x else "-"
                out.append(f"| {size(b)} | {f1(v(g))} | {pick} | {f1(v(nv))} | {f1(v(nd))} | {f1(v(nr))} | {f1(v(no))} | "
                           f"{f2(v(g) / v(nr))} | {f2((v(gn) / best) if b in gn else float('nan'))} |")
            out.append("")


def bf16_section(out):
    ns = [n for n in (4, 3, 2) if final_c2(n, "bf16")]
    if not ns:
        return
    out.append("**bf16, graph timing, final executor: GenTree plan vs NCCL default (busbw GB/s)**\n")
    out.append("| size | " + " | ".join(f"GenTree N={n} | NCCL N={n} | ratio" for n in ns) + " |")
    out.append("|---|" + "---|---|---|" * len(ns))
    d = {}
    for n in ns:
        rows = final_c2(n, "bf16")
        d[n] = ({r["bytes"]: r["busbw_med"] for r in rows if r["impl"] == "ours"},
                {r["bytes"]: r["busbw_med"] for r in rows if r["impl"] == "nccl"})
    for b in sorted(d[ns[0]][0]):
        cells = []
        for n in ns:
            g, c = d[n]
            cells += [f"{g.get(b, float('nan')):.1f}", f"{c.get(b, float('nan')):.1f}", f"{g.get(b, float('nan')) / c.get(b, float('nan')):.2f}"]
        out.append(f"| {size(b)} | " + " | ".join(cells) + " |")
    out.append("")


def pick_section(out):
    """The final build's "GenTree incl. NVLS" column: the min-GenModel pick with the plan side
    predicted on the row of the path the executor takes (gentree_plan_nvls with the OS1 and
    LL128 rows)."""
    for n in (4, 3, 2):
        final = final_c2(n, "f32")
        pk = [r for r in final if r.get("plan") == "gentree+nvls"] or jl(os.path.join(P, "c2", f"c2pick_n{n}_f32.jsonl"))
        base = final or jl(os.path.join(P, "c2", f"c2_n{n}_f32.jsonl"))
        ring = jl(os.path.join(P, "c2", f"c2_n{n}_f32_ncclring.jsonl"))
        if not pk:
            continue
        g = {r["bytes"]: r for r in base if r.get("timing") == "graph" and r["impl"] == "ours" and r["plan"] == "gentree"}
        nv = {r["bytes"]: r for r in base if r.get("timing") == "graph" and r["impl"] == "ours" and r["plan"] == "nvls"}
        nr = {r["bytes"]: r for r in ring if r.get("timing") == "graph" and r["impl"] == "nccl"}
        p = {r["bytes"]: r for r in pk if r.get("timing") == "graph" and r.get("impl", "ours") == "ours"}
        out.append(f"**{n} × B200, fp32, graph timing: GenTree incl. NVLS, the plan side predicted on the path the executor takes (one-shot / LL128 / steps)**\n")
        out.append("| size | pick | pick busbw | GenTree busbw | NVLS busbw | best of the two | pick ÷ best | pick ÷ NCCL Ring |")
        out.append("|---|---|---|---|---|---|---|---|")
        for b in sorted(p):
            best = max(g[b]["busbw_med"], nv[b]["busbw_med"]) if b in g and b in nv else float("nan")
            out.append(f"| {size(b)} | {p[b]['chosen']} | {p[b]['busbw_med']:.1f} | {g[b]['busbw_med'] if b in g else float('nan'):.1f} | "
                       f"{nv[b]['busbw_med'] if b in nv else float('nan'):.1f} | {best:.1f} | {p[b]['busbw_med'] / best:.3f} | "
                       f"{p[b]['busbw_med'] / nr[b]['busbw_med'] if b in nr else float('nan'):.2f} |")
        out.append("")


def fit_section(out):
    for tag, title in (("nvlink_r2", "NVLink ranks (one per GPU), N = 2..4"),
                       ("emulated8_shared", "8 ranks emulated on one GPU (shared HBM, reading A6e)")):
        f = os.path.join(ROOT, "profiles", f"genmodel_fit_{tag}.json")
        if not os.path.exists(f):
            continue
        d = json.load(open(f))
        ge = d["genmodel_err"]
        out.append(f"### GenModel, {title} — `profiles/genmodel_fit_{tag}.json`\n")
        out.append(f"* fit rows (CPS only): {d['fit_rows']}; held-out validation rows: {d['validation_rows']}")
        pp = d["params_per_byte"]
        out.append(f"* params per byte: " + ", ".join(f"{k} = {pp[k]:.4g}" for k in ("alpha", "beta", "gamma", "delta",
                                                                                      "epsilon", "combined")
                                                        if k in pp and isinstance(pp[k], float)) +
                   (f", w_t = {pp['w_t']}" if "w_t" in pp else ""))
        out.append(f"* held-out error: median {ge['median']:.3f}, max {ge['max']:.3f}")
        out.append("")
        out.append("| plan | median | max |")
        out.append("|---|---|---|")
        for k in ge["by_plan_max"]:
            out.append(f"| {k} | {ge['by_plan_median'][k]:.3f} | {ge['by_plan_max'][k]:.3f} |")
        if "abc_err" in d:
            out.append("")
            out.append(f"(α,β,γ) model on the same rows: median {d['abc_err']['median']:.3f}, max {d['abc_err']['max']:.3f}; "
                       f"GenModel on the paper's unfused steps: median {d['genmodel_paper_steps_err']['median']:.3f}, "
                       f"max {d['genmodel_paper_steps_err']['max']:.3f}.")
        out.append("")


def ll128_section(out):
    d = os.path.join(P, "ll128")
    if not os.path.isdir(d):
        return
    out.append("## 2c. LL128 two-shot path vs the step-table kernel (CPS plan, fp32, graph timing, busbw GB/s)\n")
    out.append("`off` = AR_LL128_MAX_KB=0 (flag protocol); `cN` = the LL128 path with N CTAs (148 = one per SM,"
               " the default); 512 KiB at N = 4 and ≤ 1 MiB at N = 2 run the one-shot path in every column.\n")
    for n in (4, 2):
        def load(f):
            return {r["bytes"]: r for r in jl(os.path.join(d, f)) if r.get("timing") == "graph" and r.get("impl") == "ours"}
        off = load(f"off_n{n}.jsonl")
        cs = {c: load(f"on_n{n}_c{c}.jsonl") for c in (32, 64, 148)}
        c296 = {r["bytes"]: r for r in jl(os.path.join(P, "c2", f"ll296_n{n}.jsonl")) if r.get("timing") == "graph"}
        if not off:
            continue
        out.append(f"**{n} × B200**\n")
        out.append("| size | off | c32 | c64 | c148 | c296 | c148 ÷ off |")
        out.append("|---|---|---|---|---|---|---|")
        for b in sorted(off):
            v = [off[b]["busbw_med"]] + [cs[c][b]["busbw_med"] if b in cs[c] else float("nan") for c in (32, 64, 148)]
            v.append(c296[b]["busbw_med"] if b in c296 else float("nan"))
            out.append(f"| {size(b)} | " + " | ".join(f"{x:.1f}" for x in v) + f" | {v[3] / v[0]:.2f} |")
        out.append("")


def push_section(out):
    rows = []
    for n in (2, 4):
        pu = {r["bytes"]: r for r in jl(os.path.join(P, "push", f"pull_n{n}.jsonl"))}
        ps = {r["bytes"]: r for r in jl(os.path.join(P, "push", f"push_n{n}.jsonl"))}
        for b in sorted(pu):
            if b in ps:
                rows.append((n, b, pu[b]["busbw_med"], ps[b]["busbw_med"]))
    if not rows:
        return
    out.append("## 4. Write-only (push) protocol vs pull → add → push, bf16, graph timing\n")
    out.append("| GPUs | size | pull (default) busbw | push (AR_PUSH_MAX_MB) busbw | push ÷ pull |")
    out.append("|---|---|---|---|---|")
    for n, b, a, c in rows:
        out.append(f"| {n} | {size(b)} | {a:.1f} | {c:.1f} | {c / a:.3f} |")
    out.append("")


def fence_section(out):
    a = {(r["bytes"], r["timing"]): r for r in jl(os.path.join(P, "latency", "fence0_n4.jsonl"))}
    b = {(r["bytes"], r["timing"]): r for r in jl(os.path.join(P, "latency", "fence1_n4.jsonl"))}
    if not a:
        return
    out.append("## 5. Entry-flag ordering: relaxed (default) vs fence.acq_rel.sys first (AR_ENTRY_FENCE=1), 4 GPUs, fp32, one-shot path off\n")
    out.append("| size | timing | relaxed µs | fenced µs | fenced ÷ relaxed |")
    out.append("|---|---|---|---|---|")
    for k in sorted(a):
        if k in b:
            out.append(f"| {size(k[0])} | {k[1]} | {a[k]['t_med'] * 1e6:.1f} | {b[k]['t_med'] * 1e6:.1f} | "
                       f"{b[k]['t_med'] / a[k]['t_med']:.3f} |")
    out.append("")


def p2p_section(out):
    rows = jl(os.path.join(P, "c3", "p2p_n4.jsonl"))
    if not rows:
        return
    out.append("## 6. C3-ii: x-to-x and x-to-1 fan-in over NVLink (4 × B200, fp32; P:418-428)\n")
    out.append("| receiver bytes | pattern | x | µs (median) | GB/s per receiver |")
    out.append("|---|---|---|---|---|")
    for r in rows:
        out.append(f"| {size(r['recv_bytes'])} | {r['pattern']} | {r['x']} | {r['t_med'] * 1e6:.1f} | {r['gbs_per_receiver']:.1f} |")
    out.append("")


def fanin_ag_section(out):
    rows = jl(os.path.join(P, "c3", "fanin_ag.jsonl"))
    if not rows:
        return
    out.append("## 7. C3-iv: Eq. 6 local fan-in alone and under an incoming NVLink AllGather stream\n")
    out.append("| x | T alone µs | T with AG µs | HBM GB/s alone | HBM GB/s with AG | AG GB/s alone | AG GB/s during | slowdown |")
    out.append("|---|---|---|---|---|---|---|---|")
    for r in rows:
        out.append(f"| {r['k']} | {r['t_med_alone'] * 1e6:.1f} | {r['t_med_with_ag'] * 1e6:.1f} | {r['hbm_gbs_alone']:.0f} | "
                   f"{r['hbm_gbs_with_ag']:.0f} | {r['ag_gbs_alone']:.0f} | {r['ag_gbs_during']:.0f} | "
                   f"{r['t_med_with_ag'] / r['t_med_alone']:.3f} |")
    out.append("")


def cpu_section(out):
    rows = jl(os.path.join(P, "cpu_oracle_timing.jsonl"))
    if not rows:
        return
    out.append("## 8. CPU oracle timing plan (SURVEY §8(d)), one pinned core of the GPU box's host\n")
    r0 = rows[0]
    out.append(f"Host: {r0['cpu_model']}, os.cpu_count() = {r0['cpu_count']}, pinned to core {r0['pinned_core']}.\n")
    out.append("| config | ranks | size/rank | dtype | plan build s | simulate s | oracle busbw GB/s |")
    out.append("|---|---|---|---|---|---|---|")
    for r in rows:
        out.append(f"| {r['config']} | {r['ranks']} | {size(r['bytes_per_rank'])} | {r['dtype']} | {r['t_plan_s']:.3f} | "
                   f"{r['t_simulate_s']:.2f} | {r['oracle_busbw_gbs']:.3f} |")
    out.append("")


def nvls_sweep_section(out):
    import glob
    files = sorted(glob.glob(os.path.join(P, "nvls_sweep", "sw_*_f32.jsonl")))
    if not files:
        return
    out.append("## 9. NVLS kernel: vectors in flight per thread (AR_NVLS_U) × CTAs, fp32, graph timing (busbw GB/s)\n")
    out.append("`nvls_sweep/`: `AR_NVLS_U=u AR_NVLS_CTAS=c T --nproc-per-node N tools/harness.py sweep --dtype f32 "
               "--plans nvls --no-nccl --timing graph --sizes 16 MiB 256 MiB 1 GiB`.\n")
    out.append("| N | U | CTAs | 16 MiB | 256 MiB | 1 GiB |")
    out.append("|---|---|---|---|---|---|")
    rows = []
    for f in files:
        tag = os.path.basename(f)[3:-len("_f32.jsonl")]          # n4_u8_c16
        n, u, c = (int(x[1:]) for x in tag.split("_"))
        d = {r["bytes"]: r["busbw_med"] for r in jl(f)}
        rows.append((n, u, c, d))
    for n, u, c, d in sorted(rows, key=lambda r: (-r[0], r[1], r[2])):
        out.append(f"| {n} | {u} | {c} | " + " | ".join(f"{d.get(b, float('nan')):.1f}" for b in (16 << 20, 256 << 20, 1 << 30)) + " |")
    out.append("")
    out.append("Once ≥ 16 CTAs × 4 vectors per thread are in flight the kernel saturates at ≈ 672–677 GB/s busbw "
               "(256 MiB) and ≈ 685–692 (1 GiB) on 4 GPUs, ≈ 400–411 on 2, whatever the split: the limit is not "
               "request concurrency.  U stays 4, CTAs 16 (N ≥ 3) / 32 (N = 2).\n")


def nvls_bf16_section(out):
    rows = jl(os.path.join(P, "nvls_bf16", "fit.jsonl"))
    if not rows:
        return
    out.append("## 10. What the switch does to a bf16 multimem.ld_reduce (reading NV2)\n")
    out.append("`nvls_bf16/fit.jsonl`: `T --nproc-per-node N tools/nvls_dump.py` (GPU; 1 Mi elements, gradient-shaped "
               "and adversarial inputs, acc::f32 and bf16 accumulation) then `python tools/nvls_bf16_fit.py` (CPU; "
               "first 200 000 elements, P(away) over the first 60 000).  The two accumulation modes return identical "
               "bits.  Best deterministic rounding hypotheses (of ~30) and how often the switch rounds AWAY from zero "
               "by where the exact sum lies between its two bf16 neighbours:\n")
    out.append("| N | data | best hypotheses (match) | inexact sums | P(away) by fraction bin | ties: P(away) |")
    out.append("|---|---|---|---|---|---|")
    for r in rows:
        if not r["case"].startswith("f32_"):
            continue
        best = ", ".join(f"{k} ({v:.4f})" for k, v in r["best"][:2])
        pa = r["p_away_by_frac"]
        bins = "; ".join(f"[{b['frac'][0]:.3g},{b['frac'][1]:.3g}) {b['p_away']:.3f}" for b in pa["bins"])
        ties = pa["ties"]
        out.append(f"| {r['world']} | {r['case'][4:]} | {best} | {pa['inexact']} | {bins or '-'} | "
                   f"{ties['p_away'] if ties['n'] else '-'} (n={ties['n']}) |")
    out.append("")
    out.append("A round-to-nearest unit would give P(away) = 0 below 1/2 and 1 above; the switch's P(away) rises "
               "with the fraction — a stochastic rounding (repeatable over calls), with no dependence on the "
               "element's index bits.  No deterministic rule of the sum reproduces it, so bf16 NVLS is checked "
               "against the 1e-2 norm-wise bound only and never enters GenTree as a bit-exact kind; fp32 NVLS "
               "(correctly rounded) does.\n")


def split_section(out):
    import glob
    files = sorted(glob.glob(os.path.join(P, "split", "split_*.jsonl")))
    if not files:
        return
    out.append("## 11. NVLS and the P2P executor side by side on one message (fp32, `tools/nvls_p2p_split.py`)\n")
    out.append("The first x·S bytes through the NVLS kernel (16 CTAs, or 8 with U = 8), the rest through the GenTree "
               "(CPS) plan on the P2P executor with 148 − NVLS CTAs, concurrently on two streams; busbw of the whole "
               "S (eager events, max over ranks, median of 20).\n")
    out.append("| run | size | " + " | ".join(f"x = {x:g}" for x in (0, 0.2, 0.3, 0.4, 0.5, 0.6, 0.7, 1)) + " |")
    out.append("|---|---|" + "---|" * 8)
    for f in files:
        rows = jl(f)
        for b in sorted({r["bytes"] for r in rows}):
            d = {r["nvls_share"]: r["busbw_med"] for r in rows if r["bytes"] == b}
            out.append(f"| {os.path.basename(f)[:-6]} (N={rows[0]['n']}) | {size(b)} | " +
                       " | ".join(f"{d[x]:.1f}" if x in d else "-" for x in (0, 0.2, 0.3, 0.4, 0.5, 0.6, 0.7, 1)) + " |")
    out.append("")
    out.append("No split passes the better single path by more than 2 % (4 GPUs, x = 0.2: 677 vs 665 at 256 MiB, "
               "701 vs 687 at 1 GiB; every other share 655–690): the two kernels share one resource, the NVLink wire.  With the P2P path at "
               "0.97 of its 682 GB/s wire ceiling (DESIGN §7) and NVLS saturated at the same busbw (§9), 720 GB/s "
               "(80 % of 900) is out of reach at N ≤ 4; NVLS's per-GPU wire volume falls to (1 + 1/N)·S at N = 8, "
               "where the fitted row predicts it above 720 (profiles/README.md §11).\n")


def cut_section(out):
    d = os.path.join(P, "cut")
    if not os.path.isdir(d):
        return
    out.append("## 12. Path cut-offs with the LL128 path in place (GenTree = CPS plan, graph timing; µs per call)\n")
    out.append("`cut/def_*`: the cut-offs of the round-2 build (one-shot to 1.5 MiB/(N−1), LL128 above it to 16 MiB); "
               "`cut/ll128all_*`: `AR_LL_MAX_KB=0 AR_LL128_MAX_KB=65536` (LL128 for every eligible size).  Sizes are "
               "LL128-eligible (equal 16-byte-aligned blocks).  ★ = the faster by more than 2 %; the new defaults "
               "(ar_default_paths: LL128 from 768 KiB/(N−1), at most 384 KiB, to 64 MiB/N) follow the ★s.\n")
    for n in (4, 2):
        for dt in ("f32", "bf16"):
            a = {r["bytes"]: r for r in jl(os.path.join(d, f"def_n{n}_{dt}.jsonl"))}
            b = {r["bytes"]: r for r in jl(os.path.join(d, f"ll128all_n{n}_{dt}.jsonl"))}
            if not a or not b:
                continue
            out.append(f"**N = {n}, {dt}**\n")
            out.append("| size | round-2 paths µs (busbw) | LL128 µs (busbw) |")
            out.append("|---|---|---|")
            for k in sorted(a):
                ta, tb = a[k]["t_med"] * 1e6, b[k]["t_med"] * 1e6
                sa = " ★" if ta * 1.02 < tb else ""
                sb = " ★" if tb * 1.02 < ta else ""
                out.append(f"| {size(k)} | {ta:.1f} ({a[k]['busbw_med']:.0f}){sa} | {tb:.1f} ({b[k]['busbw_med']:.0f}){sb} |")
            out.append("")


def llsplit_section(out):
    import glob
    files = sorted(glob.glob(os.path.join(P, "llsplit", "b_n*.jsonl")))
    if not files:
        return
    out.append("## 13. One CPS message split between the LL128 and the step-table kernel (fp32, `tools/ll128_exec_split.py`)\n")
    out.append("The first x·S bytes through the LL128 kernel (AR_LL128_MAX_KB=262144), the rest (one element short of "
               "equal blocks) through the step-table kernel with 100 CTAs (`SPLIT_EXEC_CTAS=100`; LL128 then gets ≤ 300), "
               "concurrently on two streams; x = 0 and 1 are the LL128 kernel alone.  With the step-table kernel at "
               "148 CTAs both kernels cannot be resident together and the run deadlocks into the flag timeout (a "
               "resident LL128 CTA waits for a peer's unscheduled one) — the same residency rule the LL128 path "
               "already enforces.  busbw GB/s:\n")
    shares = (0, 0.1, 0.2, 0.3, 0.4, 0.5, 1)
    out.append("| N | size | " + " | ".join(f"x = {x:g}" for x in shares) + " | C2 (r3, default paths) |")
    out.append("|---|---|" + "---|" * (len(shares) + 1))
    for f in files:
        rows = jl(f)
        n = rows[0]["n"]
        c2 = {r["bytes"]: r["busbw_med"] for r in final_c2(n, "f32")
              if r.get("timing") == "graph" and r["impl"] == "ours" and r["plan"] == "gentree"}
        for b in sorted({r["bytes"] for r in rows}):
            d = {r["ll128_share"]: r["busbw_med"] for r in rows if r["bytes"] == b}
            out.append(f"| {n} | {size(b)} | " + " | ".join(f"{d[x]:.0f}" if x in d else "-" for x in shares) +
                       f" | {c2.get(b, float('nan')):.0f} |")
    out.append("")
    out.append("No split beats the default path (the step-table kernel at 148 CTAs above the LL128 ceiling): the "
               "LL128 kernel alone falls to ≈ 390–520 GB/s from 64 MiB (its 128-byte lines pass through the "
               "owner's HBM scratch), and the step-table kernel's fixed per-call cost is already small against "
               "these sizes.  Not adopted.\n")


def simu_baselines_section(out):
    """Desk analysis of tab:gentreesimu: each baseline is one fixed plan, so its
    time is affine in S; the intercept is its latency term."""
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from tools.gentreesimu import PAPER
    a = 6.58e-3
    out.append("## 14. What tab:gentreesimu's rows fix (desk analysis of the printed table, P:1144-1190)\n")
    out.append("Every baseline is one fixed plan, so its time is affine in S: T = A + K·S.  Fitted through the "
               "1e7 and 1e8 points, each baseline predicts its printed 3.2e7 point to ±0.1 %, and A is an exact "
               "multiple of the printed α = 6.58e-3 s (CDC384: of α_cross = 3e-2 plus 4α):\n")
    out.append("| topology | plan | A (s) | A / α | K (s per float) | 3.2e7: affine vs printed |")
    out.append("|---|---|---|---|---|---|")
    for topo, rows in PAPER.items():
        for alg, (t1, t2, t3) in rows.items():
            k = (t3 - t1) / 9e7
            aa = t1 - k * 1e7
            out.append(f"| {topo} | {alg} | {aa:.4f} | {aa / a:.2f} | {k:.4e} | {(aa + k * 3.2e7) / t2 - 1:+.2%} |")
    out.append("")
    out.append("Readings: (i) on one switch every step costs 3α (CPS 2 steps → 6α, RHD(32) 10 steps → 30α) — "
               "reading Q16's α_eff = 3α — but Ring costs 2N steps (144α at N = 24, 192α at 32), two more than "
               "2(N−1): the 4 % by which the flow simulator's Ring rows sit low (§7 of ../README.md) is exactly "
               "2 × 3α; (ii) on the two-level trees a step costs 5α (CPS 10α; Ring 400α = 80 × 5α on SYM384 and "
               "ASY384, 480α = 96 × 5α on SYM512, i.e. (2·24 + 2·16) and (2·32 + 2·16) steps of a per-switch "
               "ring) and on CDC384 α_cross + 4α = 0.0563 s (CPS 2 steps, Ring 80 steps): the paper charges "
               "every step the α summed along the tree's longest server-to-server path, whatever the step's "
               "own path; (iii) GenTree's rows are not affine (its plan changes with S).  The slopes K are not "
               "reproduced by the readings checked (the flow simulator's flat and per-switch baselines, and by "
               "hand for flat CPS on SYM384: incast counted per flow, per source or per receiver, max-min or "
               "summed over hops): e.g. flat CPS on SYM384 is 2.2e-7 s/float printed against ≈ 1.05e-7 for "
               "incast-bound max-min on the server links — the "
               "unreleased simulator's bandwidth model for multi-level trees stays unknown, so the hierarchical "
               "rows remain reported, not pinned.\n")


def c2_genmodel_section(out):
    """GenModel's prediction of the GenTree plan along the C2 sweep, on the row of the path the
    executor takes (the committed fits)."""
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    try:
        import paper_2409_04202_b200 as G
    except Exception:
        return
    F = os.path.dirname(P)
    try:
        pj, oj, lj = (json.load(open(os.path.join(F, x))) for x in
                      ("genmodel_params.json", "genmodel_fit_oneshot_graph.json", "genmodel_fit_ll128_graph.json"))
    except (OSError, ValueError):
        return
    gp = G.params(pj["alpha"], pj["beta"], pj["gamma"], pj["delta"], pj["epsilon"], int(pj["w_t"]))
    op = G.params(alpha=oj["alpha"], beta=oj["beta"])
    out.append("## 15. GenModel prediction error of the GenTree plan along the C2 sweep (`r3_c2_*`, graph timing)\n")
    out.append("Each size is predicted on the row of the path the executor takes (ar_default_paths): the LL128 row "
               f"(`genmodel_fit_ll128_graph.json`, per rank count, fitted on the fp32 medians of the previous run "
               "`r3a_c2_*` — held out here), the one-shot row OS1 (round-2 fit, held out) or the executed-plan model "
               "A6x (CPS fit, `genmodel_params.json`, held out).  Error = (predicted − measured median) / measured; "
               "path: o = one-shot, l = LL128, a = A6x.\n")
    for n in (4, 2):
        paths = G.default_paths(n)
        row = lj.get("per_n", {}).get(str(n), lj)
        lp = G.params(alpha=row["alpha"], beta=row["beta"])
        for dt in ("f32", "bf16"):
            es = 4 if dt == "f32" else 2
            rows = [r for r in final_c2(n, dt) if r.get("timing") == "graph" and r["impl"] == "ours"
                    and r["plan"] == "gentree"]
            if not rows:
                continue
            cells, errs = [], []
            for r in sorted(rows, key=lambda r: r["bytes"]):
                b = r["bytes"]
                c = b // es
                if paths["ll128_min"] < b <= paths["ll128_max"]:
                    t, tag = G.genmodel_closed_form("ll128", n, b, lp)["total"], "l"
                elif b <= paths["oneshot_max"]:
                    t, tag = G.genmodel_closed_form("oneshot", n, b, op)["total"], "o"
                else:
                    t, tag = G.Plan.single_switch(n, c, dt, gp).predict_executed(gp)["total"], "a"
                e = t / r["t_med"] - 1
                errs.append(abs(e))
                cells.append(f"{size(b)} {tag} {e:+.0%}")
            e = sorted(errs)
            out.append(f"* N = {n}, {dt}: median {e[len(e) // 2]:.1%}, max {e[-1]:.1%} — " + "; ".join(cells))
    out.append("")
    out.append("Every A6x row (≥ 32 MiB) is within 2.3 %.  The largest errors are the LL128 row's: its affine "
               "α + B·β bends around the measured curve — under at its floor (512 KiB: −16 … −20 %, 1 MiB −7 … −13 %, "
               "where the fixed cost dominates) and over at 4–8 MiB on 2 GPUs (+3 … +9 %: without entry or exit barriers, "
               "back-to-back calls overlap across ranks in the graph replay, so per-call times there imply "
               "per-byte rates above the link's) — and the one-shot row at 256 KiB on 4 GPUs (+8 … +10 %).\n")


def ragged_section(out):
    d = os.path.join(P, "ragged")
    if not os.path.isdir(d):
        return

    def get(f, impl="ours"):
        return {r["bytes"]: r["busbw_med"] for r in jl(os.path.join(d, f))
                if r.get("timing") == "graph" and r["impl"] == impl and r.get("plan", "gentree") in ("gentree", "default")}
    out.append("## 16. The LL128 path for any count (its own block partition; fp32, GenTree = CPS, graph timing, busbw GB/s)\n")
    out.append("`ragged/`: the same build on aligned sizes (`aligned_*`, equal 16-byte-aligned blocks: the kernel's "
               "RAGGED = false instance) and on sizes 4 bytes longer (`ragged_*`: one fp32 element more, so blocks are "
               "unequal and the last one ends in a partial 8-byte word: RAGGED = true).  Before this change a ragged "
               "count never took the LL128 path (one-shot up to 1.5 MiB/(N−1), else the step-table kernel), and at "
               "N = 3 no power-of-two size did.  NCCL default for N = 3 from the same box (`nccl_n3_f32.jsonl`).\n")
    out.append("| size | N=4 aligned | N=4 +4 B | N=3 (+4 B) | N=3 NCCL | N=2 aligned | N=2 +4 B |")
    out.append("|---|---|---|---|---|---|---|")
    a4, r4, a3, r3, a2, r2 = (get(f"{k}_n{n}_f32.jsonl") for n in (4, 3, 2) for k in ("aligned", "ragged"))
    nc3 = get("nccl_n3_f32.jsonl", "nccl")
    for b in sorted(r4):
        base = b - 4
        out.append(f"| {size(base)} | {a4.get(base, float('nan')):.1f} | {r4[b]:.1f} | {r3.get(b, float('nan')):.1f} | "
                   f"{nc3.get(base, float('nan')):.1f} | {a2.get(base, float('nan')):.1f} | {r2.get(b, float('nan')):.1f} |")
    out.append("")
    out.append("The ragged instance costs 0–11 % against equal blocks (its last block's partial word and a few "
               "spilled registers at 3 CTAs per SM); against the paths such counts took before (N = 4, 1 MiB: the "
               "step-table kernel, 89 GB/s) it is 1.5–2× faster.  Parity: `pytest_sameproc.log` (ragged counts, "
               "N = 2/3/4, SUM/AVG, specials, back-to-back with the other paths) and the multi-GPU worker "
               "(`pytest_multi_ragged_build.log`, N = 2/3/4).\n")


def flatsteps_section(out):
    import glob
    files = sorted(glob.glob(os.path.join(P, "flatsteps", "bench_*_fs*.json")))
    if not files:
        return
    out.append("## 17. Emulated multi-step plans: step-table kernel vs ar_flatsteps_kernel (bench N = 1, 8 ranks × 256 MiB)\n")
    out.append("`flatsteps/`: `AR_FLATSTEPS=f python bench.py --force K --dtype D --no-cpu-baseline --no-e2e`.  The "
               "roofline fraction is against the measured HBM copy peak with the plan's own HBM bytes (reading A6e's D: "
               "CPS 16·S, HCPS[4,2] 22·S, HCPS[2,4] 28·S, Ring / RHD / HCPS[2,2,2] 34·S).\n")
    out.append("| plan | dtype | step-table kernel ms (frac) | ar_flatsteps_kernel ms (frac) |")
    out.append("|---|---|---|---|")
    rows = {}
    for f in files:
        d = jload(f)
        if not d:
            continue
        name = os.path.basename(f)[6:-5]           # ring_bf16_fs1
        k, dt, fs = name.rsplit("_", 2)
        rows.setdefault((k, dt), {})[fs] = d
    for (k, dt), v in sorted(rows.items()):
        cell = lambda x: f"{x['ms_per_step']:.3f} ({x['roofline']['frac']:.3f})" if x else "-"
        out.append(f"| {k} | {dt} | {cell(v.get('fs0'))} | {cell(v.get('fs1'))} |")
    out.append("")
    out.append("Barriers between steps cost what the step-table kernel's range waits save: dependent steps there "
               "overlap CTA by CTA (fp32 reaches 0.97–0.98 of the copy peak on Ring / RHD), while the grid-wide "
               "barrier serialises them (0.86–0.88).  In bf16 both sat at 0.83–0.89 — the same bytes ran at 0.98 in "
               "fp32, which does half the element work per byte: the 2-source bf16 reduce was limited by the "
               "consumer warps' work, and packing the sums with one `cvt.rn.bf16x2.f32` per pair instead of a "
               "bitwise RNE per element lifted it to 0.94–0.98 (§18).  ar_flatsteps_kernel stays "
               "an A/B option (AR_FLATSTEPS=1), off by default; its bits are tested (`pytest_exec.log`).\n")


def bf16pack_section(out):
    import glob
    files = sorted(glob.glob(os.path.join(P, "bf16pack", "bench_*_bf16.json")))
    if not files:
        return
    old = {}
    for f in glob.glob(os.path.join(P, "flatsteps", "bench_*_bf16_fs0.json")):
        d = jload(f)
        if d:
            old[os.path.basename(f)[6:-len("_bf16_fs0.json")]] = d
    out.append("## 18. bf16 stores packed with `cvt.rn.bf16x2.f32` (bench N = 1, 8 ranks × 256 MiB bf16)\n")
    out.append("`bf16pack/`: `python bench.py [--force K] --no-cpu-baseline --no-e2e` on the build that packs each "
               "pair of fp32 sums with one `cvt.rn.bf16x2.f32` (the same RNE bits for every non-NaN value; the GPU "
               "suite `pytest_gpu_1gpu.log` incl. subnormal/overflow/inf/NaN inputs passes) against the bitwise RNE "
               "of the previous build (§17's step-table column).  HBM roofline fraction and the held-out "
               "GenModel error of the A6e prediction.\n")
    out.append("| plan | before: ms (frac, pred. err) | after: ms (frac, pred. err) |")
    out.append("|---|---|---|")
    for f in files:
        d = jload(f)
        if not d:
            continue
        k = os.path.basename(f)[6:-len("_bf16.json")]
        o = old.get(k)
        cell = lambda x: f"{x['ms_per_step']:.3f} ({x['roofline']['frac']:.3f}, {x['genmodel']['pred_err']:.1%})"
        out.append(f"| {k} | {cell(o) if o else '-'} | {cell(d)} |")
    out.append("")


def main():
    out = ["# profiles/round2 — measured evidence (round 2)\n",
           "Generated by `tools/profiles_report_r2.py` from the files in this directory.  Commands:",
           "`COMMANDS.md`.  Round-1 evidence: `../README.md`.\n"]
    bench_section(out)
    c2_section(out)
    bf16_section(out)
    pick_section(out)
    ll128_section(out)
    nccl_algo_section(out)
    out.append("## 3. GenModel fit and held-out prediction error\n")
    fit_section(out)
    push_section(out)
    fence_section(out)
    p2p_section(out)
    fanin_ag_section(out)
    cpu_section(out)
    nvls_sweep_section(out)
    nvls_bf16_section(out)
    split_section(out)
    cut_section(out)
    llsplit_section(out)
    simu_baselines_section(out)
    c2_genmodel_section(out)
    ragged_section(out)
    flatsteps_section(out)
    bf16pack_section(out)
    print("\n".join(out))


if __name__ == "__main__":
    main()
