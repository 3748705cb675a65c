"""Incast-aware flow-level simulation of a plan (oracle; test infrastructure only).

SURVEY §8(f) NEXT #2; the paper's simulator is described only as "a custom-made flow-level
network simulator which is aware of the incast problem", with "computation time derived from
the γ-term and the δ-term in GenModel".  Procedure (SPEC S:382-424 with the readings
in DESIGN.md, FS1-FS3):

  for every step of the plan, in order (steps are barriers):
    flows      one per transfer (src rank -> dst rank, size·esize bytes), routed on the unique
               tree path: the uplinks from src to the LCA, then the downlinks to dst; a
               directed link is (node, "up") or (node, "down") with node's uplink parameters
    latency    α_step = max α over the links any flow uses (0 if none) — one α per step (Q16)
    comm       progressive filling (max-min fair rates), recomputed at every flow completion;
               each directed link l has capacity 1/β'_l with β'_l = β_l + max(w_l − w_t,l, 0)·ε_l
               (Eq. 10, applied per link) and w_l = 1 + the number of distinct
               source ranks among the active flows on l (reading FS1 = Q8 per link)
    compute    max over servers of Σ over its reduces with k >= 2 inputs of
               (k−1)·|b|·γ + (k+1)·|b|·δ, the server's own γ, δ
    step time  α_step + comm + compute (Fig. 1: transfer, then aggregate; no overlap)
  total = Σ step times.

All arithmetic is exact (`fractions.Fraction`); links with β' = 0 impose no constraint.
Per-term attribution: bandwidth = the comm time of the same simulation with ε = 0, incast =
comm − bandwidth, compute/memory = the γ/δ parts of the step's slowest server (first in rank
order on ties).
"""
from __future__ import annotations

from fractions import Fraction

from .genmodel import Params
from .plans import Plan, block_size


def _link_params(topo, params: Params | None):
    """node id -> (α, β, ε, w_t) per byte; server rank -> (γ, δ) per byte."""
    links, comp = {}, {}
    if params is not None:
        beta, gamma = params.effective()
    for nid, nd in topo.nodes.items():
        if nd.uplink is None:
            continue
        if params is not None:
            links[nid] = (Fraction(params.alpha), Fraction(beta), Fraction(params.epsilon), params.w_t)
        else:
            u = nd.uplink
            links[nid] = (Fraction(u["alpha"]), Fraction(u["beta"]) / 4, Fraction(u["epsilon"]) / 4, int(u["w_t"]))
    for r, sid in enumerate(topo.servers):
        if params is not None:
            comp[r] = (Fraction(gamma), Fraction(params.delta))
        else:
            c = topo.nodes[sid].compute
            comp[r] = (Fraction(c["gamma"]) / 4, Fraction(c["delta"]) / 4)
    return links, comp


def route(topo, src_rank: int, dst_rank: int) -> list:
    """Directed links of the unique tree path src -> dst: [(node, "up"), ..., (node, "down")]."""
    a, b = topo.servers[src_rank], topo.servers[dst_rank]
    up_a = [a]
    while topo.nodes[up_a[-1]].parent is not None:
        up_a.append(topo.nodes[up_a[-1]].parent)
    up_b = [b]
    while topo.nodes[up_b[-1]].parent is not None:
        up_b.append(topo.nodes[up_b[-1]].parent)
    sa = set(up_a)
    lca = next(x for x in up_b if x in sa)
    ups = [(x, "up") for x in up_a[:up_a.index(lca)]]
    downs = [(x, "down") for x in reversed(up_b[:up_b.index(lca)])]
    return ups + downs


def max_min_rates(flows: list, active: list, links: dict, with_incast: bool) -> dict:
    """Progressive filling over the active flows.  flows[i] = (src, dst, bytes, path)."""
    on_link = {}
    for i in active:
        for l in flows[i][3]:
            on_link.setdefault(l, []).append(i)
    residual = {}
    for l, fl in on_link.items():
        alpha, beta, eps, w_t = links[l[0]]
        w = 1 + len({flows[i][0] for i in fl})
        bp = beta + (max(w - w_t, 0) * eps if with_incast else 0)
        residual[l] = None if bp == 0 else 1 / bp
    rate = {}
    unfrozen = set(active)
    while unfrozen:
        best = None
        for l, fl in on_link.items():
            if residual[l] is None:
                continue
            cnt = sum(1 for i in fl if i in unfrozen)
            if cnt == 0:
                continue
            share = residual[l] / cnt
            if best is None or share < best:
                best = share
        if best is None:                      # nothing constrains the rest: infinite rate
            for i in unfrozen:
                rate[i] = None
            break
        freeze = set()
        for l, fl in on_link.items():
            if residual[l] is None:
                continue
            cnt = sum(1 for i in fl if i in unfrozen)
            if cnt and residual[l] / cnt == best:
                freeze.update(i for i in fl if i in unfrozen)
        for i in freeze:
            rate[i] = best
            for l in flows[i][3]:
                if residual[l] is not None:
                    residual[l] -= best
        unfrozen -= freeze
    return rate


def comm_time(flows: list, links: dict, with_incast: bool) -> Fraction:
    remaining = {i: Fraction(f[2]) for i, f in enumerate(flows) if f[2] > 0}
    t = Fraction(0)
    while remaining:
        rate = max_min_rates(flows, list(remaining), links, with_incast)
        inf = [i for i in remaining if rate[i] is None]
        if inf:
            for i in inf:
                del remaining[i]
            continue
        dt = min(remaining[i] / rate[i] for i in remaining)
        t += dt
        for i in list(remaining):
            remaining[i] -= rate[i] * dt
            if remaining[i] == 0:
                del remaining[i]
    return t


def simulate_flows(topo, plan: Plan, esize: int, params: Params | None = None) -> dict:
    """Flow-level time of `plan` on `topo` (exact).  params != None: uniform parameters for
    every link and server (per byte), like genmodel_predict with params."""
    links, comp = _link_params(topo, params)
    n = plan.n
    lat = bw = inc = cg = cd = Fraction(0)
    steps = []
    for st in plan.steps:
        flows = []
        for t in st.transfers:
            if t.size > 0 and t.src != t.dst:
                flows.append((t.src, t.dst, t.size * esize, route(topo, t.src, t.dst)))
        used = {l[0] for f in flows for l in f[3]}
        a = max((links[x][0] for x in used), default=Fraction(0))
        c_full = comm_time(flows, links, True)
        c_bw = comm_time(flows, links, False)
        g = [Fraction(0)] * n
        d = [Fraction(0)] * n
        for rd in st.reduces:
            k = len(rd.inputs)
            if k >= 2:
                sz = block_size(plan.count, n, rd.block) * esize
                g[rd.server] += (k - 1) * sz * comp[rd.server][0]
                d[rd.server] += (k + 1) * sz * comp[rd.server][1]
        tot = [g[r] + d[r] for r in range(n)]
        slow = max(range(n), key=lambda r: (tot[r], -r))
        step_t = a + c_full + tot[slow]
        steps.append(step_t)
        lat += a
        bw += c_bw
        inc += c_full - c_bw
        cg += g[slow]
        cd += d[slow]
    total = sum(steps, Fraction(0))
    return {"latency": lat, "bandwidth": bw, "compute": cg, "memory": cd, "incast": inc, "total": total,
            "steps": steps}
