"""GenTree — Algorithms 1 and 2 of the paper (oracle; test infrastructure only).

Algorithm 1 `generate_basic_plan` — post-order; each switch gives each of its
servers floor(N/n) blocks (+1 for the first N mod n), greedily drawing blocks the server
already holds (`taken` scan).  Reading Q12: `num_total_blocks` = N, and blocks the greedy
leaves untaken go (ascending) to the first server in document order with unmet quota.

Algorithm 2 `generate_final_plan` — post-order; per child: data-rearrangement
test (readings Q15/Q15b); plan-type selection: if the
children have equal server counts, the min-GenModel candidate of {CPS, HCPS over ordered
factorizations of the child count c with m <= 3, RHD if c is a power of two, Ring}
(reading Q13), ties by (fewer steps, larger f0, candidate order) (Q14); otherwise ACPS.
Candidate cost = Table 2 closed form at (c, full message S) (reading Q27) with the switch's
parameters: max α/β/ε and min w_t over uplinks strictly below the switch, max γ/δ over its
servers (Q16).  Switch finish = max(child finish) + best time.

Sub-plan realisation: at a switch, every block has one holder per child.  Blocks with the
same holder tuple form a group whose c holders run the chosen kind's natural RS; natural
chunk j is mapped to the blocks Algorithm 1 assigns to the participant that ends up owning
chunk j, so the sub-plan reaches exactly Algorithm 1's final placement ("their initial and
final states are matched").  Sibling sub-plans share global step indices; a parent's
steps start after all its children's.  The AllGather is the RS reversed.
"""
from __future__ import annotations

import math
from fractions import Fraction
from dataclasses import dataclass, field

from .genmodel import (Params, StepCoeffs, StepParams, closed_form_f64,
                       enumerate_hcps_factorizations, predict_f64, step_coeffs,
                       topo_step_params, uniform_step_params)
from .plans import (Plan, PlanError, Reduce, Step, add_implied_transfers, block_size,
                    build_acps, build_plan, is_pow2, kind_label, natural_rs, parse_kind,
                    realize, reverse_to_allgather, verify_allreduce)


@dataclass
class SwitchReport:
    switch: str
    chosen: str
    candidates: list = field(default_factory=list)     # (label, total seconds)
    rearranged_children: list = field(default_factory=list)
    start_time: float = 0.0
    finish_time: float = 0.0


def generate_basic_plan(topo, N: int) -> dict:
    """Algorithm 1 for every node: returns node id -> final_place (ordered dict
    rank -> list of blocks, in take order)."""
    final = {}

    def rec(nid):
        node = topo.nodes[nid]
        if node.kind == "server":
            final[nid] = {topo.rank[nid]: list(range(N))}
            return
        for ch in node.children:
            rec(ch)
        taken = [False] * N
        n = len(topo.servers_under(nid))
        num_blocks = N // n
        remain = N % n
        place, quota = {}, {}
        for ch in node.children:
            for server, blocks in final[ch].items():
                want = num_blocks
                if remain > 0:
                    want += 1
                    remain -= 1
                place[server] = []
                for b in blocks:
                    if not taken[b]:
                        taken[b] = True
                        place[server].append(b)
                        want -= 1
                        if want == 0:
                            break
                quota[server] = want
        for b in range(N):                    # reading Q12: complete the partition
            if not taken[b]:
                for server in place:
                    if quota[server] > 0:
                        place[server].append(b)
                        quota[server] -= 1
                        taken[b] = True
                        break
        final[nid] = place

    rec(topo.root)
    return final


def _switch_params(topo, nid, explicit: Params | None) -> Params:
    if explicit is not None:
        return explicit
    links = [x for x in topo.subtree(nid) if x != nid]
    ups = [topo.nodes[x].uplink for x in links]
    servers = topo.servers_under(nid)
    return Params(max(u["alpha"] for u in ups), max(u["beta"] for u in ups) / 4,
                  max(topo.nodes[s].compute["gamma"] for s in servers) / 4,
                  max(topo.nodes[s].compute["delta"] for s in servers) / 4,
                  max(u["epsilon"] for u in ups) / 4, min(u["w_t"] for u in ups))


def _uplink_step_params(topo, nid, explicit: Params | None) -> StepParams:
    if explicit is not None:
        return uniform_step_params(explicit, 1)[0]
    u = topo.nodes[nid].uplink
    return StepParams(u["alpha"], u["beta"] / 4, u["epsilon"] / 4, u["w_t"], 0.0, 0.0)


def candidates_for(c: int):
    """Reading Q13: candidate (name, fanins) list in tie-break order."""
    out = [("cps", ())]
    for f in enumerate_hcps_factorizations(c, 3):
        if len(f) >= 2:
            out.append(("hcps", f))
    if is_pow2(c):
        out.append(("rhd", ()))
    out.append(("ring", ()))
    return out


def _steps_of(name, c, f):
    if name == "cps" or name == "rb":
        return 2
    if name == "ring":
        return 2 * (c - 1)
    if name == "rhd":
        return 2 * (c - 1).bit_length()
    return 2 * len(f)


def _f0(name, c, f):
    if name == "cps":
        return c
    if name == "hcps":
        return f[0]
    return 2


def _eval_step_cost(coeff: StepCoeffs, sp: StepParams) -> float:
    return predict_f64([coeff], [sp])["total"]


def gentree(topo, count: int, esize: int, params: Params | None = None,
            force: str | None = None):
    """GenTree on `topo` for `count` elements of `esize` bytes.  Returns (Plan, reports).

    `force` (e.g. "ring", "hcps:4,2") restricts every switch's candidate set to that kind;
    "rb" is only accepted on a single-switch topology (natural Reduce-Broadcast);
    "norearrange" is tab:gentreesimu's GenTree* ("the special plan without data
    rearrangement"): Algorithm 2 without its data-rearrangement step."""
    rearrange = force != "norearrange"
    if not rearrange:
        force = None
    N = len(topo.servers)
    if count < 1:
        raise PlanError("count must be >= 1")
    S = count * esize
    if force == "nvls":
        # NVLS plan kind (readings NV1/NV2): CPS's data movement on one
        # NVSwitch, the reduce done in the switch; fp32 only (its bf16 rounding is not RNE)
        if esize != 4:
            raise PlanError("NVLS plans are fp32 only (reading NV2)")
        if sum(1 for nd in topo.nodes.values() if nd.kind != "server") != 1:
            raise PlanError("NVLS plans need a single-switch topology")
        plan, reps = gentree(topo, count, esize, params, "cps")
        plan.switch_reduce = True
        for rp in reps:
            rp.chosen = "nvls"
        return plan, reps
    if force is not None:
        fname, ff = parse_kind(force)
        if fname == "rb":
            if any(topo.nodes[c].kind != "server" for c in topo.nodes[topo.root].children):
                raise PlanError("rb is only defined on a single-switch topology")
            plan = build_plan("rb", N, count)
            verify_allreduce(plan)
            return plan, [SwitchReport(topo.root, "rb")]
    basic = generate_basic_plan(topo, N)
    owner_at = {}                               # switch -> block -> owner rank
    local = {}                                  # node -> list of local RS Steps
    finish = {}                                 # node -> finish time
    place_now = {}                              # node -> rank -> set(blocks) seen by parent
    reports = []

    def servers_of(nid):
        return set(topo.ranks_under(nid))

    def rec(nid):
        node = topo.nodes[nid]
        if node.kind == "server":
            local[nid], finish[nid] = [], 0.0
            place_now[nid] = {topo.rank[nid]: set(range(N))}
            return
        for ch in node.children:
            rec(ch)
        own = {}
        for r, bl in basic[nid].items():
            for b in bl:
                own[b] = r
        owner_at[nid] = own
        rep = SwitchReport(nid, "")
        # ---- data rearrangement
        for ch in node.children:
            if not rearrange or topo.nodes[ch].kind == "server":
                continue
            ch_servers = topo.ranks_under(ch)
            ni = len(ch_servers)
            if ni < 2:
                continue
            # subset = the lowest-indexed ceil(n_i / r) servers (reading Q15), exact rationals
            ratio = topo.convergence_ratio(nid, ch)
            k = math.ceil(Fraction(ni) / ratio)
            k = max(1, min(ni, k))
            if k >= ni:
                continue
            subset = ch_servers[:k]
            cur = place_now[ch]
            held = sorted((b, r) for r, bl in cur.items() for b in bl)
            rearr = {r: set() for r in ch_servers}
            moves = []
            for j, (b, r) in enumerate(held):
                dst = subset[j % k]
                rearr[dst].add(b)
                if dst != r:
                    moves.append((r, dst, b))
            ch_set = set(ch_servers)

            def out_time(pl):
                B, senders = 0, set()
                for r, bl in pl.items():
                    for b in bl:
                        if own[b] not in ch_set:
                            B += block_size(count, N, b) * esize
                            senders.add(r)
                return _eval_step_cost(StepCoeffs(1, B, 0, 0, len(senders)),
                                       _uplink_step_params(topo, ch, params))

            t_origin = out_time(cur)
            sent, recv, snd = {}, {}, {}
            for (r, d, b) in moves:
                sz = block_size(count, N, b) * esize
                sent[r] = sent.get(r, 0) + sz
                recv[d] = recv.get(d, 0) + sz
                snd.setdefault(d, set()).add(r)
            Bm = max(list(sent.values()) + list(recv.values()) + [0])
            wm = 1 + max([len(v) for v in snd.values()] + [0])
            if params is not None:
                sp = uniform_step_params(params, 1)[0]
            else:
                links = set()
                for (r, d, b) in moves:
                    links.update(topo.path_links(topo.servers[r], topo.servers[d]))
                ups = [topo.nodes[x].uplink for x in sorted(links)]
                sp = (StepParams(max(u["alpha"] for u in ups), max(u["beta"] for u in ups) / 4,
                                 max(u["epsilon"] for u in ups) / 4, min(u["w_t"] for u in ups),
                                 0.0, 0.0) if ups else StepParams(0.0, 0.0, 0.0, 1 << 30, 0.0, 0.0))
            t_cps = _eval_step_cost(StepCoeffs(1, Bm, 0, 0, wm), sp)
            t_rearr = t_cps + out_time(rearr)
            if moves and t_rearr < t_origin:
                st = Step("rs", f"{ch}:rearrange")
                for (r, d, b) in sorted(moves, key=lambda x: x[2]):
                    st.reduces.append(Reduce(d, b, (r,)))
                local[ch].append(st)
                finish[ch] += t_cps
                place_now[ch] = rearr
                rep.rearranged_children.append(ch)
        start = max(finish[ch] for ch in node.children)
        # ---- plan-type selection
        init = {}
        for ch in node.children:
            for r, bl in place_now[ch].items():
                init.setdefault(r, set()).update(bl)
        holders = {b: [] for b in range(N)}
        for r in sorted(init):
            for b in init[r]:
                holders[b].append(r)
        c = len(node.children)
        counts = {len(topo.servers_under(ch)) for ch in node.children}
        regular = (len(counts) == 1 and
                   all(len(holders[b]) == c and own[b] in holders[b] for b in range(N)))
        sp_x = _switch_params(topo, nid, params)
        if c == 1:
            rep.chosen = "none"
            cands, best = [], None
        elif regular:
            cands = candidates_for(c)
            if force is not None:
                fname, ff = parse_kind(force)
                if fname == "hcps":
                    p = 1
                    for x in ff:
                        p *= x
                    if p != c or any(x < 2 for x in ff):
                        raise PlanError(f"hcps fan-ins {list(ff)} do not multiply to "
                                        f"{c} at switch {nid!r}")
                if fname == "rhd" and not is_pow2(c):
                    raise PlanError(f"rhd needs a power-of-two child count at {nid!r}")
                cands = [(fname, ff)]
        else:
            cands = [("acps", ())]
        best_key, best = None, None
        for idx, (name, f) in enumerate(cands):
            if name == "acps":
                st = build_acps(init, basic[nid], count, N, f"{nid}:acps")
                tmp = Plan(N, count, st + reverse_to_allgather(st))
                coeffs = step_coeffs(tmp, esize)
                total = predict_f64(coeffs, uniform_step_params(sp_x, len(coeffs)))["total"]
                nst = len(coeffs)
            else:
                total = closed_form_f64(name, c, S, sp_x, f)["total"]
                nst = _steps_of(name, c, f)
            rep.candidates.append((kind_label(name, f), total))
            key = (total, nst, -_f0(name, c, f), idx)
            if best_key is None or key < best_key:
                best_key, best = key, (name, f, total)
        steps = []
        if best is not None:
            name, f, total = best
            rep.chosen = kind_label(name, f)
            if name == "acps":
                steps = build_acps(init, basic[nid], count, N, f"{nid}:acps")
            else:
                groups = {}
                for b in range(N):
                    groups.setdefault(tuple(holders[b]), []).append(b)
                nat, natowner = natural_rs(name, c, f)
                lab = f"{nid}:{kind_label(name, f)}"
                for tup, blocks in sorted(groups.items(), key=lambda kv: kv[1][0]):
                    chunk_of = [sorted(b for b in blocks if own[b] == p) for p in tup]
                    chunk_blocks = [chunk_of[natowner[j]] for j in range(c)]
                    gst = realize(nat, chunk_blocks, list(tup), count, N, lab)
                    for i, s in enumerate(gst):
                        if i == len(steps):
                            steps.append(Step("rs", lab))
                        steps[i].reduces.extend(s.reduces)
            rep.finish_time = start + total
        else:
            rep.finish_time = start
        rep.start_time = start
        local[nid] = steps
        finish[nid] = rep.finish_time
        place_now[nid] = {r: set(bl) for r, bl in basic[nid].items()}
        reports.append(rep)

    rec(topo.root)
    # ---- composition: global step index = max over children of (start + length)
    start_idx, length = {}, {}

    def sched(nid):
        node = topo.nodes[nid]
        if node.kind == "server":
            start_idx[nid] = 0
            length[nid] = 0
            return
        s = 0
        for ch in node.children:
            sched(ch)
            s = max(s, start_idx[ch] + length[ch])
        start_idx[nid] = s
        length[nid] = len(local[nid])

    sched(topo.root)
    total_rs = start_idx[topo.root] + length[topo.root]
    rs = [Step("rs", "") for _ in range(total_rs)]
    labels = [[] for _ in range(total_rs)]

    def compose(nid):
        node = topo.nodes[nid]
        if node.kind == "server":
            return
        for ch in node.children:
            compose(ch)
        # a child's rearrangement step sits at the end of the child's local list
        for i, st in enumerate(local[nid]):
            g = start_idx[nid] + i
            rs[g].reduces.extend(st.reduces)
            labels[g].append(st.label)

    compose(topo.root)
    steps = []
    for g, st in enumerate(rs):
        if not st.reduces:
            continue
        st.label = "+".join(labels[g])
        add_implied_transfers(st, count, N)
        steps.append(st)
    plan = Plan(N, count, steps + reverse_to_allgather(steps))
    verify_allreduce(plan)
    return plan, reports


def predict_plan(topo, plan: Plan, esize: int, params: Params | None = None) -> dict:
    """a6: per-step GenModel of the executed plan (fixed-order float64)."""
    coeffs = step_coeffs(plan, esize)
    sp = (uniform_step_params(params, len(coeffs)) if params is not None
          else topo_step_params(topo, plan))
    return predict_f64(coeffs, sp)


def oneshot_eligible(plan: Plan) -> bool:
    """A plan the executor's one-shot path runs with the plan's own bits: an
    RS step of N reduces, one per block, each over all N ranks in one common order, then one
    AG step."""
    if plan.switch_reduce or len(plan.steps) != 2:
        return False
    rs, ag = plan.steps
    if rs.phase != "rs" or ag.phase != "ag" or len(rs.reduces) != plan.n:
        return False
    order = rs.reduces[0].inputs
    return (sorted(order) == list(range(plan.n)) and all(r.inputs == order for r in rs.reduces)
            and sorted(r.block for r in rs.reduces) == list(range(plan.n)))


def gentree_nvls(topo, count: int, esize: int, params: Params, nvls_params: Params,
                 oneshot_params: Params | None = None, oneshot_max_bytes: int = 0,
                 ll128_params: Params | None = None, ll128_max_bytes: int = 0, ll128_min_bytes: int = 0):
    """GenTree with the NVLS plan kind as one more candidate (reading NV1; the paper's
    minimum-GenModel choice): on a single-switch topology in fp32, the NVLS plan
    replaces GenTree's plan iff the NVLS row's closed form (P:441-444 with its own α, β) is
    strictly below the prediction of the path the executor runs GenTree's plan on — the
    LL128 row for one-shot-eligible plans with N <= 8, at least 8 bytes per rank and block, and
    a size in (min(ll128_min_bytes, oneshot_max_bytes), ll128_max_bytes] when its parameters are
    given, else the one-shot row (reading OS1) for one-shot-eligible plans up to
    oneshot_max_bytes when given, else the executed-plan prediction (ties keep the plan).
    The cut-offs are the executor's (a measured engineering choice, not the paper's)."""
    from .genmodel import predict_executed
    plan, reps = gentree(topo, count, esize, params)
    single = sum(1 for nd in topo.nodes.values() if nd.kind != "server") == 1
    if esize == 4 and single:
        t_plan = predict_executed(plan, esize, params)["total"]
        n = len(topo.servers)
        S = count * esize
        if (ll128_params is not None and oneshot_eligible(plan) and n <= 8 and S >= 8 * n
                and min(ll128_min_bytes, oneshot_max_bytes) < S <= ll128_max_bytes):
            t_plan = closed_form_f64("ll128", n, S, ll128_params)["total"]
        elif oneshot_params is not None and S <= oneshot_max_bytes and oneshot_eligible(plan):
            t_plan = closed_form_f64("oneshot", n, S, oneshot_params)["total"]
        t_nvls = closed_form_f64("nvls", len(topo.servers), count * esize, nvls_params)["total"]
        if t_nvls < t_plan:
            return gentree(topo, count, esize, params, "nvls")
    return plan, reps
