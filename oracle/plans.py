"""AllReduce plans (oracle; test infrastructure only).

A plan is "an ordering of the data movement and reducing steps".  Every rank holds
one buffer of `count` elements split into N final blocks; block b has count//N elements
plus one if b < count % N (reading Q3).  The same block lives at the same
offset in every rank's buffer.

Step semantics:
  RS step: each Reduce(server r, block b, inputs I) sets buf[r][b] = sum over q in I of
           buf[q][b], summed left to right in the order of I (ascending rank, reading Q1).
           A Reduce with one input is a pure move (GenTree data rearrangement).
           The step's transfers are the implied (q -> r, b) for q in I, q != r.
  AG step: each Transfer(src, dst, b) sets buf[dst][b] = buf[src][b].
Within a step all ops are concurrent; `check_step_hazards` enforces that no op writes a
(rank, block) another op of the same step reads or writes.

Natural ReduceScatter builders over c participants and c "chunks":
  cps  — participant k reduces chunk k from all c
  ring — step j: participant i reduces chunk (i-j) mod c from its left neighbour's
         partial and its own; chunk k ends at participant (k-2) mod c (reading Q10)
  rhd  — masks 1,2,4,..; the pair (i, i^mask) halves its chunk range, the lower rank keeping
         the lower half (reading Q11); chunk j ends at participant bitrev(j)
  hcps — [f0..f_{m-1}], participant k = d0 + f0*(d1 + f1*(...)); level-i group = ranks
         differing only in digit d_i ("orthogonal"); level-i region = the d_i-th
         consecutive 1/f_i of the level-(i-1) region (reading Q4)
  rb   — participant 0 reduces every chunk from all c (root = 0)
The AllGather phase is the RS reversed: steps in reverse order, every transfer flipped,
reduces dropped ("AllGather can be performed in the reverse order"; reading Q10b).
"""
from __future__ import annotations

import json
from dataclasses import dataclass, field


class PlanError(ValueError):
    """Invalid plan request or failed verification."""


@dataclass(frozen=True)
class Reduce:
    server: int
    block: int
    inputs: tuple            # ranks, summation order


@dataclass(frozen=True)
class Transfer:
    src: int
    dst: int
    block: int
    size: int                # elements


@dataclass
class Step:
    phase: str               # "rs" | "ag"
    label: str
    reduces: list = field(default_factory=list)
    transfers: list = field(default_factory=list)


@dataclass
class Plan:
    n: int
    count: int
    steps: list
    # NVLS plan kind (readings NV1/NV2): the CPS data movement
    # with every fan-in-N reduce done in the NVSwitch — each element becomes the correctly
    # rounded fp32 sum of the ranks' inputs, not a plan-order sum
    switch_reduce: bool = False

    @property
    def nsteps(self) -> int:
        return len(self.steps)


# ---------------------------------------------------------------- blocks (reading Q3)

def block_size(count: int, n: int, b: int) -> int:
    return count // n + (1 if b < count % n else 0)


def block_offset(count: int, n: int, b: int) -> int:
    return b * (count // n) + min(b, count % n)


# ---------------------------------------------------------------- natural RS builders

def is_pow2(x: int) -> bool:
    return x >= 1 and (x & (x - 1)) == 0


def bitrev(j: int, bits: int) -> int:
    r = 0
    for k in range(bits):
        if j & (1 << k):
            r |= 1 << (bits - 1 - k)
    return r


def natural_rs(kind: str, c: int, fanins: tuple = ()):
    """Natural RS schedule over c participants / c chunks.

    Returns (steps, natowner): steps is a list of steps, each a list of
    (participant, chunk, input_participants); natowner[j] = participant that holds the
    fully reduced chunk j after the RS.
    """
    if c < 2:
        raise PlanError("need at least 2 participants")
    if kind == "cps":
        return [[(k, k, tuple(range(c))) for k in range(c)]], list(range(c))
    if kind == "rb":
        return [[(0, j, tuple(range(c))) for j in range(c)]], [0] * c
    if kind == "ring":
        steps = []
        for j in range(c - 1):
            steps.append([(i, (i - j) % c, ((i - 1) % c, i)) for i in range(c)])
        return steps, [(k - 2) % c for k in range(c)]
    if kind == "rhd":
        if not is_pow2(c):
            raise PlanError("natural rhd needs a power-of-two participant count")
        bits = c.bit_length() - 1
        lo, hi = [0] * c, [c] * c
        steps = []
        for k in range(bits):
            mask = 1 << k
            st = []
            nlo, nhi = lo[:], hi[:]
            for i in range(c):
                p = i ^ mask
                mid = (lo[i] + hi[i]) // 2
                if i & mask:
                    nlo[i] = mid
                else:
                    nhi[i] = mid
                for j in range(nlo[i], nhi[i]):
                    st.append((i, j, (min(i, p), max(i, p))))
            lo, hi = nlo, nhi
            steps.append(st)
        return steps, [bitrev(j, bits) for j in range(c)]
    if kind == "hcps":
        f = tuple(fanins)
        prod = 1
        for x in f:
            if x < 2:
                raise PlanError("hcps fan-ins must be >= 2")
            prod *= x
        if prod != c or not f:
            raise PlanError(f"hcps fan-ins {list(f)} do not multiply to {c}")
        m = len(f)

        def digits(k):
            d = []
            for x in f:
                d.append(k % x)
                k //= x
            return d

        def place(d):  # participant from digits
            k, mul = 0, 1
            for i in range(m):
                k += d[i] * mul
                mul *= f[i]
            return k

        steps = []
        for i in range(m):
            st = []
            for k in range(c):
                d = digits(k)
                lo, size = 0, c
                for l in range(i + 1):
                    size //= f[l]
                    lo += d[l] * size
                group = []
                for x in range(f[i]):
                    dd = d[:]
                    dd[i] = x
                    group.append(place(dd))
                for j in range(lo, lo + size):
                    st.append((k, j, tuple(group)))
            steps.append(st)
        natowner = []
        for j in range(c):
            # j = sum_i d_i * size_i  with size_i = c / (f0...f_i)
            d, rem, size = [], j, c
            for i in range(m):
                size //= f[i]
                d.append(rem // size)
                rem %= size
            natowner.append(place(d))
        return steps, natowner
    raise PlanError(f"unknown kind {kind!r}")


def realize(nat_steps, chunk_blocks, participants, count, n, label, phase="rs"):
    """Map natural (participant, chunk) steps to rank/block Reduces.

    chunk_blocks[j] = actual blocks of natural chunk j; participants[k] = rank.
    """
    out = []
    for st in nat_steps:
        step = Step(phase, label)
        for (k, j, ins) in st:
            r = participants[k]
            ranks = tuple(sorted(participants[q] for q in ins))
            for b in chunk_blocks[j]:
                step.reduces.append(Reduce(r, b, ranks))
        out.append(step)
    return out


def add_implied_transfers(step: Step, count: int, n: int) -> Step:
    tr = []
    for rd in step.reduces:
        for q in rd.inputs:
            if q != rd.server:
                tr.append(Transfer(q, rd.server, rd.block, block_size(count, n, rd.block)))
    step.transfers = tr
    return step


def reverse_to_allgather(rs_steps: list) -> list:
    """P:559 / S:238-246: steps reversed, transfers flipped, reduces dropped."""
    ag = []
    for st in reversed(rs_steps):
        ag.append(Step("ag", st.label, [],
                       [Transfer(t.dst, t.src, t.block, t.size) for t in st.transfers]))
    return ag


def rhd_rs_general(n: int, count: int) -> list:
    """RHD RS on any N (oracle only): fold the first r = N - 2^floor(log N) even ranks into
    their odd neighbour, then recursive halving over the block index range on the
    2^floor(log N) core ranks (lower rank keeps the lower half)."""
    p = 1 << (n.bit_length() - 1)
    r = n - p
    steps = []
    if r > 0:
        st = Step("rs", "rhd:fold")
        for i in range(r):
            for b in range(n):
                st.reduces.append(Reduce(2 * i + 1, b, (2 * i, 2 * i + 1)))
        steps.append(st)
    core = [2 * i + 1 for i in range(r)] + list(range(2 * r, n))
    lo, hi = [0] * p, [n] * p
    bits = p.bit_length() - 1
    for k in range(bits):
        mask = 1 << k
        st = Step("rs", "rhd")
        nlo, nhi = lo[:], hi[:]
        for i in range(p):
            q = i ^ mask
            mid = lo[i] + (hi[i] - lo[i]) // 2
            if i & mask:
                nlo[i] = mid
            else:
                nhi[i] = mid
            a, b2 = sorted((core[i], core[q]))
            for blk in range(nlo[i], nhi[i]):
                st.reduces.append(Reduce(core[i], blk, (a, b2)))
        lo, hi = nlo, nhi
        steps.append(st)
    return steps


def parse_kind(kind: str):
    """'cps' | 'ring' | 'rhd' | 'rb' | 'hcps:4,2' -> (name, fanins)."""
    if kind.startswith("hcps:"):
        try:
            f = tuple(int(x) for x in kind[5:].split(","))
        except ValueError:
            raise PlanError(f"bad hcps spec {kind!r}") from None
        return "hcps", f
    if kind in ("cps", "ring", "rhd", "rb"):
        return kind, ()
    raise PlanError(f"unknown kind {kind!r}")


def kind_label(name: str, fanins: tuple = ()) -> str:
    if name == "hcps":
        return "hcps[" + ",".join(str(x) for x in fanins) + "]"
    return name


def build_plan(kind: str, n: int, count: int) -> Plan:
    """a full AllReduce of the given kind on a single switch, ranks 0..n-1,
    natural labelling (chunk j = block j)."""
    if n < 2:
        raise PlanError("fewer than 2 servers")
    if count < 1:
        raise PlanError("count must be >= 1")
    name, f = parse_kind(kind)
    if name == "rhd" and not is_pow2(n):
        rs = rhd_rs_general(n, count)
    else:
        nat, _ = natural_rs(name, n, f)
        rs = realize(nat, [[j] for j in range(n)], list(range(n)), count, n,
                     kind_label(name, f))
    for st in rs:
        add_implied_transfers(st, count, n)
    return Plan(n, count, rs + reverse_to_allgather(rs))


def build_acps(initial: dict, final: dict, count: int, n: int, label="acps") -> list:
    """P:629 footnote / S:230-237: Asymmetric CPS — every block not at its final owner is
    sent directly; the owner reduces all partials (ascending rank).

    initial: rank -> set of blocks held (partials); final: rank -> blocks owned.
    Returns the RS step list (empty if nothing moves)."""
    holders = {}
    for r, bl in initial.items():
        for b in bl:
            holders.setdefault(b, []).append(r)
    owner = {}
    for r, bl in final.items():
        for b in bl:
            if b in owner:
                raise PlanError(f"block {b} has two owners")
            owner[b] = r
    if set(owner) != set(holders):
        raise PlanError("initial and final placements cover different blocks")
    st = Step("rs", label)
    for b in sorted(owner):
        hs = tuple(sorted(holders[b]))
        if hs == (owner[b],):
            continue
        st.reduces.append(Reduce(owner[b], b, hs))
    if not st.reduces:
        return []
    add_implied_transfers(st, count, n)
    return [st]


# ---------------------------------------------------------------- verification

def check_step_hazards(step: Step):
    """Within a step no op may write a (rank, block) that another op reads or writes."""
    writes, reads = {}, {}
    ops = []
    if step.phase == "rs":
        for i, rd in enumerate(step.reduces):
            ops.append((i, [(q, rd.block) for q in rd.inputs], (rd.server, rd.block)))
    else:
        for i, t in enumerate(step.transfers):
            ops.append((i, [(t.src, t.block)], (t.dst, t.block)))
    for i, rs, w in ops:
        if w in writes:
            raise PlanError(f"step {step.label}: {w} written twice")
        writes[w] = i
        for x in rs:
            reads.setdefault(x, set()).add(i)
    for w, i in writes.items():
        if reads.get(w, set()) - {i}:
            raise PlanError(f"step {step.label}: {w} written while read by another op")


def verify_allreduce(plan: Plan):
    """Symbolic execution on contribution tags.  Server i's block b starts with
    tag {i}; reduces union the inputs' tag sets (a repeated tag = double counting); copies
    move them.  Pass iff every server ends with the full tag set on every block."""
    n = plan.n
    tags = [[frozenset([r]) for _ in range(n)] for r in range(n)]
    for si, st in enumerate(plan.steps):
        check_step_hazards(st)
        new = {}
        if st.phase == "rs":
            for rd in st.reduces:
                acc = set()
                for q in rd.inputs:
                    t = tags[q][rd.block]
                    if acc & t:
                        raise PlanError(f"step {si}: duplicate contribution into "
                                        f"rank {rd.server} block {rd.block}")
                    acc |= t
                new[(rd.server, rd.block)] = frozenset(acc)
        else:
            for t in st.transfers:
                new[(t.dst, t.block)] = tags[t.src][t.block]
        for (r, b), v in new.items():
            tags[r][b] = v
    full = frozenset(range(n))
    for r in range(n):
        for b in range(n):
            if tags[r][b] != full:
                missing = sorted(full - tags[r][b])
                raise PlanError(f"rank {r} block {b} misses contributions {missing}")
    return True


# ---------------------------------------------------------------- canonical JSON (O9)

def plan_to_obj(plan: Plan, dtype: str) -> dict:
    steps = []
    for st in plan.steps:
        steps.append({
            "label": st.label,
            "phase": st.phase,
            "reduces": [{"block": r.block, "fan_in": len(r.inputs), "inputs": list(r.inputs),
                         "server": r.server}
                        for r in sorted(st.reduces, key=lambda r: (r.server, r.block))],
            "transfers": [{"block": t.block, "dst": t.dst, "size": t.size, "src": t.src}
                          for t in sorted(st.transfers, key=lambda t: (t.dst, t.block, t.src))],
        })
    obj = {"count": plan.count, "dtype": dtype, "n": plan.n, "steps": steps}
    if plan.switch_reduce:
        obj["switch_reduce"] = True
    return obj


def plan_to_json(plan: Plan, dtype: str) -> str:
    """Canonical plan JSON: sorted keys, compact separators, integers only."""
    return json.dumps(plan_to_obj(plan, dtype), sort_keys=True, separators=(",", ":"))


def plan_aggregates(plan: Plan, esize: int = 1):
    """per-rank totals (in units of esize bytes per element)."""
    n = plan.n
    agg = [{"sent": 0, "received": 0, "mem_ops": 0, "compute_ops": 0, "max_fan_in": 0}
           for _ in range(n)]
    for st in plan.steps:
        for t in st.transfers:
            agg[t.src]["sent"] += t.size * esize
            agg[t.dst]["received"] += t.size * esize
        for rd in st.reduces:
            k = len(rd.inputs)
            if k >= 2:
                sz = block_size(plan.count, n, rd.block) * esize
                agg[rd.server]["mem_ops"] += (k + 1) * sz
                agg[rd.server]["compute_ops"] += (k - 1) * sz
                agg[rd.server]["max_fan_in"] = max(agg[rd.server]["max_fan_in"], k)
    return agg
