"""GenModel (oracle; test infrastructure only).

T = A·α + B·β + C·γ + D·δ + max(w − w_t, 0)·B·ε

  A  communication rounds (steps)
  B  data through a link per step, here per rank max(sent, received)   (reading Q9)
  C  reduce operations: a fan-in-f reduce of a block costs (f−1)·|block|
  D  memory operations: a fan-in-f reduce of a block costs (f+1)·|block|
  w  fan-in of the step: 1 + the most distinct senders into one receiver   (Q8)

Units: bytes; α in seconds, β/γ/δ/ε in seconds per byte (Table 5's per-float values / 4,
exact in binary; reading Q17).

Two evaluations are provided and both are pinned by tests:
  * exact rational (`fractions.Fraction`) — used for every identity the paper fixes
    (Tables 1/2, Theorem 1/2, Eq. 6);
  * fixed-order float64 — the contract the C-ABI library reproduces bit for bit
    (DESIGN.md "cost evaluation order"):  per step  ((((α + B·β) + C·γ) + D·δ) + I·ε)  with
    I = max(w − w_t, 0)·B formed in integers, steps summed in plan order; closed forms as
    (((A·α + (Bn/den)·β) + (Cn/den)·γ) + (Dn/den)·δ) + (In/den)·ε with integer numerators.
"""
from __future__ import annotations

from dataclasses import dataclass
from fractions import Fraction

from .plans import Plan, block_size, is_pow2


@dataclass(frozen=True)
class Params:
    """Per-byte GenModel parameters.  `combined` = fitted 2β+γ."""
    alpha: float
    beta: float
    gamma: float
    delta: float
    epsilon: float
    w_t: int
    combined: float | None = None

    def effective(self):
        """(β, γ) actually used: with only 2β+γ known, β_eff = combined/2, γ_eff = 0
        ("bandwidth=(B/2)·combined, compute=0"; exact in binary)."""
        if self.combined is not None:
            return self.combined * 0.5, 0.0
        return self.beta, self.gamma


def params_per_float(alpha, beta, gamma, delta, epsilon, w_t) -> Params:
    """Table 5 units (per float) -> per byte."""
    return Params(alpha, beta / 4, gamma / 4, delta / 4, epsilon / 4, w_t)


@dataclass(frozen=True)
class StepCoeffs:
    A: int
    B: int      # bytes
    C: int      # bytes
    D: int      # bytes
    w: int


@dataclass(frozen=True)
class StepParams:
    alpha: float
    beta: float
    epsilon: float
    w_t: int
    gamma: float
    delta: float


def step_coeffs(plan: Plan, esize: int) -> list:
    """Per-step (A, B, C, D, w) of a plan.  Each quantity is the max over
    ranks of that rank's per-step total (ranks run in parallel)."""
    n, out = plan.n, []
    for st in plan.steps:
        sent, recv = [0] * n, [0] * n
        senders = [set() for _ in range(n)]
        for t in st.transfers:
            sent[t.src] += t.size * esize
            recv[t.dst] += t.size * esize
            senders[t.dst].add(t.src)
        cc, dd = [0] * n, [0] * n
        for rd in st.reduces:
            k = len(rd.inputs)
            if k >= 2:
                sz = block_size(plan.count, n, rd.block) * esize
                cc[rd.server] += (k - 1) * sz
                dd[rd.server] += (k + 1) * sz
        B = max(max(sent), max(recv))
        w = 1 + max(len(s) for s in senders)
        out.append(StepCoeffs(1, B, max(cc), max(dd), w))
    return out


def uniform_step_params(p: Params, nsteps: int) -> list:
    beta, gamma = p.effective()
    return [StepParams(p.alpha, beta, p.epsilon, p.w_t, gamma, p.delta)] * nsteps


def topo_step_params(topo, plan: Plan) -> list:
    """Per-step parameters from the links the step's transfers traverse: max α, β, ε and
    min w_t over traversed uplinks (reading Q16); γ, δ = max over servers.  Per byte."""
    gamma = max(topo.nodes[s].compute["gamma"] for s in topo.servers) / 4
    delta = max(topo.nodes[s].compute["delta"] for s in topo.servers) / 4
    out = []
    for st in plan.steps:
        links = set()
        for t in st.transfers:
            links.update(topo.path_links(topo.servers[t.src], topo.servers[t.dst]))
        if links:
            ups = [topo.nodes[x].uplink for x in sorted(links)]
            out.append(StepParams(max(u["alpha"] for u in ups), max(u["beta"] for u in ups) / 4,
                                  max(u["epsilon"] for u in ups) / 4,
                                  min(u["w_t"] for u in ups), gamma, delta))
        else:
            out.append(StepParams(0.0, 0.0, 0.0, 1 << 30, gamma, delta))
    return out


def _breakdown(lat, bw, comp, mem, inc, tot):
    return {"latency": lat, "bandwidth": bw, "compute": comp, "memory": mem,
            "incast": inc, "total": tot}


def predict_exact(coeffs: list, sparams: list) -> dict:
    """Exact rational GenModel of a plan, summed over steps."""
    F = Fraction
    lat = bw = comp = mem = inc = F(0)
    for c, p in zip(coeffs, sparams):
        lat += c.A * F(p.alpha)
        bw += c.B * F(p.beta)
        comp += c.C * F(p.gamma)
        mem += c.D * F(p.delta)
        inc += max(c.w - p.w_t, 0) * c.B * F(p.epsilon)
    return _breakdown(lat, bw, comp, mem, inc, lat + bw + comp + mem + inc)


def predict_f64(coeffs: list, sparams: list) -> dict:
    """Fixed-order float64 GenModel (the library's contract, bit for bit)."""
    lat = bw = comp = mem = inc = tot = 0.0
    for c, p in zip(coeffs, sparams):
        a = float(c.A) * p.alpha
        b = float(c.B) * p.beta
        g = float(c.C) * p.gamma
        d = float(c.D) * p.delta
        i = float(max(c.w - p.w_t, 0) * c.B) * p.epsilon
        t = (((a + b) + g) + d) + i
        lat += a
        bw += b
        comp += g
        mem += d
        inc += i
        tot += t
    return _breakdown(lat, bw, comp, mem, inc, tot)


# ---------------------------------------------------------------- closed forms (Tables 1, 2)

def _ceil_log2(c: int) -> int:
    return (c - 1).bit_length()


def closed_form_terms(kind: str, c: int, S: int, w_t: int, fanins: tuple = ()):
    """Integer numerators over a common denominator for Table 2's row of `kind` at
    N = c servers and S bytes: returns (A, Bn, Cn, Dn, In, den) with the ε coefficient
    I = In/den already multiplied by the max(·, 0) factors.

    RB   P:459 (γ = (N−1)S, reading Q7)      Ring P:460      RHD P:461 (+χ(N) fold)
    CPS  P:462                               HCPS P:463 with readings Q5 (memory) and Q6
    (incast): D = (2·Σ_{i=1}^{m−1} Π_{j=i}^{m−1} f_j + N + 1)·S/N,
              I = Σ_i max(0, f_i − w_t)·2(f_i − 1)·Π_{j>i} f_j·S/N.
    """
    if c < 2:
        raise ValueError("closed forms need N >= 2")
    if kind == "rb":
        return 2, 2 * (c - 1) * S, (c - 1) * S, (c + 1) * S, 2 * (c - 1) * S * max(c - w_t, 0), 1
    if kind == "cps":
        return 2, 2 * (c - 1) * S, (c - 1) * S, (c + 1) * S, 2 * (c - 1) * S * max(c - w_t, 0), c
    if kind == "ring":
        return 2 * (c - 1), 2 * (c - 1) * S, (c - 1) * S, 3 * (c - 1) * S, 0, c
    if kind == "rhd":
        chi = 0 if is_pow2(c) else 1
        return (2 * _ceil_log2(c), 2 * (c - 1) * S + chi * 2 * S * c, (c - 1) * S + chi * S * c,
                3 * (c - 1) * S + chi * 3 * S * c, 0, c)
    if kind == "hcps":
        f = tuple(fanins)
        prod = 1
        for x in f:
            prod *= x
        if prod != c or any(x < 2 for x in f) or not f:
            raise ValueError(f"invalid factorization {f} of {c}")
        m = len(f)
        suffix_sum = 0
        for i in range(1, m):
            p = 1
            for j in range(i, m):
                p *= f[j]
            suffix_sum += p
        inc = 0
        for i in range(m):
            tail = 1
            for j in range(i + 1, m):
                tail *= f[j]
            inc += max(0, f[i] - w_t) * 2 * (f[i] - 1) * tail
        return (2 * m, 2 * (c - 1) * S, (c - 1) * S, (2 * suffix_sum + c + 1) * S, inc * S, c)
    if kind == "nvls":
        # SURVEY §8(f) NEXT #1, reading NV1: CPS's two steps with the fan-in-N
        # reduce done in the switch.  Per GPU and direction it sends its S/N slice to each
        # of the N switch reductions (S) plus its reduced block once (S/N), and receives its
        # reduced block (S/N) plus N multicast blocks (S): B = (N+1)·S/N.  No GPU-side
        # reduce (C = D = 0) and no unicast many-to-one flows (I = 0).
        return 2, (c + 1) * S, 0, 0, 0, c
    if kind == "oneshot":
        # NOT a paper row: a measured-protocol row of this executor (reading OS1),
        # kept here only so the library's evaluation of it has a checked counterpart.  Its B
        # counts the executor's own wire format (16-byte lines carrying 8 payload bytes), so it
        # describes the kernel, not the method; nothing in the paper pins it.  One round; every rank
        # sends its whole input to each of the N-1 others as 16-byte lines carrying 8 payload
        # bytes (B = 2(N-1)S per direction), then reduces all N blocks itself in plan order
        # (C = (N-1)S, D = (N+1)S); every rank receives from N-1 senders (w = N, as CPS).
        return 1, 2 * (c - 1) * S, (c - 1) * S, (c + 1) * S, 2 * (c - 1) * S * max(c - w_t, 0), 1
    if kind == "ll128":
        # NOT a paper row: the executor's LL128 two-shot path, a measured-protocol
        # row like "oneshot".  One round (the flags travel in the data); every rank writes its
        # N-1 slices of S/N and its result to N-1 peers as 128-byte lines of 120 payload bytes
        # (B = 2(N-1)S/N · 128/120 per direction), reduces its own block from N inputs (CPS's
        # C and D), and receives from N-1 senders (w = N, as CPS).  Common denominator 15N.
        return (1, 32 * (c - 1) * S, 15 * (c - 1) * S, 15 * (c + 1) * S,
                32 * (c - 1) * S * max(c - w_t, 0), 15 * c)
    raise ValueError(f"no closed form for {kind!r}")


def closed_form_exact(kind, c, S, p: Params, fanins=()) -> dict:
    A, Bn, Cn, Dn, In, den = closed_form_terms(kind, c, S, p.w_t, fanins)
    beta, gamma = p.effective()
    F = Fraction
    lat = A * F(p.alpha)
    bw = F(Bn, den) * F(beta)
    comp = F(Cn, den) * F(gamma)
    mem = F(Dn, den) * F(p.delta)
    inc = F(In, den) * F(p.epsilon)
    return _breakdown(lat, bw, comp, mem, inc, lat + bw + comp + mem + inc)


def closed_form_f64(kind, c, S, p: Params, fanins=()) -> dict:
    A, Bn, Cn, Dn, In, den = closed_form_terms(kind, c, S, p.w_t, fanins)
    beta, gamma = p.effective()
    dd = float(den)
    lat = float(A) * p.alpha
    bw = (float(Bn) / dd) * beta
    comp = (float(Cn) / dd) * gamma
    mem = (float(Dn) / dd) * p.delta
    inc = (float(In) / dd) * p.epsilon
    return _breakdown(lat, bw, comp, mem, inc, (((lat + bw) + comp) + mem) + inc)


def abc_table1_terms(kind: str, c: int, S: int):
    """Table 1, the (α,β,γ) model, as exact (A, B, C) Fractions."""
    F = Fraction
    if kind == "rb":
        return 2, F(2 * (c - 1) * S), F(2 * (c - 1) * S)
    if kind == "cps":
        return 2, F(2 * (c - 1) * S, c), F((c - 1) * S, c)
    if kind == "ring":
        return 2 * (c - 1), F(2 * (c - 1) * S, c), F((c - 1) * S, c)
    if kind == "rhd":
        chi = 0 if is_pow2(c) else 1
        return (2 * _ceil_log2(c), F(2 * (c - 1) * S, c) + chi * 2 * S,
                F((c - 1) * S, c) + chi * S)
    raise ValueError(kind)


def memory_lower_bound(c: int, S) -> Fraction:
    """Theorem 1 / Eq. 11: (N+1)S/N (times δ)."""
    return Fraction(c + 1, c) * S


def bandwidth_optimal_traffic(c: int, S) -> Fraction:
    """Eq. 2: 2(N−1)S/N."""
    return Fraction(2 * (c - 1), c) * S


def optimality_flags(kind: str, c: int, S: int, w_t: int, fanins=()) -> dict:
    """§3.3.1-3.3.2: δ-optimal iff D = (N+1)S/N exactly; ε-optimal iff the
    incast coefficient is 0."""
    A, Bn, Cn, Dn, In, den = closed_form_terms(kind, c, S, w_t, fanins)
    return {"delta_optimal": Fraction(Dn, den) == memory_lower_bound(c, S),
            "epsilon_optimal": In == 0}


def enumerate_hcps_factorizations(n: int, max_steps: int) -> list:
    """ordered factorizations, each f_i >= 2, 1 <= m <= max_steps; shorter lists
    first, then lexicographically descending."""
    found = []

    def rec(rem, pref):
        if rem == 1:
            if pref:
                found.append(tuple(pref))
            return
        if len(pref) == max_steps:
            return
        for d in range(2, rem + 1):
            if rem % d == 0:
                rec(rem // d, pref + [d])

    rec(n, [])
    out = []
    for m in range(1, max_steps + 1):
        out.extend(sorted((f for f in found if len(f) == m), reverse=True))
    return out


# ---------------------------------------------------------------- the executed plan (reading A6x)

def executed_steps(plan: Plan) -> list:
    """The plan as the executor runs it (reading A6x), as a list of steps, each a
    list of ops (rank, block, inputs, dests): rank computes block from `inputs` (summed in
    order; one input = a copy) and writes it to every rank in `dests`.

    A Reduce(r, b, I) of an RS step is the op (r, b, I, (r,)); the Transfers (r -> d, b) of an
    AG step with the same source and block form one op (r, b, (r,), (d1, d2, ...)) — the
    sender reads its block once and writes it to each peer ("each processor sends the block
    that it reduced to others").  Fusion rule ("one read / one write per element", SURVEY
    §8(a) row a4; the δ saving of P:402): when AG step s+1 directly follows RS step s, every
    transfer (r -> d, b) of step s+1 whose source r reduced block b in step s with fan-in >= 2
    is executed by that reduce — the reduced value goes from the reducer straight to d —
    and leaves step s+1.  If the fused step s would contain a hazard (an op writing a
    (rank, block) that another op of the step reads or writes; the concurrency rule of S:212),
    nothing of step s+1 is fused.  Ops on blocks of zero elements (N > count, reading Q3)
    move nothing and are not executed; steps left without ops vanish."""
    ops = []
    live = [block_size(plan.count, plan.n, b) > 0 for b in range(plan.n)]
    for st in plan.steps:
        if st.phase == "rs":
            ops.append([[rd.server, rd.block, tuple(rd.inputs), (rd.server,)] for rd in st.reduces if live[rd.block]])
        else:
            by = {}
            for t in st.transfers:
                if live[t.block]:
                    by.setdefault((t.src, t.block), []).append(t.dst)
            ops.append([[r, b, (r,), tuple(sorted(d))] for (r, b), d in sorted(by.items())])
    for s in range(len(plan.steps) - 1):
        if plan.steps[s].phase != "rs" or plan.steps[s + 1].phase != "ag":
            continue
        fused = [list(o) for o in ops[s]]
        rest = []
        for o in ops[s + 1]:
            r, b, _, dsts = o
            tgt = [f for f in fused if f[0] == r and f[1] == b and len(f[2]) >= 2]
            if tgt:
                tgt[0][3] = tgt[0][3] + dsts
            else:
                rest.append(o)
        if len(rest) == len(ops[s + 1]) or not _hazard_free(fused):
            continue
        ops[s], ops[s + 1] = fused, rest
    return [st for st in ops if st]


def _hazard_free(step_ops) -> bool:
    for i, (_, b, _, dsts) in enumerate(step_ops):
        for j, (_, b2, ins2, dsts2) in enumerate(step_ops):
            if i == j or b != b2:
                continue
            if set(dsts) & (set(ins2) | set(dsts2)):
                return False
    return True


def executed_step_coeffs(plan: Plan, esize: int) -> list:
    """Per-step GenModel coefficients of the executed plan (reading A6x; P:441-444 applied
    to executed_steps): the entry flag round first (A = 1, nothing moved: its α is the
    round trip that makes the inputs visible), then per executed step

      B = max over ranks of max(bytes into the rank, bytes out of it) — every input read from
          another rank moves bytes from it to the reader, every destination on another rank
          moves bytes from the writer to it; NVLink is full duplex, so a fused step's RS and
          AG traffic overlap ("data through a link");
      C = max over ranks of Σ (k − 1)·|block| over its ops with k >= 2 inputs;
      D = max over ranks of Σ (k + 1)·|block| over the same ops (copies 0);
      w = 1 + the most distinct ranks sending into one rank (reading Q8)."""
    n = plan.n
    out = [StepCoeffs(1, 0, 0, 0, 1)]
    for st in executed_steps(plan):
        inb, outb, cc, dd = [0] * n, [0] * n, [0] * n, [0] * n
        senders = [set() for _ in range(n)]
        for r, b, ins, dsts in st:
            L = block_size(plan.count, n, b) * esize
            for q in ins:
                if q != r:
                    inb[r] += L
                    outb[q] += L
                    senders[r].add(q)
            for d in dsts:
                if d != r:
                    outb[r] += L
                    inb[d] += L
                    senders[d].add(r)
            if len(ins) >= 2:
                cc[r] += (len(ins) - 1) * L
                dd[r] += (len(ins) + 1) * L
        out.append(StepCoeffs(1, max(max(inb), max(outb)), max(cc), max(dd),
                              1 + max(len(x) for x in senders)))
    return out


def executed_step_coeffs_shared(plan: Plan, esize: int) -> list:
    """The executed plan when ALL ranks share one GPU (emulated ranks, config C5's "8 ranks
    per GPU" on one device; reading A6e).  Every rank's data movement then goes through the
    same HBM, so a step costs its total memory traffic: D = Σ over ranks and ops of
    (k reads + one write per destination)·|block| (the memory-access term of P:402 summed
    over the ranks sharing the memory), C = Σ (k − 1)·|block| (the SMs are shared too), and
    no link term (B = 0, w = 1).  The entry round comes first, as in executed_step_coeffs."""
    n = plan.n
    out = [StepCoeffs(1, 0, 0, 0, 1)]
    for st in executed_steps(plan):
        cc = dd = 0
        for r, b, ins, dsts in st:
            L = block_size(plan.count, n, b) * esize
            dd += (len(ins) + len(dsts)) * L
            if len(ins) >= 2:
                cc += (len(ins) - 1) * L
        out.append(StepCoeffs(1, 0, cc, dd, 1))
    return out


def predict_executed(plan: Plan, esize: int, p: Params, shared: bool = False) -> dict:
    """GenModel of the executed plan, fixed-order float64 (the library's contract, bit for
    bit: genmodel_predict_executed / genmodel_predict_executed_shared)."""
    if plan.switch_reduce:   # NVLS plan: the NV1 row
        if shared:
            raise ValueError("an NVLS plan cannot run on ranks sharing one GPU")
        return closed_form_f64("nvls", plan.n, plan.count * esize, p)
    co = executed_step_coeffs_shared(plan, esize) if shared else executed_step_coeffs(plan, esize)
    return predict_f64(co, uniform_step_params(p, len(co)))
