"""Pins for oracle.genmodel (CPU only).

Fixed by the paper: Table 1 vs Table 2 coefficient identities;
Theorem 1 as a bound over every built-in plan; Theorem 2 at plan
level; Eq. 6's monotonicity; the printed GenModel and (α,β,γ)
bars of fig:costmodel and its 2.6 % / 19.8 % error claims; SPEC's
hand-substituted worked examples.
"""
from fractions import Fraction

import pytest

from oracle import genmodel as G
from oracle import plans as P
from oracle import topology as T

Sf = 10 ** 8          # floats
Sb = 4 * Sf           # bytes


def table5_params():
    m, s = T.TABLE5["middle_sw"], T.TABLE5["server"]
    return G.params_per_float(m["alpha"], m["beta"], s["gamma"], s["delta"], m["epsilon"], m["w_t"])


@pytest.mark.parametrize("kind", ["cps", "ring", "rhd", "rb"])
@pytest.mark.parametrize("n", [2, 3, 5, 8, 12, 16, 24])
def test_table2_minus_new_terms_is_table1(kind, n):
    """dropping δ and ε from Table 2 reproduces Table 1 exactly (RB γ exempt, Q7)."""
    S = 1000
    A, Bn, Cn, Dn, In, den = G.closed_form_terms(kind, n, S, 9)
    a1, b1, c1 = G.abc_table1_terms(kind, n, S)
    assert A == a1
    assert Fraction(Bn, den) == b1
    if kind == "rb":
        assert 2 * Fraction(Cn, den) == c1        # Table 1 prints 2(N-1)S γ (Q7)
    else:
        assert Fraction(Cn, den) == c1


def test_hcps_reduces_to_cps():
    """Reading Q6: HCPS[N] must equal the CPS row, including incast."""
    for n in (4, 9, 12, 24):
        for wt in (2, 9, 30):
            assert G.closed_form_terms("hcps", n, 77, wt, (n,))[1:] == \
                   G.closed_form_terms("cps", n, 77, wt)[1:]


@pytest.mark.parametrize("n", range(2, 65))
def test_theorem1_memory_bound_all_kinds(n):
    """Theorem 1: every plan's memory term >= (N+1)S/N δ; equality for CPS; Ring = 3(N−1)S/N."""
    S = 1
    lb = G.memory_lower_bound(n, S)
    kinds = [("cps", ()), ("ring", ()), ("rhd", ()), ("rb", ())]
    kinds += [("hcps", f) for f in G.enumerate_hcps_factorizations(n, 3)]
    for name, f in kinds:
        A, Bn, Cn, Dn, In, den = G.closed_form_terms(name, n, S, 9, f)
        assert Fraction(Dn, den) >= lb
    assert Fraction(G.closed_form_terms("cps", n, S, 9)[3], n) == lb
    assert Fraction(G.closed_form_terms("ring", n, S, 9)[3], n) == Fraction(3 * (n - 1), n)


@pytest.mark.parametrize("n", range(2, 65))
def test_theorem2_plan_level(n):
    """with w_t = 9 no built-in plan is both δ- and ε-optimal when N > 9; CPS is
    both when N <= 9."""
    kinds = [("cps", ()), ("ring", ()), ("rb", ())]
    if P.is_pow2(n):
        kinds.append(("rhd", ()))
    kinds += [("hcps", f) for f in G.enumerate_hcps_factorizations(n, 3)]
    both = [k for k in kinds
            if all(G.optimality_flags(k[0], n, 1000, 9, k[1]).values())]
    if n > 9:
        assert both == []
    else:
        assert ("cps", ()) in both


def test_optimality_flags_examples():
    assert G.optimality_flags("cps", 24, 100, 9) == {"delta_optimal": True, "epsilon_optimal": False}
    assert G.optimality_flags("ring", 24, 100, 9) == {"delta_optimal": False, "epsilon_optimal": True}
    assert G.optimality_flags("cps", 4, 100, 9) == {"delta_optimal": True, "epsilon_optimal": True}


def test_eq6_per_op_cost_decreasing():
    """T(x)/(x−1) = ((x+1)/(x−1))Sδ + Sγ strictly decreasing; the δ share
    at x = 16 is <= 37.8 % of x = 2 ("saved by 66.7% at max")."""
    vals = [Fraction(x + 1, x - 1) + Fraction(1, 3) for x in range(2, 17)]
    assert all(a > b for a, b in zip(vals, vals[1:]))
    assert Fraction(17, 15) / 3 <= Fraction(378, 1000)
    assert 1 - Fraction(1, 3) == Fraction(2, 3)         # the 66.7 % limit


def test_spec_worked_examples(spec_examples):
    p = table5_params()
    cps = G.closed_form_exact("cps", 24, 4 * 10 ** 7, p)
    e = spec_examples["cps_24_1e7"]
    assert float(cps["total"]) == pytest.approx(e["total"], rel=e["rel_tol"])
    h = G.closed_form_exact("hcps", 24, 4 * 10 ** 7, p, (8, 3))
    e = spec_examples["hcps_8_3_24_1e7"]
    for key in ("total", "latency", "bandwidth", "compute", "memory"):
        assert float(h[key]) == pytest.approx(e[key], rel=e["rel_tol"])
    assert h["incast"] == 0


def costmodel_params():
    """SURVEY App. A back-solve of fig:costmodel: α = 4.0e-3 s, (2β+γ)S = 0.6638 s,
    Sδ = 0.0391 s, Sε = 0.01066 s, w_t = 9 (S = 1e8 floats)."""
    return G.Params(4.0e-3, 0.0, 0.0, 0.0391 / Sb, 0.01066 / Sb, 9, combined=0.6638 / Sb)


def test_fig_costmodel_genmodel_bars(golden):
    """All 10 printed GenModel predictions within 1.5 % (bars are printed to ~3 digits)."""
    p = costmodel_params()
    for n in ("12", "15"):
        for kind, v in golden["fig_costmodel"][n]["genmodel"].items():
            name, f = P.parse_kind(kind)
            got = float(G.closed_form_exact(name, int(n), Sb, p, f)["total"])
            assert got == pytest.approx(v, rel=0.015), (n, kind)


def test_fig_costmodel_abc_bars(golden):
    """The (α,β,γ) bars are reproduced exactly by Table 1 with α = 4e-3, (2β+γ)S = 0.66164
    (HCPS rows use 2mα + 2(N−1)S/N β + (N−1)S/N γ, i.e. Table 2 with δ = ε = 0)."""
    p = G.Params(4.0e-3, 0.0, 0.0, 0.0, 0.0, 9, combined=0.66164 / Sb)
    for n in ("12", "15"):
        for kind, v in golden["fig_costmodel"][n]["abc"].items():
            name, f = P.parse_kind(kind)
            got = float(G.closed_form_exact(name, int(n), Sb, p, f)["total"])
            assert got == pytest.approx(v, abs=2e-8), (n, kind)


def test_fig_costmodel_error_claims(golden):
    """max GenModel error 2.6 %, max (α,β,γ) error 19.8 %, error = |pred−meas|/meas."""
    eg, ea = [], []
    for n in ("12", "15"):
        d = golden["fig_costmodel"][n]
        for k, meas in d["measured"].items():
            eg.append(abs(d["genmodel"][k] - meas) / meas)
            ea.append(abs(d["abc"][k] - meas) / meas)
    assert round(max(eg), 3) == golden["fig_costmodel"]["max_error_genmodel"]
    assert round(max(ea), 3) == golden["fig_costmodel"]["max_error_abc"]


@pytest.mark.parametrize("kind", ["cps", "ring", "rhd", "hcps:4,2", "hcps:2,4", "hcps:2,2,2",
                                  "hcps:2,3", "hcps:3,2", "hcps:6,2", "hcps:2,2,3"])
@pytest.mark.parametrize("wt", [2, 3, 9])
def test_per_step_evaluator_equals_closed_form(kind, wt):
    """Per-step GenModel of a built plan ≡ Table 2 row on a uniform single switch, N | S,
    exact rationals."""
    name, f = P.parse_kind(kind)
    n = 8
    if name == "hcps":
        n = 1
        for x in f:
            n *= x
    S = n * 96
    p = G.Params(1e-6, 1e-9, 3e-10, 2e-10, 5e-11, wt)
    plan = P.build_plan(kind, n, S // 4)
    got = G.predict_exact(G.step_coeffs(plan, 4), G.uniform_step_params(p, plan.nsteps))
    ref = G.closed_form_exact(name, n, S, p, f)
    for key in ref:
        assert got[key] == ref[key], key


def test_rb_per_step_incast_is_half_of_printed():
    """Reading Q7: the broadcast step has w = 2, so the per-step evaluator charges incast on
    the reduce phase only: exactly half of Table 2's printed RB incast."""
    n, S = 12, 12 * 40
    p = G.Params(0, 1e-9, 0, 0, 1e-10, 3)
    plan = P.build_plan("rb", n, S // 4)
    got = G.predict_exact(G.step_coeffs(plan, 4), G.uniform_step_params(p, 2))
    ref = G.closed_form_exact("rb", n, S, p)
    assert got["incast"] * 2 == ref["incast"]
    assert got["bandwidth"] == ref["bandwidth"]


def test_f64_close_to_exact():
    p = table5_params()
    for kind in ("cps", "ring", "rhd", "rb"):
        for n in (4, 8, 24):
            ex = G.closed_form_exact(kind, n, Sb, p)
            fl = G.closed_form_f64(kind, n, Sb, p)
            assert abs(fl["total"] - float(ex["total"])) <= 1e-14 * float(ex["total"])


def test_factorizations(spec_examples):
    assert [list(f) for f in G.enumerate_hcps_factorizations(24, 2)] == \
           spec_examples["factorizations_24_2"]
    assert G.enumerate_hcps_factorizations(7, 2) == [(7,)]
    assert (3, 2, 2) in G.enumerate_hcps_factorizations(12, 3)


def test_hcps_memory_nonincreasing_in_f0():
    """§3.3: "the larger the prior steps' fan-in degrees, the less the memory
    access overhead" — for m = 2 and fixed N, D decreases as f0 grows."""
    for n in (12, 24, 36, 64):
        fs = [f for f in G.enumerate_hcps_factorizations(n, 2) if len(f) == 2]
        d = {f[0]: Fraction(G.closed_form_terms("hcps", n, 1, 99, f)[3], n) for f in fs}
        keys = sorted(d)
        assert all(d[a] >= d[b] for a, b in zip(keys, keys[1:]))


def _nvls_wire_bytes(n: int, S: int):
    """Brute-force byte count of the NVLS data movement (DESIGN.md §6 NVLS, reading NV1):
    owner r of block r issues one switch reduce (every GPU g ships its copy of block r into
    the switch; the sum comes back to r) and one multicast store (r ships the sum; the switch
    delivers it to every GPU).  Returns per-GPU (bytes out, bytes in)."""
    blk = S // n
    out = [0] * n
    inn = [0] * n
    for r in range(n):
        for g in range(n):            # multimem.ld_reduce: each GPU serves its copy
            out[g] += blk
        inn[r] += blk                 # reduced vector returns to the issuer
        out[r] += blk                 # multimem.st: issuer sends once
        for g in range(n):            # switch replicates to every GPU
            inn[g] += blk
    return out, inn


@pytest.mark.parametrize("n", [2, 3, 4, 8, 16])
def test_nvls_row_matches_wire_count(n):
    """NEXT #1 row: B = max per-GPU bytes per direction of the counted movement; C = D = I = 0;
    two latency rounds (reduce, multicast).  Also CPS's B by the same count ratio at N = 2."""
    S = n * 1000
    out, inn = _nvls_wire_bytes(n, S)
    A, Bn, Cn, Dn, In, den = G.closed_form_terms("nvls", n, S, 1)
    assert Fraction(Bn, den) == max(max(out), max(inn))
    assert (A, Cn, Dn, In) == (2, 0, 0, 0)
    p = G.Params(Fraction(3, 10**6), Fraction(7, 10**13), 0, 0, 0, 1)
    e = G.closed_form_exact("nvls", n, S, p)
    assert e["total"] == 2 * p.alpha + max(max(out), max(inn)) * p.beta
    # vs P2P CPS's 2(N-1)S/N (Eq. 2): more at N = 2, equal at 3, less from 4 on
    _, Bc, _, _, _, dc = G.closed_form_terms("cps", n, S, 99)
    assert (Fraction(Bn, den) > Fraction(Bc, dc)) == (n == 2)
    assert (Fraction(Bn, den) == Fraction(Bc, dc)) == (n == 3)


def test_nvls_fit_recovers_parameters():
    """fit_nvls on rows built from the wire count (not from the closed form) recovers α, β."""
    from oracle import fit as F
    alpha, beta = 11e-6, 1.75e-12
    rows = []
    for n in (2, 4, 8):
        for S in (1 << 20, 1 << 24, 1 << 28):
            out, inn = _nvls_wire_bytes(n, S)
            rows.append((n, S, 2 * alpha + max(max(out), max(inn)) * beta))
    f = F.fit_nvls(rows)
    assert f["alpha"] == pytest.approx(alpha, rel=1e-9)
    assert f["beta"] == pytest.approx(beta, rel=1e-9)


@pytest.mark.parametrize("n", [2, 3, 4, 8])
def test_oneshot_row_matches_line_count(n):
    """Reading OS1: count the one-shot path's traffic line by line — every rank writes each
    8-byte payload word of its S-byte input as one 16-byte line {d0, e, d1, e} into each of the
    N-1 peers' scratch — and its local work (all N blocks reduced from N inputs)."""
    S = 8 * 1000 * n
    lines = S // 8
    out = [0] * n
    inn = [0] * n
    for src in range(n):
        for dst in range(n):
            if dst != src:
                out[src] += 16 * lines
                inn[dst] += 16 * lines
    A, Bn, Cn, Dn, In, den = G.closed_form_terms("oneshot", n, S, 1 << 20)
    assert A == 1 and Fraction(Bn, den) == max(max(out), max(inn))
    assert Fraction(Cn, den) == (n - 1) * S and Fraction(Dn, den) == (n + 1) * S and In == 0
    # incast as CPS: every rank receives from N-1 senders (w = N, reading Q8)
    _, _, _, _, In2, den2 = G.closed_form_terms("oneshot", n, S, 1)
    assert Fraction(In2, den2) == max(n - 1, 0) * Fraction(Bn, den)


# ---------------------------------------------------------------- executed plan (reading A6x/A6e)

def _exact_executed(plan, p, shared=False):
    co = G.executed_step_coeffs_shared(plan, 4) if shared else G.executed_step_coeffs(plan, 4)
    return co, G.predict_exact(co, G.uniform_step_params(p, len(co)))


@pytest.mark.parametrize("n", [2, 3, 4, 5, 8, 12, 16])
@pytest.mark.parametrize("wt", [2, 5, 64])
def test_executed_cps_is_table2_row(n, wt):
    """CPS fuses its one RS step with its AG step, and the entry round takes the AG step's α:
    A = 2 and the full-duplex B of the fused step = 2(N−1)S/N — Table 2's CPS row
    term for term, incast included (w = N), exact rationals."""
    S = n * 96
    p = G.Params(1e-6, 1e-9, 3e-10, 2e-10, 5e-11, wt)
    _, got = _exact_executed(P.build_plan("cps", n, S // 4), p)
    ref = G.closed_form_exact("cps", n, S, p)
    for key in ref:
        assert got[key] == ref[key], key


@pytest.mark.parametrize("kind", ["ring", "rhd", "hcps:4,2", "hcps:2,4", "hcps:2,2,2", "hcps:3,2",
                                  "hcps:2,3", "hcps:2,2,3", "hcps:6,2"])
def test_executed_multistep_equals_table2_below_threshold(kind):
    """Ring / RHD / HCPS: the fused step moves RS and AG bytes at once, but since every rank
    sends and receives equally, max(in, out) summed over the executed steps equals Table 2's B
    (Eq. 2: 2(N−1)S/N); A (entry + executed steps) equals 2(N−1), 2·log N, 2m; C and D
    unchanged.  Exact when no step reaches the incast threshold."""
    name, f = P.parse_kind(kind)
    n = 8
    if name == "hcps":
        n = 1
        for x in f:
            n *= x
    S = n * 96
    p = G.Params(1e-6, 1e-9, 3e-10, 2e-10, 5e-11, 64)
    _, got = _exact_executed(P.build_plan(kind, n, S // 4), p)
    ref = G.closed_form_exact(name, n, S, p, f)
    for key in ref:
        assert got[key] == ref[key], key


@pytest.mark.parametrize("n", [2, 3, 4, 8, 12])
def test_executed_rb_halves_bandwidth_and_incast(n):
    """RB fused: the root pulls (N−1)S and pushes (N−1)S in the same step; full duplex makes
    B = (N−1)S, half of Table 2's 2(N−1)S, and the incast charged on it (w = N, the
    root's N−1 senders) half of the printed value; A, C, D as printed (γ = (N−1)S, Q7)."""
    S = n * 96
    p = G.Params(1e-6, 1e-9, 3e-10, 2e-10, 5e-11, 1)
    co, got = _exact_executed(P.build_plan("rb", n, S // 4), p)
    ref = G.closed_form_exact("rb", n, S, p)
    assert [c.A for c in co] == [1, 1]
    assert got["bandwidth"] * 2 == ref["bandwidth"]
    assert got["incast"] * 2 == ref["incast"]
    for key in ("latency", "compute", "memory"):
        assert got[key] == ref[key], key


def test_executed_ring4_hand_count():
    """Ring at N = 4, S bytes, hand-counted (reading Q10b: the AG runs the other way
    round the ring).  Entry; RS steps 0 and 1: each rank pulls S/4 from its left neighbour
    (B = S/4, C = S/4, D = 3S/4, w = 2); RS step 2 fused with AG step 0: it pulls S/4 and pushes
    its result S/4 to its right... neighbour in the reversed ring, receiving from both sides
    (B = S/2, w = 3); AG steps 1 and 2: copies of S/4 (B = S/4, C = D = 0, w = 2)."""
    S = 4 * 1000
    co = G.executed_step_coeffs(P.build_plan("ring", 4, S // 4), 4)
    q = S // 4
    assert [(c.A, c.B, c.C, c.D, c.w) for c in co] == [
        (1, 0, 0, 0, 1), (1, q, q, 3 * q, 2), (1, q, q, 3 * q, 2), (1, 2 * q, q, 3 * q, 3),
        (1, q, 0, 0, 2), (1, q, 0, 0, 2)]


def test_executed_rhd4_is_hcps22():
    """N = 4: RHD and HCPS[2,2] execute the same steps (SURVEY §8(c) degenerate identity),
    hand count: entry; S/2 pairwise reduce (B = S/2, C = S/2, D = 3S/2); fused S/4 reduce +
    S/4 send to the same partner (B = S/2, C = S/4, D = 3S/4); S/2 copy; all w = 2."""
    S = 4 * 1000
    h = S // 2
    want = [(1, 0, 0, 0, 1), (1, h, h, 3 * h, 2), (1, h, h // 2, 3 * h // 2, 2), (1, h, 0, 0, 2)]
    for kind in ("rhd", "hcps:2,2"):
        co = G.executed_step_coeffs(P.build_plan(kind, 4, S // 4), 4)
        assert [(c.A, c.B, c.C, c.D, c.w) for c in co] == want, kind


@pytest.mark.parametrize("n", [2, 3, 4, 8, 16])
def test_executed_shared_hbm_bytes(n):
    """Reading A6e (all ranks on one GPU): the memory term counts every byte any rank reads or
    writes.  CPS: each rank buffer is read once and written once, D = 2·N·S (bench.py's
    algorithmic bytes); Ring: per rank (N−1) two-input reduces (3 block accesses each), one
    extra fused write and N−2 copies (2 accesses each): D = (5N − 6)·S; RB: the root reads N
    buffers and writes N: D = 2·N·S.  C = Σ (k − 1)|b| = (N−1)·S for all three."""
    S = n * 96
    for kind, dmul in (("cps", 2 * n), ("ring", 5 * n - 6), ("rb", 2 * n)):
        co = G.executed_step_coeffs_shared(P.build_plan(kind, n, S // 4), 4)
        assert sum(c.D for c in co) == dmul * S, kind
        assert sum(c.C for c in co) == (n - 1) * S, kind
        assert all(c.B == 0 and c.w == 1 for c in co)


def test_executed_fusion_refused_on_hazard():
    """The fusion rule's hazard clause: an AG step whose transfer would make the fused RS
    step write a (rank, block) another op of that step reads is left unfused."""
    n, count = 2, 8
    rs = P.Step("rs", "x", [P.Reduce(0, 0, (0, 1)), P.Reduce(1, 1, (0, 1))])
    P.add_implied_transfers(rs, count, n)
    # rank 0 sends block 0 to rank 1 — but rank 1's reduce of step 0 reads only block 1, so
    # this one fuses; a transfer of block 1 from rank 0 (who did not reduce it) cannot
    ag = P.Step("ag", "y", [], [P.Transfer(0, 1, 0, 4), P.Transfer(1, 0, 1, 4)])
    ex = G.executed_steps(P.Plan(n, count, [rs, ag]))
    assert len(ex) == 1 and sorted(tuple(o) for o in ex[0]) == [(0, 0, (0, 1), (0, 1)), (1, 1, (0, 1), (1, 0))]
    # N = 3: rank 2's reduce of block 0 reads (1, 0); fusing rank 0's send of block 0 to rank 1
    # would write (1, 0) in the same step -> no fusion at all (both RS steps are hazard-free)
    n3, c3 = 3, 9
    rs2 = P.Step("rs", "x", [P.Reduce(0, 0, (0, 1)), P.Reduce(2, 0, (1, 2))])
    P.check_step_hazards(rs2)
    P.add_implied_transfers(rs2, c3, n3)
    ag2 = P.Step("ag", "y", [], [P.Transfer(0, 1, 0, 3)])
    assert len(G.executed_steps(P.Plan(n3, c3, [rs2, ag2]))) == 2


@pytest.mark.parametrize("n", [2, 3, 4, 8])
def test_ll128_row_matches_line_count(n):
    """The LL128 row (measured-protocol), counted line by line: every rank writes
    its slice of each of the N-1 other blocks, then its reduced block to each of the N-1 peers,
    as 128-byte lines carrying 120 payload bytes; it reduces its own block from N inputs."""
    S = 120 * 16 * n          # bytes per rank: whole lines per block
    blk = S // n
    lines = -(-blk // 120)
    out = [0] * n
    inn = [0] * n
    for r in range(n):
        for o in range(n):
            if o != r:
                out[r] += 128 * lines          # RS: my slice of block o -> owner o
                inn[o] += 128 * lines
                out[o] += 128 * lines          # AG: owner o's result -> me
                inn[r] += 128 * lines
    A, Bn, Cn, Dn, In, den = G.closed_form_terms("ll128", n, S, 1 << 20)
    assert A == 1 and Fraction(Bn, den) == max(max(out), max(inn))
    assert Fraction(Cn, den) == Fraction((n - 1) * S, n) and Fraction(Dn, den) == Fraction((n + 1) * S, n)
    assert In == 0
    _, _, _, _, In2, den2 = G.closed_form_terms("ll128", n, S, 1)
    assert Fraction(In2, den2) == (n - 1) * Fraction(Bn, den)
