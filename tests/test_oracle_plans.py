"""Pins for oracle.topology and oracle.plans (CPU only).

Every assertion is fixed by the paper/SPEC text or by mathematics, not by re-running the
oracle's own code path: step counts = Table 2's A coefficients, per-rank traffic
= Eq. 2, memory coefficients = Table 2's D, the tag
conservation invariant with mutations, structural identities.
"""
import json
import random
from fractions import Fraction

import pytest

from oracle import plans as P
from oracle import topology as T


# ------------------------------------------------------------------ topology

def test_parse_single_switch_24():
    t = T.parse_topology(T.single_switch_doc(24, T.TABLE5["middle_sw"], T.TABLE5["server"]))
    assert len(t.servers) == 24 and t.root == "sw"
    assert t.servers_under("s3") == ["s3"]


def test_parse_sym384():
    doc = T.two_level_doc([24] * 16, T.TABLE5["root_sw"], T.TABLE5["middle_sw"], T.TABLE5["server"])
    t = T.parse_topology(doc)
    assert len(t.servers) == 384
    assert len(t.servers_under("M3")) == 24
    assert t.ranks_under("M1") == list(range(24, 48))


@pytest.mark.parametrize("mutate, msg", [
    (lambda d: d["nodes"].__delitem__(slice(2, None)), "fewer than 2"),
    (lambda d: d["nodes"][1].__setitem__("bogus", 1), "unknown keys"),
    (lambda d: d["nodes"][1].__setitem__("parent", "nope"), "does not exist"),
    (lambda d: d["nodes"].append({"id": "lone", "kind": "switch", "parent": "sw",
                                  "uplink": T.TABLE5["root_sw"]}), "leaf"),
    (lambda d: d["nodes"][1].__setitem__("compute", None), "compute"),
    (lambda d: d["nodes"][0].__setitem__("parent", "s0"), "root"),
    (lambda d: d["nodes"][1]["uplink"].__setitem__("w_t", 0), "w_t"),
])
def test_parse_rejects(mutate, msg):
    d = json.loads(T.single_switch_doc(3, T.TABLE5["middle_sw"], T.TABLE5["server"]))
    mutate(d)
    with pytest.raises(T.TopologyError):
        T.parse_topology(json.dumps(d))


def test_parse_rejects_cycle_and_syntax():
    nodes = [{"id": "a", "kind": "switch", "parent": "b", "uplink": T.TABLE5["root_sw"]},
             {"id": "b", "kind": "switch", "parent": "a", "uplink": T.TABLE5["root_sw"]},
             {"id": "r", "kind": "switch", "parent": None, "uplink": None},
             {"id": "s0", "kind": "server", "parent": "r", "uplink": T.TABLE5["middle_sw"],
              "compute": T.TABLE5["server"]},
             {"id": "s1", "kind": "server", "parent": "r", "uplink": T.TABLE5["middle_sw"],
              "compute": T.TABLE5["server"]}]
    with pytest.raises(T.TopologyError):
        T.parse_topology(json.dumps({"nodes": nodes}))
    with pytest.raises(T.TopologyError):
        T.parse_topology("{not json")


def test_convergence_ratio(spec_examples):
    t = T.parse_topology(T.single_switch_doc(4, T.TABLE5["middle_sw"], T.TABLE5["server"]))
    assert t.convergence_ratio_f64("sw", "s2") == spec_examples["convergence"]["equal4"]
    d = json.loads(T.single_switch_doc(3, T.TABLE5["middle_sw"], T.TABLE5["server"]))
    for nd, b in zip(d["nodes"][1:], (1e-9, 1e-9, 2e-9)):
        nd["uplink"]["beta"] = b
    t = T.parse_topology(json.dumps(d))
    assert t.convergence_ratio_f64("sw", "s2") == pytest.approx(5, rel=1e-15)
    # exact rationals (reading Q15): 2e-9 is exactly 2 x 1e-9 in binary, so r = 2e-9 *
    # (2/1e-9 + 1/2e-9) = 5 exactly, and equal uplinks give r = the child count exactly
    from fractions import Fraction
    assert t.convergence_ratio("sw", "s2") == 5
    assert t.convergence_ratio("sw", "s0") == Fraction(5, 2)
    t4 = T.parse_topology(T.single_switch_doc(4, T.TABLE5["middle_sw"], T.TABLE5["server"]))
    assert t4.convergence_ratio("sw", "s2") == 4
    # 6.4e-9 is not exactly 10 x 6.4e-10 in binary: the exact ratio differs from 10
    d2 = json.loads(T.single_switch_doc(2, T.TABLE5["middle_sw"], T.TABLE5["server"]))
    d2["nodes"][1]["uplink"]["beta"], d2["nodes"][2]["uplink"]["beta"] = 6.4e-10, 6.4e-9
    r = T.parse_topology(json.dumps(d2)).convergence_ratio("sw", "s1")
    assert r == Fraction(6.4e-9) * (Fraction(1) / Fraction(6.4e-10) + Fraction(1) / Fraction(6.4e-9))
    assert r != 11


# ------------------------------------------------------------------ blocks

@pytest.mark.parametrize("count,n", [(10, 3), (7, 8), (1, 2), (1 << 20, 8), (1000003, 7)])
def test_blocks_partition(count, n):
    sizes = [P.block_size(count, n, b) for b in range(n)]
    assert sum(sizes) == count
    assert max(sizes) - min(sizes) <= 1
    assert sizes == sorted(sizes, reverse=True)          # first count % n get the extra one
    for b in range(1, n):
        assert P.block_offset(count, n, b) == P.block_offset(count, n, b - 1) + sizes[b - 1]


# ------------------------------------------------------------------ step counts (Table 2 A)

def ceil_log2(n):
    k = 0
    while (1 << k) < n:
        k += 1
    return k


@pytest.mark.parametrize("n", range(2, 33))
def test_step_counts_and_conservation(n):
    assert P.build_plan("cps", n, 5 * n + 1).nsteps == 2            # P:462 "2α"
    assert P.build_plan("rb", n, 3 * n).nsteps == 2
    assert P.build_plan("ring", n, 2 * n + 3).nsteps == 2 * (n - 1)
    assert P.build_plan("rhd", n, 4 * n).nsteps == 2 * ceil_log2(n)
    for kind in ("cps", "rb", "ring", "rhd"):
        P.verify_allreduce(P.build_plan(kind, n, 3 * n + 2))


@pytest.mark.parametrize("f", [(2, 2), (4, 2), (2, 4), (2, 2, 2), (6, 4), (3, 5), (5, 3),
                               (2, 3, 4), (8, 3), (8, 4), (4, 3, 2)])
def test_hcps_steps_and_conservation(f):
    n = 1
    for x in f:
        n *= x
    p = P.build_plan("hcps:" + ",".join(map(str, f)), n, 2 * n + 1)
    assert p.nsteps == 2 * len(f)                                    # P:463 "2mα"
    P.verify_allreduce(p)


def test_fig4_hcps_6x4_groups():
    """Figure 4: 6x4 HCPS — step 1 groups of 6, step 2 orthogonal groups of 4."""
    p = P.build_plan("hcps:6,4", 24, 24)
    g0 = {tuple(r.inputs) for r in p.steps[0].reduces}
    g1 = {tuple(r.inputs) for r in p.steps[1].reduces}
    assert all(len(g) == 6 for g in g0) and len(g0) == 4
    assert all(len(g) == 4 for g in g1) and len(g1) == 6
    for a in g0:
        for b in g1:
            assert len(set(a) & set(b)) == 1                           # orthogonal


# ------------------------------------------------------------------ mutations

def test_mutation_detected():
    p = P.build_plan("ring", 5, 20)
    P.verify_allreduce(p)
    rnd = random.Random(7)
    for _ in range(30):
        q = P.Plan(p.n, p.count, [P.Step(s.phase, s.label, list(s.reduces), list(s.transfers))
                                  for s in p.steps])
        si = rnd.randrange(len(q.steps))
        st = q.steps[si]
        if st.phase == "ag":
            del st.transfers[rnd.randrange(len(st.transfers))]
        else:
            i = rnd.randrange(len(st.reduces))
            rd = st.reduces[i]
            st.reduces[i] = P.Reduce(rd.server, rd.block, rd.inputs[:1])
        with pytest.raises(P.PlanError):
            P.verify_allreduce(q)


def test_double_count_detected():
    p = P.build_plan("cps", 3, 9)
    rd = p.steps[0].reduces[0]
    p.steps[0].reduces[0] = P.Reduce(rd.server, rd.block, rd.inputs + (rd.inputs[0],))
    with pytest.raises(P.PlanError, match="duplicate"):
        P.verify_allreduce(p)


def test_reverse_involution():
    for kind in ("cps", "ring", "rhd", "hcps:2,3"):
        p = P.build_plan(kind, 6, 61) if kind != "rhd" else P.build_plan(kind, 8, 61)
        rs = [s for s in p.steps if s.phase == "rs"]
        ag = P.reverse_to_allgather(rs)
        back = P.reverse_to_allgather(ag)
        assert [sorted(s.transfers, key=str) for s in back] == \
               [sorted(s.transfers, key=str) for s in rs]


# ------------------------------------------------------------------ Eq. 2 and Table 2's D

@pytest.mark.parametrize("kind,n", [("cps", 8), ("ring", 8), ("rhd", 8), ("hcps:4,2", 8),
                                    ("hcps:2,2,2", 8), ("cps", 12), ("ring", 7),
                                    ("hcps:3,4", 12), ("rhd", 16)])
def test_bandwidth_optimal_traffic(kind, n):
    S = n * 60
    agg = P.plan_aggregates(P.build_plan(kind, n, S))
    for a in agg:                      # Eq. 2: sends and receives 2(N-1)S/N each
        assert a["sent"] == 2 * (n - 1) * S // n
        assert a["received"] == 2 * (n - 1) * S // n


def hcps_D(f, n):
    """Reading Q5 written out: (2 Σ_{i=1}^{m-1} Π_{j=i}^{m-1} f_j + N + 1) / N."""
    m = len(f)
    s = 0
    for i in range(1, m):
        p = 1
        for j in range(i, m):
            p *= f[j]
        s += p
    return Fraction(2 * s + n + 1, n)


@pytest.mark.parametrize("kind,n,coef", [
    ("cps", 8, Fraction(9, 8)), ("ring", 8, Fraction(21, 8)), ("rhd", 8, Fraction(21, 8)),
    ("hcps:4,2", 8, Fraction(13, 8)), ("hcps:2,4", 8, Fraction(17, 8)),
    ("hcps:2,2,2", 8, Fraction(21, 8)), ("cps", 24, Fraction(25, 24)),
    ("hcps:6,4", 24, hcps_D((6, 4), 24)), ("hcps:2,3,4", 24, hcps_D((2, 3, 4), 24))])
def test_memory_coefficient(kind, n, coef):
    """D summed over the critical rank = Table 2's memory coefficient x S (P:402-403,
    P:460-463); C4's factors 9/13/17/21."""
    S = n * 48
    agg = P.plan_aggregates(P.build_plan(kind, n, S))
    assert {a["mem_ops"] for a in agg} == {coef * S}
    assert {a["compute_ops"] for a in agg} == {Fraction(n - 1, n) * S}


def test_spec_cps_aggregates(spec_examples):
    p = P.build_plan("cps", 4, 4)
    rs = P.Plan(4, 4, [s for s in p.steps if s.phase == "rs"])
    exp = spec_examples["aggregates_cps_4_4"]
    for a in P.plan_aggregates(rs):
        assert (a["sent"], a["received"], a["mem_ops"], a["compute_ops"]) == \
               (exp["sent"], exp["received"], exp["mem_ops"], exp["compute_ops"])


# ------------------------------------------------------------------ structural identities

def _rs_multiset(p):
    return [sorted((r.server, r.block, r.inputs) for r in s.reduces)
            for s in p.steps if s.phase == "rs"]


def test_degenerate_n2_identical():
    """CPS(2) ≡ RHD(2) ≡ HCPS[2] ≡ Ring(2)."""
    ref = _rs_multiset(P.build_plan("cps", 2, 11))
    for k in ("rhd", "hcps:2", "ring"):
        assert _rs_multiset(P.build_plan(k, 2, 11)) == ref


@pytest.mark.parametrize("n", [3, 5, 8, 12])
def test_hcps_single_level_is_cps(n):
    assert _rs_multiset(P.build_plan(f"hcps:{n}", n, 3 * n)) == \
           _rs_multiset(P.build_plan("cps", n, 3 * n))


@pytest.mark.parametrize("k", [1, 2, 3, 4])
def test_hcps_all_twos_is_rhd(k):
    n = 1 << k
    assert _rs_multiset(P.build_plan("hcps:" + ",".join(["2"] * k), n, 5 * n)) == \
           _rs_multiset(P.build_plan("rhd", n, 5 * n))


def test_rhd_owner_is_bitrev():
    """Reading Q11: after the RS, block b is owned by bitrev(b)."""
    p = P.build_plan("rhd", 8, 8)
    last = [s for s in p.steps if s.phase == "rs"][-1]
    own = {r.block: r.server for r in last.reduces}
    assert own == {b: int(f"{b:03b}"[::-1], 2) for b in range(8)}


def test_ring_owner_after_rs():
    """Reading Q10: with P:143's indices, rank i finishes the RS owning block (i+2) mod N."""
    n = 6
    p = P.build_plan("ring", n, n)
    last = [s for s in p.steps if s.phase == "rs"][-1]
    assert {r.server: r.block for r in last.reduces} == {i: (i + 2) % n for i in range(n)}
    # in step j, processor i receives block (i-j) mod N from the left neighbour
    for j, st in enumerate(s for s in p.steps if s.phase == "rs"):
        for t in st.transfers:
            assert t.src == (t.dst - 1) % n and t.block == (t.dst - j) % n


def test_canonical_json_deterministic():
    p = P.build_plan("hcps:2,3", 6, 17)
    a, b = P.plan_to_json(p, "f32"), P.plan_to_json(P.build_plan("hcps:2,3", 6, 17), "f32")
    assert a == b and json.loads(a)["n"] == 6 and " " not in a


def test_acps_identity_and_swap():
    assert P.build_acps({0: {0}, 1: {1}}, {0: [0], 1: [1]}, 2, 2) == []
    st = P.build_acps({0: {0, 1}, 1: {0, 1}}, {0: [1], 1: [0]}, 2, 2)
    assert len(st) == 1 and len(st[0].transfers) == 2 and len(st[0].reduces) == 2
