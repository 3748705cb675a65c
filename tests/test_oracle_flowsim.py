"""Pins for oracle.flowsim, the incast-aware flow-level simulator (CPU).

Pinned against: one transfer over one link = α + Sβ (Eq. 7); the x-to-x test's cost
α + Sβ + max(x − w_t, 0)·S·ε (constant up to w_t, linear beyond); a textbook
max-min allocation worked by hand; the per-step GenModel evaluator (itself pinned to the
paper's tables) on every symmetric single-switch plan; the paper's printed single-switch rows
of tab:gentreesimu within 5 % (golden/gentreesimu.json); monotonicity in β and w_t; Ring's
zero incast.
"""
import json
import os
import random
from fractions import Fraction as F

import pytest

from oracle import flowsim as FS
from oracle import genmodel as G
from oracle import gentree as GT
from oracle import plans as P
from oracle import topology as T

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def link(alpha, beta, eps=0.0, w_t=9):
    return {"alpha": alpha, "beta": beta, "epsilon": eps, "w_t": w_t}


COMP0 = {"gamma": 0.0, "delta": 0.0}


def one_step(n, count, transfers, reduces=()):
    return P.Plan(n, count, [P.Step("rs", "s0", list(reduces), list(transfers))])


def test_single_transfer_is_alpha_plus_s_beta():
    topo = T.parse_topology(T.single_switch_doc(2, link(1e-3, 8e-9), COMP0))
    S = 1000                                   # floats
    plan = one_step(2, 2 * S, [P.Transfer(0, 1, 0, S)])
    r = FS.simulate_flows(topo, plan, 4)
    assert r["total"] == F(1e-3) + 4 * S * F(8e-9) / 4


@pytest.mark.parametrize("x", [2, 3, 5, 9, 10, 12, 16])
def test_x_to_x_incast_regime(x):
    """every communicator receives S from the other x-1; no overhead up to w_t,
    then max(x − w_t, 0)·S·ε (w = fan-in x, reading Q8)."""
    alpha, beta, eps, w_t = 2e-3, 4e-9, 1e-10, 9
    topo = T.parse_topology(T.single_switch_doc(x, link(alpha, beta, eps, w_t), COMP0))
    part = 120                                  # floats per (src, dst)
    tr = [P.Transfer(s, d, 0, part) for s in range(x) for d in range(x) if s != d]
    r = FS.simulate_flows(topo, one_step(x, x * 1000, tr), 4)
    S = F(4 * part * (x - 1))                   # bytes received per communicator
    want = F(alpha) + S * F(beta) / 4 + max(x - w_t, 0) * S * F(eps) / 4
    assert r["total"] == want
    assert (r["incast"] == 0) == (x <= w_t)


def test_textbook_max_min():
    """Two flows share s2's downlink (capacity C); flow A also crosses M0's uplink with
    capacity C/4.  Max-min: A = C/4, B = 3C/4.  A carries 100 bytes, B 300 bytes: both end at
    t = 400/C (A: 100/(C/4); B: 300/(3C/4)).  Then a second case with B = 600 bytes: B runs at
    3C/4 until t = 400/C (300 bytes done), then alone at C for 300/C more: 700/C."""
    beta = 8e-9                                  # per float -> C = 4/beta bytes/s
    fast = link(0.0, beta)
    slow = link(0.0, 4 * beta)
    vfast = link(0.0, beta / 128)                # never the bottleneck
    doc = {"nodes": [{"id": "R", "kind": "switch", "parent": None, "uplink": None},
                     {"id": "M0", "kind": "switch", "parent": "R", "uplink": slow},
                     {"id": "M1", "kind": "switch", "parent": "R", "uplink": vfast},
                     {"id": "s0", "kind": "server", "parent": "M0", "uplink": vfast, "compute": COMP0},
                     {"id": "s1", "kind": "server", "parent": "M1", "uplink": vfast, "compute": COMP0},
                     {"id": "s2", "kind": "server", "parent": "M1", "uplink": fast, "compute": COMP0}]}
    topo = T.parse_topology(json.dumps(doc))
    C = 4 / F(beta)
    r = FS.simulate_flows(topo, one_step(3, 300, [P.Transfer(0, 2, 0, 25), P.Transfer(1, 2, 1, 75)]), 4)
    assert r["total"] == 400 / C
    r = FS.simulate_flows(topo, one_step(3, 300, [P.Transfer(0, 2, 0, 25), P.Transfer(1, 2, 1, 150)]), 4)
    assert r["total"] == 700 / C


@pytest.mark.parametrize("w_t", [1, 5, 9, 64])
@pytest.mark.parametrize("kind,n", [("cps", 8), ("cps", 12), ("ring", 8), ("ring", 5), ("rhd", 8),
                                    ("rb", 6), ("hcps:4,2", 8), ("hcps:3,4", 12), ("hcps:2,2,2", 8)])
def test_symmetric_plans_equal_per_step_evaluator(kind, n, w_t):
    """On one switch with uniform parameters every step is symmetric, so max-min sharing gives
    each step B·β' and the simulation equals the pinned GenModel evaluator exactly."""
    p = G.Params(6.58e-3, 6.4e-9 / 4, 6e-10 / 4, 1.87e-10 / 4, 1.22e-10 / 4, w_t)
    topo = T.parse_topology(T.single_switch_doc(n, T.TABLE5["middle_sw"], T.TABLE5["server"]))
    plan = P.build_plan(kind, n, n * 720)
    sim = FS.simulate_flows(topo, plan, 4, p)
    ev = G.predict_exact(G.step_coeffs(plan, 4), G.uniform_step_params(p, len(plan.steps)))
    for k in ("latency", "compute", "memory", "total"):
        assert sim[k] == ev[k], k
    assert sim["bandwidth"] + sim["incast"] == ev["bandwidth"] + ev["incast"]


def test_tab_gentreesimu_single_switch_rows():
    gold = json.load(open(os.path.join(GOLD, "gentreesimu.json")))
    a3 = dict(T.TABLE5["middle_sw"], alpha=3 * 6.58e-3)
    worst = 0.0
    for name, n in (("SS24", 24), ("SS32", 32)):
        topo = T.parse_topology(T.single_switch_doc(n, a3, T.TABLE5["server"]))
        for alg, vals in gold[name].items():
            for S, want in zip(gold["sizes"], vals):
                plan, _ = GT.gentree(topo, S, 4, force=None if alg == "gentree" else alg)
                got = float(FS.simulate_flows(topo, plan, 4)["total"])
                worst = max(worst, abs(got / want - 1))
                assert abs(got / want - 1) < 0.05, (name, alg, S, got, want)
    assert worst > 0.005      # not a tautology: the paper's simulator is not our formula


def _random_tree(rnd, n_groups):
    nodes = [{"id": "R", "kind": "switch", "parent": None, "uplink": None}]
    k = 0
    for g in range(n_groups):
        nodes.append({"id": f"M{g}", "kind": "switch", "parent": "R",
                      "uplink": link(1e-4 * rnd.randint(1, 5), 1e-9 * rnd.randint(1, 8), 1e-11 * rnd.randint(0, 3),
                                     rnd.randint(2, 4))})
        for _ in range(rnd.randint(1, 4)):
            nodes.append({"id": f"s{k}", "kind": "server", "parent": f"M{g}",
                          "uplink": link(1e-4, 1e-9 * rnd.randint(1, 8), 1e-11, rnd.randint(2, 4)),
                          "compute": {"gamma": 1e-11, "delta": 1e-11}})
            k += 1
    return nodes


def test_monotone_in_beta_and_w_t():
    rnd = random.Random(7)
    for trial in range(6):
        nodes = _random_tree(rnd, rnd.randint(2, 3))
        topo = T.parse_topology(json.dumps({"nodes": nodes}))
        plan, _ = GT.gentree(topo, 600, 4)
        base = FS.simulate_flows(topo, plan, 4)["total"]
        victim = rnd.choice([x for x in nodes if x["uplink"] is not None])
        victim["uplink"] = dict(victim["uplink"], beta=victim["uplink"]["beta"] * 2)
        slower = FS.simulate_flows(T.parse_topology(json.dumps({"nodes": nodes})), plan, 4)["total"]
        assert slower >= base
        for x in nodes:
            if x["uplink"] is not None:
                x["uplink"] = dict(x["uplink"], w_t=x["uplink"]["w_t"] + 2)
        relaxed = FS.simulate_flows(T.parse_topology(json.dumps({"nodes": nodes})), plan, 4)["total"]
        assert relaxed <= slower


def test_ring_has_no_incast():
    """Ring generates no competing flows — fan-in 2 (Q8), so no incast for any w_t >= 2."""
    topo = T.parse_topology(T.single_switch_doc(12, dict(T.TABLE5["middle_sw"], w_t=2), T.TABLE5["server"]))
    plan = P.build_plan("ring", 12, 1200)
    assert FS.simulate_flows(topo, plan, 4)["incast"] == 0
