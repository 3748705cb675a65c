"""Host-side executor logic on CPU: the step tables `allreduce_exec` launches
(ar_plan_lowering_json) are run by a CTA-level interpreter of the kernel's flag protocol
under random schedules, and must produce the oracle's result with no deadlock.

The interpreter models what the kernel does: every rank runs its step list on C CTAs; a CTA
may start a step only when its waits are satisfied (paired: the producer's same-index CTA
has posted the slot for this call; full: all producer CTAs have); it then executes its slice
of every op (sources read, summed left to right in fp32, written to every destination) and
posts the step's slot to every consumer.  A rank's call k+1 starts only after all its CTAs
finished call k (stream order).  Random interleavings expose any missing dependency (RAW,
WAR, WAW, across steps or across calls) as a wrong result."""
import random

import numpy as np
import pytest

import paper_2409_04202_b200 as G
from oracle import gentree as GT
from oracle import simulate as SM
from oracle import topology as T
from synth import generator as GEN


def single_switch(world):
    return T.single_switch_doc(world, {"alpha": 3e-6, "beta": 4 / 900e9, "epsilon": 0.0, "w_t": 9},
                               {"gamma": 0.0, "delta": 4 / 6.54e12})


def cta_elems(off, len_, esize, k, C):
    """The kernel's slicing rule (exec.cu cta_elems): whole 16-byte vectors split evenly and
    contiguously over C CTAs, CTA 0 adds the unaligned head, CTA C-1 the tail."""
    E = 16 // esize
    vb, ve = (off * esize + 15) // 16, (off + len_) * esize // 16
    if vb >= ve:
        return (off, off + len_) if k == 0 else (0, 0)
    nv = ve - vb
    e0, e1 = (vb + nv * k // C) * E, (vb + nv * (k + 1) // C) * E
    if k == 0:
        e0 = off
    if k == C - 1:
        e1 = off + len_
    return e0, e1


def interpret(low: dict, inputs: list, ctas: int, calls: int, rnd: random.Random, esize: int = 4,
              avg: bool = False) -> list:
    n = len(low["ranks"])
    bufs = [x.astype(np.float32).copy() for x in inputs]
    flags = {}                                  # (consumer, slot, producer, cta) -> epoch
    pc = [[0] * ctas for _ in range(n)]         # step index per CTA
    epoch = [[1] * ctas for _ in range(n)]      # call number per CTA
    done = [[False] * ctas for _ in range(n)]

    def runnable(r, c):
        if done[r][c]:
            return False
        prog = low["ranks"][r]["steps"]
        if pc[r][c] == 0 and epoch[r][c] > 1:
            # stream order: call k+1 starts after every CTA of this rank finished call k
            if any(epoch[r][cc] < epoch[r][c] for cc in range(ctas)):
                return False
        st = prog[pc[r][c]]
        e = epoch[r][c]
        for (t, slot, kind, p_off, p_len, c_off, c_len) in st["waits"]:
            if kind == 0:
                cs = [c]
            elif kind == 1:
                cs = range(ctas)
            else:
                m0, m1 = cta_elems(c_off, c_len, esize, c, ctas)
                cs = []
                for k in range(ctas):
                    p0, p1 = cta_elems(p_off, p_len, esize, k, ctas)
                    if m0 < m1 and p0 < p1 and m0 < p1 and p0 < m1:
                        cs.append(k)
            if any(flags.get((r, slot, t, cc), 0) < e for cc in cs):
                return False
        return True

    def step(r, c):
        st = low["ranks"][r]["steps"][pc[r][c]]
        for op in st["ops"]:
            lo, hi = cta_elems(op["off"], op["len"], esize, c, ctas)
            if hi <= lo:
                continue
            acc = bufs[op["src"][0]][lo:hi].copy()
            for q in op["src"][1:]:
                acc = acc + bufs[q][lo:hi]
            if avg and op["fin"]:
                acc = acc / np.float32(n)
            for d in op["dst"]:
                bufs[d][lo:hi] = acc
        for consumer in st["notify"]:
            flags[(consumer, st["slot"], r, c)] = epoch[r][c]
        pc[r][c] += 1
        if pc[r][c] == len(low["ranks"][r]["steps"]):
            if epoch[r][c] == calls:
                done[r][c] = True
            else:
                epoch[r][c] += 1
                pc[r][c] = 0

    agents = [(r, c) for r in range(n) for c in range(ctas)]
    while True:
        ready = [a for a in agents if runnable(*a)]
        if not ready:
            assert all(done[r][c] for r, c in agents), "deadlock in the lowered flag protocol"
            return bufs
        step(*rnd.choice(ready))


CASES = [(single_switch(w), w, k) for w in (2, 3, 4, 8) for k in (None, "cps", "ring", "rb")]
CASES += [(single_switch(8), 8, k) for k in ("rhd", "hcps:4,2", "hcps:2,4", "hcps:2,2,2")]
CASES += [(single_switch(6), 6, k) for k in ("hcps:3,2", "hcps:2,3")]
from tests.topologies import cross_dc  # noqa: E402

CASES += [(cross_dc(2, 2, 2, 2), 8, None), (cross_dc(2, 4, 2, 2), 12, None)]
CASES += [(T.two_level_doc([2, 2], T.TABLE5["root_sw"], T.TABLE5["middle_sw"], T.TABLE5["server"]), 4, None),
          (T.two_level_doc([3, 4], T.TABLE5["root_sw"], T.TABLE5["middle_sw"], T.TABLE5["server"]), 7, None),
          (T.two_level_doc([2, 2, 2], T.TABLE5["root_sw"], T.TABLE5["middle_sw"], T.TABLE5["server"]), 6, None)]


@pytest.mark.parametrize("doc,world,force", CASES)
def test_lowered_protocol_random_schedules(doc, world, force):
    count = 37 * world + 5
    plan = G.Plan.from_topology(doc, count, "f32", None, force)
    low = plan.lowering()
    oplan, _ = GT.gentree(T.parse_topology(doc), count, 4, force=force)
    xs = [(GEN.generate(3, r, count, "f32", "integer")) for r in range(world)]
    want = SM.simulate(oplan, SM.simulate(oplan, xs, "f32"), "f32")
    rnd = random.Random(world * 100 + len(force or ""))
    for trial in range(6):
        got = interpret(low, xs, ctas=rnd.choice([1, 2, 3, 5]), calls=2, rnd=rnd)
        for r in range(world):
            assert np.array_equal(got[r], want[r]), (force, trial, r)


def test_cps_is_one_fused_step_with_two_flag_rounds():
    """CPS lowers to entry -> one fused pull-reduce-push op -> exit: the AG step disappears
    (P:402's one read/one write per element; A = 2 flag round trips)."""
    low = G.Plan.from_topology(single_switch(8), 8000, "bf16", None, "cps").lowering()
    for r, rk in enumerate(low["ranks"]):
        slots = [s["slot"] for s in rk["steps"]]
        assert slots == [0, 1, 0]
        entry, work, exit_ = rk["steps"]
        assert sorted(entry["notify"]) == [q for q in range(8) if q != r]
        (op,) = work["ops"]
        assert op["src"] == list(range(8)) and sorted(op["dst"]) == list(range(8)) and op["dst"][0] == r
        assert all(w[2] == 0 for w in exit_["waits"]) and len(exit_["waits"]) == 7


def test_lowering_rejects_bad_buffer_query():
    plan = G.Plan.from_topology(single_switch(2), 10, "f32")
    assert plan.lowering()["ranks"][1]["steps"]


@pytest.mark.parametrize("doc,world,force", [c for c in CASES if c[2] in ("ring", "hcps:3,2", "rb", None)])
def test_lowered_avg_divides_once_at_the_final_reduce(doc, world, force):
    """AR_OP_AVG (reading AV1): the lowering's `fin` ops are exactly the plan's last RS
    reduces of each block (the interpreter divides there) — two AVG calls match the oracle."""
    count = 29 * world + 3
    plan = G.Plan.from_topology(doc, count, "f32", None, force)
    low = plan.lowering()
    oplan, _ = GT.gentree(T.parse_topology(doc), count, 4, force=force)
    xs = [(GEN.generate(5, r, count, "f32", "gradient")) for r in range(world)]
    want = SM.simulate(oplan, SM.simulate(oplan, xs, "f32", op="avg"), "f32", op="avg")
    rnd = random.Random(world * 7 + 1)
    for trial in range(3):
        got = interpret(low, xs, ctas=rnd.choice([1, 2, 3]), calls=2, rnd=rnd, avg=True)
        for r in range(world):
            assert np.array_equal(got[r].view(np.uint32), want[r].view(np.uint32)), (force, trial, r)


def test_full_waits_variant_is_also_correct(monkeypatch):
    """AR_WAITS=full (the A/B baseline of the range waits) replaces every inter-step range wait
    by a wait on all producer CTAs; the protocol stays correct under random schedules."""
    monkeypatch.setenv("AR_WAITS", "full")
    doc, world = single_switch(8), 8
    for force in ("ring", "hcps:4,2", "rhd"):
        count = 37 * world + 5
        plan = G.Plan.from_topology(doc, count, "f32", None, force)
        low = plan.lowering()
        kinds = {w[2] for r in low["ranks"] for st in r["steps"] for w in st["waits"]}
        assert 2 not in kinds and 1 in kinds
        oplan, _ = GT.gentree(T.parse_topology(doc), count, 4, force=force)
        xs = [GEN.generate(3, r, count, "f32", "integer") for r in range(world)]
        want = SM.simulate(oplan, SM.simulate(oplan, xs, "f32"), "f32")
        rnd = random.Random(5)
        got = interpret(low, xs, ctas=3, calls=2, rnd=rnd)
        for r in range(world):
            assert np.array_equal(got[r], want[r])


def test_lowering_rejects_oversized_ops():
    """A plan that fails verification with duplicated inputs (fan-in 100 at N = 2) loads as a
    data-movement plan but cannot be lowered: the kernel's per-op source table holds
    AR_MAX_RANKS entries (such a plan used to overrun OpShared::src)."""
    import json
    world, count = 2, 1024
    bad = {"count": count, "dtype": "f32", "n": world, "steps": [
        {"label": "rs", "phase": "rs", "transfers": [],
         "reduces": [{"block": b, "fan_in": 100, "inputs": [0] * 50 + [1] * 50, "server": b}
                     for b in range(world)]}]}
    plan = G.Plan.from_json(json.dumps(bad))
    assert not plan.is_allreduce
    with pytest.raises(Exception, match="AR_MAX_RANKS"):
        plan.lowering()
