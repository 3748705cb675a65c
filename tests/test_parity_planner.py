"""Library (C-ABI, host planning core) vs oracle: plan structure and costs (CPU only).

The bar (BASELINE.json north star): plan generation and cost predictions are bit-exact —
canonical plan JSON byte-identical, GenModel doubles bit-identical (fixed evaluation order,
DESIGN.md).  Fits are compared within 1e-9 relative on noiseless data.
"""
import json
import random
import struct

import pytest

import paper_2409_04202_b200 as G
from oracle import fit as OF
from oracle import genmodel as OG
from oracle import gentree as GT
from oracle import plans as OP
from oracle import topology as T
from tests.test_oracle_gentree import _gtplan_topos, _random_tree, row

ES = {"f32": 4, "bf16": 2}


def bits(x: float) -> int:
    return struct.unpack("<Q", struct.pack("<d", x))[0]


def same_breakdown(a: dict, b: dict):
    for k in ("latency", "bandwidth", "compute", "memory", "incast", "total"):
        assert bits(a[k]) == bits(b[k]), (k, a[k], b[k])


def lib_params(p: OG.Params) -> G.GmParams:
    return G.params(p.alpha, p.beta, p.gamma, p.delta, p.epsilon, p.w_t, p.combined)


def check_topology(doc, count, dtype="f32", params=None, force=None):
    t = T.parse_topology(doc)
    oplan, oreps = GT.gentree(t, count, ES[dtype], params=params, force=force)
    lplan = G.Plan.from_topology(doc, count, dtype, lib_params(params) if params else None, force)
    assert lplan.to_json() == OP.plan_to_json(oplan, dtype)
    lrep = lplan.report()
    assert [r["chosen"] for r in lrep] == [r.chosen for r in oreps]
    for lr, orp in zip(lrep, oreps):
        assert lr["switch"] == orp.switch
        assert lr["rearranged_children"] == orp.rearranged_children
        assert [c["kind"] for c in lr["candidates"]] == [k for k, _ in orp.candidates]
        for c, (_, v) in zip(lr["candidates"], orp.candidates):
            assert bits(c["total"]) == bits(v)
    same_breakdown(lplan.predict(lib_params(params) if params else None),
                   GT.predict_plan(t, oplan, ES[dtype], params))
    return lplan, oplan


def test_c1():
    doc = T.two_level_doc([2, 2], T.TABLE5["root_sw"], T.TABLE5["middle_sw"], T.TABLE5["server"])
    lp, _ = check_topology(doc, 262144)
    assert lp.predict()["total"] == pytest.approx(0.029064844, rel=1e-8)


@pytest.mark.parametrize("S", [10 ** 7, 32 * 10 ** 6, 10 ** 8, 32 * 10 ** 7])
def test_c5_64_ranks(S):
    nic = {"alpha": 6.58e-3, "beta": 4e-11, "epsilon": 6e-12, "w_t": 9}
    nvl = {"alpha": 1e-5, "beta": 4.0 / 900e9, "epsilon": 1e-13, "w_t": 9}
    check_topology(T.two_level_doc([8] * 8, nic, nvl, T.TABLE5["server"]), S)


@pytest.mark.parametrize("n", [2, 3, 4, 5, 6, 7, 8, 12, 16])
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_single_switch_gentree(n, dtype):
    doc = T.single_switch_doc(n, row("middle_sw"), T.TABLE5["server"])
    for count in (1, n - 1, 1000 * n + 3, 10 ** 7):
        if count >= 1:
            check_topology(doc, count, dtype)


@pytest.mark.parametrize("force", ["cps", "ring", "rhd", "hcps:4,2", "hcps:2,4", "hcps:2,2,2", "rb"])
def test_forced_kinds_8(force):
    doc = T.single_switch_doc(8, row("middle_sw"), T.TABLE5["server"])
    p = OG.Params(2e-6, 1.0 / 770e9, 1e-14, 1.0 / 6.5e12, 1e-14, 6)
    for count in (8, 1001, 1 << 20):
        check_topology(doc, count, "bf16", params=p, force=force)


def test_explicit_and_combined_params():
    doc = T.single_switch_doc(12, row("middle_sw"), T.TABLE5["server"])
    Sb = 4 * 10 ** 8
    p = OG.Params(4.0e-3, 0.0, 0.0, 0.0391 / Sb, 0.01066 / Sb, 9, combined=0.6638 / Sb)
    lp, _ = check_topology(doc, 10 ** 8, params=p)
    assert lp.report()[-1]["chosen"] == "hcps[6,2]"


@pytest.mark.slow
def test_gtplan_topologies():
    for name, doc in _gtplan_topos().items():
        for S in (10 ** 7, 10 ** 8):
            check_topology(doc, S)


def test_random_trees():
    rnd = random.Random(4202)
    done = 0
    while done < 80:
        doc = _random_tree(rnd, max_servers=40)
        try:
            t = T.parse_topology(doc)
        except T.TopologyError:
            continue
        N = len(t.servers)
        check_topology(doc, rnd.randint(1, 40 * N), rnd.choice(["f32", "bf16"]))
        done += 1


@pytest.mark.parametrize("kind", ["cps", "ring", "rhd", "rb", "hcps:4,2", "hcps:2,3,4", "hcps:8,3"])
def test_closed_form_bits(kind):
    name, f = OP.parse_kind(kind)
    n = 8 if name != "hcps" else 1
    for x in f:
        n *= x
    p = OG.Params(6.58e-3, 6.4e-9 / 4, 6e-10 / 4, 1.87e-10 / 4, 1.22e-10 / 4, 9)
    for S in (4, 4 * 10 ** 7 + 12, 123456789):
        same_breakdown(G.genmodel_closed_form(kind, n, S, lib_params(p)),
                       OG.closed_form_f64(name, n, S, p, f))


def test_invalid_inputs_rejected():
    bad = [T.single_switch_doc(1, row("middle_sw"), T.TABLE5["server"]), "{nope", '{"nodes": []}']
    for doc in bad:
        with pytest.raises(G.ArInvalid):
            G.Plan.from_topology(doc, 10)
        with pytest.raises(T.TopologyError):
            T.parse_topology(doc)
    doc = T.single_switch_doc(8, row("middle_sw"), T.TABLE5["server"])
    for force in ("hcps:3,3", "bogus", "hcps:x"):
        with pytest.raises(G.ArInvalid):
            G.Plan.from_topology(doc, 100, force=force)
    with pytest.raises(G.ArInvalid):
        G.Plan.from_topology(doc, 0)


def test_fit_parity_noiseless():
    truth = (6.58e-3, 1.34e-9 / 4, 1.87e-10 / 4, 1.22e-10 / 4, 6)
    rows = []
    for n in range(2, 9):
        for s in (1 << 20, 1 << 24, 1 << 28):
            rows.append((n, s, OF.cps_forward(n, s, *truth)))
    o = OF.fit_params(rows, 2, 8)
    lp, sse = G.genmodel_fit(rows, 2, 8)
    assert lp.w_t == o["w_t"] == 6 and lp.has_combined == 1
    for a, b in ((lp.alpha, o["alpha"]), (lp.combined, o["combined"]), (lp.delta, o["delta"]),
                 (lp.epsilon, o["epsilon"])):
        assert a == pytest.approx(b, rel=1e-9)
    lp2, _ = G.genmodel_fit(rows, 2, 8, link_bytes_per_s=900e9)
    assert lp2.beta == 1.0 / 900e9 and lp2.gamma == pytest.approx(truth[1] - 2 / 900e9, rel=1e-9)


@pytest.mark.parametrize("shape", [(2, 2, 2, 2), (2, 3, 2, 3), (2, 4, 2, 2)])
def test_rearrangement_topologies(shape):
    """Data rearrangement adopted + ACPS: library and oracle agree bit for bit."""
    from tests.topologies import cross_dc
    doc = cross_dc(*shape)
    lp, op = check_topology(doc, 10 ** 6)
    assert any(r["rearranged_children"] for r in lp.report())
    assert any(len(r.inputs) == 1 for st in op.steps for r in st.reduces)   # moves present


def test_nvls_row_and_fit_parity():
    """NEXT #1: the NVLS closed-form row and its (α, β) fit, library vs oracle."""
    p = OG.Params(9.4e-6, 1.7e-12, 0, 0, 0, 1)
    for n in (2, 4, 8):
        for S in (4, 1 << 20, 123456789):
            same_breakdown(G.genmodel_closed_form("nvls", n, S, lib_params(p)),
                           OG.closed_form_f64("nvls", n, S, p))
    rows = [(n, s, 2 * 9e-6 + (n + 1) * s / n * 1.8e-12 * (1 + 0.01 * ((n * s) % 7)))
            for n in (2, 4) for s in (1 << 20, 1 << 24, 1 << 28)]
    lp, sse = G.genmodel_fit_nvls(rows)
    o = OF.fit_nvls(rows)
    assert lp.alpha == pytest.approx(o["alpha"], rel=1e-9)
    assert lp.beta == pytest.approx(o["beta"], rel=1e-9)
    assert sse == pytest.approx(o["sse"], rel=1e-6)


def test_ll128_row_parity():
    """The LL128 row: library closed form and fit ≡ oracle."""
    p = OG.Params(3e-6, 1.5e-12, 0.0, 0.0, 0.0, 1)
    for n in (2, 3, 4, 8):
        for S in (4096, 1 << 20, 12345678):
            same_breakdown(G.genmodel_closed_form("ll128", n, S, lib_params(p)), OG.closed_form_f64("ll128", n, S, p))
    rows = [(n, s, OG.closed_form_f64("ll128", n, s, p)["total"]) for n in (2, 4) for s in (1 << 20, 1 << 22, 1 << 24)]
    lp, _ = G.genmodel_fit_row("ll128", rows)
    o = OF.fit_row("ll128", rows)
    assert lp.alpha == pytest.approx(o["alpha"], rel=1e-9) and lp.beta == pytest.approx(o["beta"], rel=1e-9)
    assert lp.alpha == pytest.approx(3e-6, rel=1e-9) and lp.beta == pytest.approx(1.5e-12, rel=1e-9)


def test_oneshot_row_and_fit_parity():
    p = OG.Params(4e-6, 1.0e-12, 2e-13, 3e-13, 1e-14, 3)
    for n in (2, 4, 8):
        for S in (16, 1 << 16, 1234567):
            same_breakdown(G.genmodel_closed_form("oneshot", n, S, lib_params(p)),
                           OG.closed_form_f64("oneshot", n, S, p))
    rows = [(n, s, 4e-6 + 2 * (n - 1) * s * 3e-12 * (1 + 0.02 * ((n + s) % 5))) for n in (2, 4)
            for s in (1 << 12, 1 << 16, 1 << 19)]
    lp, sse = G.genmodel_fit_row("oneshot", rows)
    o = OF.fit_row("oneshot", rows)
    assert lp.alpha == pytest.approx(o["alpha"], rel=1e-9) and lp.beta == pytest.approx(o["beta"], rel=1e-9)
    ln, _ = G.genmodel_fit_row("nvls", [(4, 1 << 20, 2e-5), (4, 1 << 24, 5e-5), (2, 1 << 22, 3e-5)])
    on = OF.fit_nvls([(4, 1 << 20, 2e-5), (4, 1 << 24, 5e-5), (2, 1 << 22, 3e-5)])
    assert ln.alpha == pytest.approx(on["alpha"], rel=1e-9) and ln.beta == pytest.approx(on["beta"], rel=1e-9)
    with pytest.raises(G.ArInvalid):
        G.genmodel_fit_row("cps", rows)


def test_choose_nvls():
    """genmodel_choose_nvls = (executed-plan prediction) vs (NVLS closed form)."""
    pp = G.params(alpha=9.4e-6, combined=2.93e-12, w_t=4)
    nv = G.params(alpha=8e-6, beta=1.75e-12)
    for n, count in ((2, 1 << 26), (4, 1 << 26), (2, 1 << 12), (4, 1 << 12)):
        plan = G.Plan.single_switch(n, count, "bf16", pp)
        c = plan.choose_nvls(pp, nv)
        assert c["t_plan"] == plan.predict_executed(pp)["total"]
        assert c["t_nvls"] == G.genmodel_closed_form("nvls", n, 2 * count, nv)["total"]
        assert c["use_nvls"] == (c["t_nvls"] < c["t_plan"])
    # the wire model: NVLS loses at N = 2 and wins at N = 4 for large messages with equal β
    eq = G.params(alpha=9.4e-6, beta=1.465e-12)
    assert not G.Plan.single_switch(2, 1 << 27, "bf16", pp).choose_nvls(pp, eq)["use_nvls"]
    assert G.Plan.single_switch(4, 1 << 27, "bf16", pp).choose_nvls(pp, eq)["use_nvls"]


def _sim_close(a: dict, b: dict):
    for k in ("latency", "bandwidth", "compute", "memory", "incast", "total"):
        assert a[k] == pytest.approx(float(b[k]), rel=1e-9, abs=1e-15), k


@pytest.mark.parametrize("which", ["SS24", "two_level", "asym", "cdc_small"])
def test_flow_simulator_parity(which):
    """NEXT #2: gt_plan_simulate vs oracle.flowsim (exact rationals), 1e-9 relative."""
    from oracle import flowsim as FS
    from tests.topologies import cross_dc
    docs = {"SS24": _gtplan_topos()["SS24"],
            "two_level": T.two_level_doc([4, 4, 4], row("root_sw"), row("middle_sw"), T.TABLE5["server"]),
            "asym": T.two_level_doc([6, 2, 3], row("root_sw"), row("middle_sw"), T.TABLE5["server"]),
            "cdc_small": cross_dc(2, 4, 2, 2)}
    doc = docs[which]
    t = T.parse_topology(doc)
    for S in (10 ** 6, 32 * 10 ** 6):
        for force in (None, "cps", "ring"):
            lib = G.Plan.from_topology(doc, S, "f32", None, force)
            oplan, _ = GT.gentree(t, S, 4, force=force)
            _sim_close(lib.simulate(), FS.simulate_flows(t, oplan, 4))
    # a flat plan routed over the tree (topology_json)
    n = len(t.servers)
    flat = G.Plan.single_switch(n, 12345, "f32", G.params(alpha=1e-3, beta=1e-9), "cps")
    oflat = OP.build_plan("cps", n, 12345)
    _sim_close(flat.simulate(topology_json=doc), FS.simulate_flows(t, oflat, 4))
    # uniform params
    p = OG.Params(1e-4, 2e-12, 1e-13, 3e-13, 5e-14, 3)
    lib = G.Plan.from_topology(doc, 99999, "bf16")
    oplan, _ = GT.gentree(t, 99999, 2)
    _sim_close(lib.simulate(lib_params(p)), FS.simulate_flows(t, oplan, 2, p))


@pytest.mark.parametrize("shared", [False, True])
def test_predict_executed_parity(shared):
    """genmodel_predict_executed[_shared] (the library derives the executed steps from its
    lowered device tables) vs oracle.genmodel.predict_executed (executed steps derived from
    the plan and the stated fusion rule, reading A6x / A6e): bit-identical doubles over every
    plan kind, single-switch N = 2..16, the C1/C5/asymmetric trees and rearrangement trees,
    degenerate (count < N), ragged and divisible counts, f32 and bf16."""
    from tests.topologies import cross_dc
    p = OG.Params(3e-6, 1 / 900e9, 1e-13, 1 / 6.54e12, 2e-13, 3)
    lp = lib_params(p)

    def ss(n):
        return T.single_switch_doc(n, {"alpha": 3e-6, "beta": 4 / 900e9, "epsilon": 0.0, "w_t": 9},
                                   {"gamma": 0.0, "delta": 4 / 6.54e12})
    docs = [(n, ss(n)) for n in (2, 3, 4, 5, 6, 8, 12, 16)]
    docs += [(4, T.two_level_doc([2, 2], T.TABLE5["root_sw"], T.TABLE5["middle_sw"], T.TABLE5["server"])),
             (7, T.two_level_doc([3, 4], T.TABLE5["root_sw"], T.TABLE5["middle_sw"], T.TABLE5["server"])),
             (64, T.two_level_doc([8] * 8, T.TABLE5["root_sw"], T.TABLE5["middle_sw"], T.TABLE5["server"]))]
    docs += [(sh[0] * sh[1] + sh[2] * sh[3], cross_dc(*sh)) for sh in [(2, 2, 2, 2), (2, 4, 2, 2)]]
    checked = 0
    for n, doc in docs:
        t = T.parse_topology(doc)
        for kind in (None, "cps", "ring", "rb", "rhd", "hcps:2,2", "hcps:4,2", "hcps:2,2,2", "hcps:2,4", "hcps:3,2"):
            for count in (1, n - 1, 1000003, 1000000, 7777):
                for dtype in ("f32", "bf16"):
                    try:
                        gplan = G.Plan.from_topology(doc, count, dtype, None, kind)
                    except G.ArInvalid:
                        continue
                    oplan, _ = GT.gentree(t, count, ES[dtype], force=kind)
                    want = OG.predict_executed(oplan, ES[dtype], p, shared)
                    got = (gplan.predict_executed_shared if shared else gplan.predict_executed)(lp)
                    same_breakdown(got, want)
                    checked += 1
    assert checked > 500


def test_default_paths():
    """The executor's default path cut-offs (ar_default_paths; measured): one-shot
    to 1.5 MiB/(N-1) (at most 1.5 MiB), LL128 from 768 KiB/(N-1) (at most 384 KiB, never above
    the one-shot cut-off) to 64 MiB/N, 256-byte / 1 MiB granularity."""
    want = {2: (1536 << 10, 384 << 10, 32 << 20), 3: (768 << 10, 384 << 10, 21 << 20),
            4: (512 << 10, 256 << 10, 16 << 20), 8: (224512, 112128, 8 << 20)}
    for n, (om, lmin, lmax) in want.items():
        assert G.default_paths(n) == {"oneshot_max": om, "ll128_min": lmin, "ll128_max": lmax}
    with pytest.raises(G.ArInvalid):
        G.default_paths(1)


def test_nvls_plan_kind_parity():
    """NVLS as a GenTree plan kind (NEXT #1, readings NV1/NV2): force "nvls" and the
    min-GenModel choice gentree_plan_nvls give byte-identical plan JSON (CPS movement +
    "switch_reduce") and bit-identical predictions in library and oracle; bf16 and multi-level
    topologies are refused; the JSON round-trips and a non-CPS switch_reduce plan is refused."""
    pp = OG.Params(9.4e-6, 1.465e-12, 0.0, 0.0, 0.0, 4)
    nv_cheap = OG.Params(5.7e-6, 0.9e-12, 0.0, 0.0, 0.0, 1)
    nv_dear = OG.Params(50e-6, 3e-12, 0.0, 0.0, 0.0, 1)
    for n in (2, 3, 4, 8):
        doc = T.single_switch_doc(n, {"alpha": 3e-6, "beta": 4 / 900e9, "epsilon": 0.0, "w_t": 9},
                                  {"gamma": 0.0, "delta": 4 / 6.54e12})
        t = T.parse_topology(doc)
        for count in (1, n - 1, 1000003, 1 << 20):
            lp = G.Plan.from_topology(doc, count, "f32", lib_params(pp), "nvls")
            op, orep = GT.gentree(t, count, 4, params=pp, force="nvls")
            assert lp.to_json() == OP.plan_to_json(op, "f32")
            assert lp.switch_reduce and '"switch_reduce":true' in lp.to_json()
            assert lp.report()[-1]["chosen"] == "nvls" == orep[-1].chosen
            same_breakdown(lp.predict_executed(lib_params(nv_cheap)), OG.predict_executed(op, 4, nv_cheap))
            back = G.Plan.from_json(lp.to_json())
            assert back.to_json() == lp.to_json() and back.is_allreduce
            osp = OG.Params(4.61e-6, 2.963e-12, 0.0, 0.0, 0.0, 1)     # one-shot row (reading OS1)
            paths = G.default_paths(n)
            cut = paths["oneshot_max"]
            for nvp in (nv_cheap, nv_dear):
                lg = G.Plan.from_topology_nvls(doc, count, "f32", lib_params(pp), lib_params(nvp))
                og, _ = GT.gentree_nvls(t, count, 4, pp, nvp)
                assert lg.to_json() == OP.plan_to_json(og, "f32")
                lo = G.Plan.from_topology_nvls(doc, count, "f32", lib_params(pp), lib_params(nvp), lib_params(osp), cut)
                oo, _ = GT.gentree_nvls(t, count, 4, pp, nvp, osp, cut)
                assert lo.to_json() == OP.plan_to_json(oo, "f32")
                llp = OG.Params(5.1e-6, 1.74e-12, 0.0, 0.0, 0.0, 1)   # LL128 row
                # ragged / aligned blocks; below, between and above the LL128 floor and ceiling
                for c2 in (count, n * 4 * 4096, n * 4 * 256, n * 4 * 16384, n * 4 * (1 << 20)):
                    for lmin, lmax in ((0, 16 << 20), (paths["ll128_min"], paths["ll128_max"])):
                        l2 = G.Plan.from_topology_nvls(doc, c2, "f32", lib_params(pp), lib_params(nvp),
                                                       lib_params(osp), cut, lib_params(llp), lmax, lmin)
                        o2, _ = GT.gentree_nvls(t, c2, 4, pp, nvp, osp, cut, llp, lmax, lmin)
                        assert l2.to_json() == OP.plan_to_json(o2, "f32")
                lb = G.Plan.from_topology_nvls(doc, count, "bf16", lib_params(pp), lib_params(nvp))
                assert not lb.switch_reduce        # bf16 never takes NVLS
        # large messages: the cheap NVLS row ((N+1)/N·0.9 < 2(N-1)/N·1.465 per byte) wins at
        # every N, the dear one never
        big = 1 << 26
        assert G.Plan.from_topology_nvls(doc, big, "f32", lib_params(pp), lib_params(nv_cheap)).switch_reduce
        assert not G.Plan.from_topology_nvls(doc, big, "f32", lib_params(pp), lib_params(nv_dear)).switch_reduce
        # small messages: the one-shot row (4.6 µs) beats the NVLS row's 2α = 11.4 µs, so the
        # plan stays although NVLS beats the flag-protocol prediction (2 × 9.4 µs)
        small = 4096
        assert G.Plan.from_topology_nvls(doc, small, "f32", lib_params(pp), lib_params(nv_cheap)).switch_reduce
        assert not G.Plan.from_topology_nvls(doc, small, "f32", lib_params(pp), lib_params(nv_cheap),
                                             lib_params(OG.Params(4.61e-6, 2.963e-12, 0, 0, 0, 1)), 1 << 20).switch_reduce
        with pytest.raises(G.ArInvalid):
            G.Plan.from_topology(doc, 1024, "bf16", lib_params(pp), "nvls")
        with pytest.raises(G.ArInvalid):
            G.Plan.from_topology(doc, 1024, "f32", lib_params(pp), "nvls").lowering()
    two = T.two_level_doc([2, 2], T.TABLE5["root_sw"], T.TABLE5["middle_sw"], T.TABLE5["server"])
    with pytest.raises(G.ArInvalid):
        G.Plan.from_topology(two, 1024, "f32", None, "nvls")
    ring = json.loads(G.Plan.single_switch(4, 1000, "f32", lib_params(pp), "ring").to_json())
    ring["switch_reduce"] = True
    with pytest.raises(G.ArInvalid):
        G.Plan.from_json(json.dumps(ring))


@pytest.mark.parametrize("shape", [(2, 2, 2, 2), (2, 3, 2, 3), (2, 4, 2, 2)])
def test_gentree_star_without_rearrangement(shape):
    """tab:gentreesimu's GenTree* ("the special plan without data rearrangement"):
    force "norearrange" — library and oracle agree bit for bit, no child is rearranged, no
    rearrangement moves (single-input reduces) appear, while GenTree does rearrange here.
    (The rearrangement decision is local — transfer-out time of one child with vs without it,
    P:705-715 — so the whole-plan GenModel can still price GenTree* lower; it does on these
    small topologies, in both implementations alike.)"""
    from tests.topologies import cross_dc
    doc = cross_dc(*shape)
    star, ostar = check_topology(doc, 10 ** 6, force="norearrange")
    assert not any(r["rearranged_children"] for r in star.report())
    assert not any(len(r.inputs) == 1 for st in ostar.steps for r in st.reduces)
    full, _ = check_topology(doc, 10 ** 6)
    assert any(r["rearranged_children"] for r in full.report())


def test_gentree_star_equals_gentree_without_rearrangement():
    """Where GenTree rearranges nothing, GenTree* is the same plan (byte-identical JSON)."""
    for name, doc in _gtplan_topos().items():
        for S in (10 ** 7, 10 ** 8):
            a, _ = check_topology(doc, S)
            if not any(r["rearranged_children"] for r in a.report()):
                b, _ = check_topology(doc, S, force="norearrange")
                assert a.to_json() == b.to_json()
