"""GPU parity: the CUDA path (through the C-ABI) vs the CPU oracle, element by element.

Single GPU: the emulated communicator runs all ranks of a plan in one cooperative launch on
one B200 (same step tables, same flag protocol as the multi-process path), so every plan kind
is exercised at 2..64 ranks.  Inputs come from the device generator (ar_fill_synthetic),
which is itself checked bit-for-bit against synth/generator.py first.  Bar: bit-exact
(BASELINE.json north star), NaNs by isnan.
"""
import numpy as np
import pytest

from tests.gpu_util import assert_bits_equal, cuda_ok, emulated_buffer, rank_views

pytestmark = pytest.mark.gpu

if cuda_ok():
    import torch

    import paper_2409_04202_b200 as G
    from oracle import gentree as GT
    from oracle import plans as OP
    from oracle import simulate as SM
    from oracle import topology as T
    from synth import generator as GEN
else:  # collected but skipped on CPU-only hosts
    pytest.skip("needs a CUDA GPU", allow_module_level=True)

MODES = {"gradient": 0, "integer": 1, "specials": 2}
SEED = GEN.config_seed(1)


def nominal():
    """Nominal B200 GenModel parameters per byte: α = 3 µs, β = 1/900 GB/s,
    δ = 1/6.54 TB/s, no incast below 9."""
    return G.params(3e-6, 1 / 900e9, 0.0, 1 / 6.54e12, 0.0, 9)


def oracle_params():
    from oracle import genmodel as OG
    return OG.Params(3e-6, 1 / 900e9, 0.0, 1 / 6.54e12, 0.0, 9)


def single_switch(world):
    return T.single_switch_doc(world, {"alpha": 3e-6, "beta": 4 / 900e9, "epsilon": 0.0, "w_t": 9},
                               {"gamma": 0.0, "delta": 4 / 6.54e12})


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("mode", ["gradient", "integer", "specials"])
def test_device_generator_matches_numpy(dtype, mode):
    count, start = 70001, 123457
    buf = torch.zeros(count * 4, dtype=torch.uint8, device="cuda")
    for rank in (0, 5):
        G.fill_synthetic(buf.data_ptr(), count, dtype, SEED, rank, MODES[mode], start)
        torch.cuda.synchronize()
        raw = buf.cpu().numpy()[: count * (4 if dtype == "f32" else 2)]
        got = raw.view(np.uint32 if dtype == "f32" else np.uint16)
        want = GEN.generate(SEED, rank, count, dtype, mode, start=start)
        want = want.view(np.uint32) if dtype == "f32" else want
        assert np.array_equal(got, want)


def run_emulated(doc, world, count, dtype, force=None, mode="gradient", params=None, ctas=0, calls=1, red="sum",
                 expect_kernel=None):
    plan = G.Plan.from_topology(doc, count, dtype, params, force)
    comm = G.Comm.local(world, 0)
    if ctas:
        comm.set_ctas(ctas)
    buf, stride = emulated_buffer(world, count, dtype, SEED, MODES[mode])
    inputs = rank_views(buf, world, count, dtype, stride)
    t = T.parse_topology(doc)
    from oracle import genmodel as OG
    op = None
    if params is not None:
        op = OG.Params(params.alpha, params.beta, params.gamma, params.delta, params.epsilon, params.w_t,
                       params.combined if params.has_combined else None)
    oplan, _ = GT.gentree(t, count, 4 if dtype == "f32" else 2, params=op, force=force)
    assert plan.to_json() == OP.plan_to_json(oplan, dtype)
    want = inputs
    for _ in range(calls):
        G.allreduce_exec(plan, comm, buf, op=red)
        want = SM.simulate(oplan, want, dtype, op=red)
    torch.cuda.synchronize()
    comm.async_error()
    got = rank_views(buf, world, count, dtype, stride)
    for r in range(world):
        assert_bits_equal(got[r], want[r], dtype, f"rank {r}")
    assert comm.last_launch_count() == 1
    if expect_kernel:
        assert comm.last_kernel() == expect_kernel, comm.last_kernel()
    return got


@pytest.mark.parametrize("world", [2, 3, 4, 5, 8])
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_gentree_single_switch(world, dtype):
    for count in (1, world - 1, 4096 * world + 3, 100003):
        run_emulated(single_switch(world), world, count, dtype)


@pytest.mark.parametrize("force", ["cps", "ring", "rhd", "rb", "hcps:4,2", "hcps:2,4", "hcps:2,2,2"])
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_forced_kinds_8_ranks(force, dtype):
    for count in (8 * 1024, 262147):
        run_emulated(single_switch(8), 8, count, dtype, force=force)


@pytest.mark.parametrize("force", ["cps", "ring", "hcps:3,2", "hcps:2,3"])
def test_forced_kinds_6_ranks(force):
    run_emulated(single_switch(6), 6, 60001, "f32", force=force)


@pytest.mark.parametrize("mode", ["integer", "specials"])
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_modes(mode, dtype):
    got = run_emulated(single_switch(8), 8, 40000, dtype, force="ring", mode=mode)
    if mode == "integer":
        xs = GEN.generate_all(SEED, 8, 40000, dtype, "integer")
        ref = sum(GEN.as_f64(x, dtype).astype(np.int64) for x in xs)
        assert np.array_equal(GEN.as_f64(got[3], dtype).astype(np.int64), ref)


def test_c1_two_level_tree():
    doc = T.two_level_doc([2, 2], T.TABLE5["root_sw"], T.TABLE5["middle_sw"], T.TABLE5["server"])
    run_emulated(doc, 4, 262144, "f32")


def test_c5_64_ranks_8_per_gpu():
    """C5: the 64-rank two-level tree (8 nodes x 8 GPUs), all 64 ranks on one GPU."""
    nic = {"alpha": 6.58e-3, "beta": 4e-11, "epsilon": 6e-12, "w_t": 9}
    nvl = {"alpha": 1e-5, "beta": 4.0 / 900e9, "epsilon": 1e-13, "w_t": 9}
    doc = T.two_level_doc([8] * 8, nic, nvl, T.TABLE5["server"])
    run_emulated(doc, 64, 64 * 1000 + 17, "f32")


def test_asymmetric_tree_acps():
    doc = T.two_level_doc([3, 4], T.TABLE5["root_sw"], T.TABLE5["middle_sw"], T.TABLE5["server"])
    run_emulated(doc, 7, 70001, "bf16")


def test_repeated_calls_and_plan_interleave():
    """Epoch progression: 3 back-to-back calls, then a different plan on the same comm."""
    run_emulated(single_switch(4), 4, 50000, "f32", force="ring", calls=3)
    doc = single_switch(4)
    comm = G.Comm.local(4, 0)
    count = 30000
    p1 = G.Plan.from_topology(doc, count, "f32", None, "cps")
    p2 = G.Plan.from_topology(doc, count, "f32", None, "hcps:2,2")
    buf, stride = emulated_buffer(4, count, "f32", SEED)
    x = rank_views(buf, 4, count, "f32", stride)
    t = T.parse_topology(doc)
    o1, _ = GT.gentree(t, count, 4, force="cps")
    o2, _ = GT.gentree(t, count, 4, force="hcps:2,2")
    for plan, oplan in ((p1, o1), (p2, o2), (p1, o1), (p2, o2)):
        G.allreduce_exec(plan, comm, buf)
        x = SM.simulate(oplan, x, "f32")
    torch.cuda.synchronize()
    got = rank_views(buf, 4, count, "f32", stride)
    for r in range(4):
        assert_bits_equal(got[r], x[r], "f32", f"rank {r}")


@pytest.mark.parametrize("force", ["ring", "rhd", "hcps:4,2", "rb", "cps"])
def test_stress_back_to_back(force, monkeypatch):
    """300 back-to-back calls (epoch progression, bulk-copy pipeline phases across ops and
    calls) with a 2 s device wait bound: no wait may time out; then one more call checked
    bit-exact.  Caught the copy-tile parity hang (SURVEY §4 "stress: back-to-back launches")."""
    monkeypatch.setenv("AR_FLAG_TIMEOUT_MS", "2000")
    world, count, dtype = 8, (1 << 22) + 5, "f32"
    doc = single_switch(world)
    plan = G.Plan.from_topology(doc, count, dtype, None, force)
    comm = G.Comm.local(world, 0)
    buf, stride = emulated_buffer(world, count, dtype, SEED, MODES["integer"])
    ex = G.Executor(plan, comm, buf)
    for _ in range(300):
        ex()
    torch.cuda.synchronize()
    comm.async_error()
    for r in range(world):
        G.fill_synthetic(buf.data_ptr() + r * stride, count, dtype, SEED, r, 0)
    ex()
    torch.cuda.synchronize()
    comm.async_error()
    oplan, _ = GT.gentree(T.parse_topology(doc), count, 4, force=force)
    want = SM.simulate(oplan, GEN.generate_all(SEED, world, count, dtype), dtype)
    got = rank_views(buf, world, count, dtype, stride)
    for r in (0, world - 1):
        assert_bits_equal(got[r], want[r], dtype, f"rank {r}")


@pytest.mark.parametrize("force", ["ring", "hcps:2,4", "rhd", None])
def test_jitter_injection(force, monkeypatch):
    """random delays (up to 20 us) before every flag post; any missing dependency
    or ordering bug then shows up as a non-bit-exact result."""
    monkeypatch.setenv("AR_JITTER_NS", "20000")
    run_emulated(single_switch(8), 8, 300007, "bf16", force=force, calls=3)


@pytest.mark.parametrize("force", ["cps", "ring", "rhd", "rb", "hcps:3,2", "hcps:2,3", None])
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_avg_op(force, dtype):
    """AR_OP_AVG (NEXT #4, reading AV1): fused division in the final reduce, bit-exact vs the
    oracle, ragged sizes, alternating with SUM on the same plan (cached launch arguments)."""
    world = 6 if force != "rhd" else 8
    for count in (world - 1, 4096 * world + 5, 200003):
        run_emulated(single_switch(world), world, count, dtype, force=force, red="avg", calls=2)
        run_emulated(single_switch(world), world, count, dtype, force=force, red="sum")


def test_avg_rearrangement_and_c5():
    from tests.topologies import cross_dc
    run_emulated(cross_dc(2, 4, 2, 2), 12, 77777, "bf16", red="avg")
    doc = T.two_level_doc([8] * 8, T.TABLE5["root_sw"], T.TABLE5["middle_sw"], T.TABLE5["server"])
    run_emulated(doc, 64, 64 * 1000 + 17, "bf16", red="avg")


@pytest.mark.parametrize("ctas", [1, 3, 17])
def test_cta_counts(ctas):
    run_emulated(single_switch(8), 8, 123457, "bf16", force="hcps:4,2", ctas=ctas)


@pytest.mark.parametrize("mode,dtype", [("gradient", "bf16"), ("specials", "bf16"), ("gradient", "f32")])
def test_full_size_bench_config_full_buffer(mode, dtype):
    """bench.py's N=1 workload in the launch configuration bench.py times: 8 emulated ranks,
    256 MiB per rank (bf16, and the `--dtype f32` line), GenTree plan (CPS) on ar_flat_kernel
    with dynamic tiles, bench's seed — EVERY element of EVERY rank compared with the oracle's
    step-by-step simulation (a single wrong tile anywhere fails), for gradient-shaped and
    special-value inputs."""
    es = 2 if dtype == "bf16" else 4
    world, count = 8, (256 << 20) // es
    seed = 0x240904202 ^ 4
    doc = single_switch(world)
    plan = G.Plan.from_topology(doc, count, dtype)
    comm = G.Comm.local(world, 0)
    stride = G.rank_stride_bytes(count, dtype)
    buf = torch.empty(world * stride, dtype=torch.uint8, device="cuda")
    for r in range(world):
        G.fill_synthetic(buf.data_ptr() + r * stride, count, dtype, seed, r, MODES[mode])
    G.allreduce_exec(plan, comm, buf)
    torch.cuda.synchronize()
    comm.async_error()
    assert comm.last_kernel() == "ar_flat_kernel"
    oplan, _ = GT.gentree(T.parse_topology(doc), count, es)
    assert OP.plan_to_json(oplan, dtype) == plan.to_json()
    want = SM.simulate(oplan, GEN.generate_all(seed, world, count, dtype, mode), dtype)
    host = buf.cpu().numpy()
    for r in range(world):
        got = host[r * stride: r * stride + es * count].view(np.uint16 if dtype == "bf16" else np.float32)
        assert_bits_equal(got, want[r], dtype, f"rank {r}")
    del host, want


@pytest.mark.parametrize("force", [None, "ring", "rhd", "rb", "hcps:4,2", "hcps:2,2,2"])
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_large_all_kinds_full_buffer(force, dtype):
    """Every plan kind at 32 MiB per rank (8 emulated ranks, thousands of tiles per op,
    ragged count), every element of every rank vs the oracle."""
    world = 8
    count = (32 << 20) // (4 if dtype == "f32" else 2) + 13
    run_emulated(single_switch(world), world, count, dtype, force=force)


@pytest.mark.parametrize("mode", ["integer", "specials"])
@pytest.mark.parametrize("force", [None, "ring", "rhd", "rb", "hcps:4,2", "hcps:2,4", "hcps:2,2,2"])
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_modes_every_kind(mode, force, dtype):
    """±0, subnormals, ±max-finite (overflow -> inf), ±inf, NaN, and integer-valued inputs
    through every plan kind — CPS on the flat kernel (dynamic tiles) and on the step-table
    kernel's flag protocol, Ring, RHD, RB, HCPS — SUM and AVG (reading AV1).  Integer inputs
    must give the exact int64 sum (every partial exact)."""
    world, count = 8, 300007
    got = run_emulated(single_switch(world), world, count, dtype, force=force, mode=mode)
    if mode == "integer":
        xs = GEN.generate_all(SEED, world, count, dtype, "integer")
        ref = sum(GEN.as_f64(x, dtype).astype(np.int64) for x in xs)
        for r in (0, world - 1):
            assert np.array_equal(GEN.as_f64(got[r], dtype).astype(np.int64), ref)
    run_emulated(single_switch(world), world, count, dtype, force=force, mode=mode, red="avg")


@pytest.mark.parametrize("mode", ["integer", "specials"])
def test_modes_cps_flag_protocol(mode, monkeypatch):
    """The same edge-case inputs through CPS on the step-table kernel (AR_FLAT=0)."""
    monkeypatch.setenv("AR_FLAT", "0")
    for dtype in ("f32", "bf16"):
        run_emulated(single_switch(8), 8, 300007, dtype, force="cps", mode=mode)
        run_emulated(single_switch(8), 8, 300007, dtype, force="cps", mode=mode, red="avg")


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("k", [1, 2, 3, 8, 13])
def test_local_reduce(dtype, k):
    count = 1 << 16
    es = 4 if dtype == "f32" else 2
    ins = []
    for i in range(k):
        b = torch.empty(count * es, dtype=torch.uint8, device="cuda")
        G.fill_synthetic(b, count, dtype, SEED, i, 0)
        ins.append(b)
    out = torch.empty(count * es, dtype=torch.uint8, device="cuda")
    G.local_reduce(ins, out, count, dtype)
    torch.cuda.synchronize()
    xs = [GEN.generate(SEED, i, count, dtype) for i in range(k)]
    plan = OP.Plan(1, count, [])
    if dtype == "f32":
        acc = xs[0].copy()
        for x in xs[1:]:
            acc = acc + x
        want = acc
    else:
        acc = SM.bf16_bits_to_f32(xs[0]).copy()
        for x in xs[1:]:
            acc = acc + SM.bf16_bits_to_f32(x)
        want = SM.f32_to_bf16_rne(acc) if k > 1 else xs[0]
    got = out.cpu().numpy().view(np.float32 if dtype == "f32" else np.uint16)
    assert_bits_equal(got, want, dtype)
    del plan


def test_errors_are_loud():
    comm = G.Comm.local(4, 0)
    plan = G.Plan.from_topology(single_switch(8), 1000, "f32")
    buf = torch.zeros(1 << 20, dtype=torch.uint8, device="cuda")
    with pytest.raises(G.ArInvalid):
        G.allreduce_exec(plan, comm, buf)          # world mismatch
    plan4 = G.Plan.from_topology(single_switch(4), 1000, "f32")
    with pytest.raises(G.ArInvalid):
        G.allreduce_exec(plan4, comm, buf, count=999)
    with pytest.raises(G.ArInvalid):
        G.allreduce_exec(plan4, comm, buf.data_ptr() + 4)   # misaligned
    mc = G.Comm.create(0, 2, 0)
    with pytest.raises(G.ArInvalid):
        G.allreduce_exec(G.Plan.from_topology(single_switch(2), 1000, "f32"), mc, buf)  # unregistered


@pytest.mark.parametrize("shape", [(2, 2, 2, 2), (2, 4, 2, 2)])
def test_rearrangement_and_acps(shape):
    """NEXT #3 rows on one GPU: a GenTree plan with data rearrangement (moves) and an
    asymmetric CPS root, emulated ranks, bit-exact."""
    from tests.topologies import cross_dc
    world = shape[0] * shape[1] + shape[2] * shape[3]
    run_emulated(cross_dc(*shape), world, 123457, "bf16")


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_gentree_star_executes(dtype):
    """tab:gentreesimu's GenTree* (force "norearrange") runs through the same executor
    on the topology where GenTree rearranges: emulated ranks, bit-exact vs the oracle."""
    from tests.topologies import cross_dc
    run_emulated(cross_dc(2, 3, 2, 3), 12, 123457, dtype, force="norearrange")


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_emulated_cps_flag_protocol(dtype, monkeypatch):
    """Emulated CPS plans normally run flag-free (ar_flat_kernel); AR_FLAT=0 keeps them on the
    step-table kernel and its flag protocol — both must give the plan's bits."""
    monkeypatch.setenv("AR_FLAT", "0")
    for world in (3, 8):
        for count in (world * 4096 + 7, 300001):
            run_emulated(single_switch(world), world, count, dtype, force="cps", calls=2)
            run_emulated(single_switch(world), world, count, dtype, force="cps", red="avg")


@pytest.mark.parametrize("dyn", ["0", "1"])
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_flat_kernel_static_and_dynamic_tiles(dyn, dtype, monkeypatch):
    """ar_flat_kernel with static slices (AR_DYN=0) and with tiles handed out by the per-block
    atomic counters (default): same plan bits, over back-to-back calls (the counters must be
    back at zero for the next launch), ragged sizes, SUM and AVG, R = 2..8 (dynamic) and 9."""
    monkeypatch.setenv("AR_DYN", dyn)
    for world in (2, 5, 8, 9):
        for count in (world * 4096 + 7, 1000003):
            run_emulated(single_switch(world), world, count, dtype, force="cps", calls=3)
            run_emulated(single_switch(world), world, count, dtype, force="cps", red="avg")


@pytest.mark.parametrize("force", [None, "ring"])
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_exec_host_end_to_end(force, dtype):
    """allreduce_exec_host from pinned host memory: natural-CPS plans run chunked (sub-plans
    per element range, H2D/AllReduce/D2H overlapped on three streams), other plans in one
    piece — both must return the plan's bits in the host buffer."""
    world = 4
    count = (9 << 20) // (4 if dtype == "f32" else 2) + 333      # > 8 MiB per rank, ragged
    es = 4 if dtype == "f32" else 2
    stride = G.rank_stride_bytes(count, dtype)
    plan = G.Plan.from_topology(single_switch(world), count, dtype, None, force)
    comm = G.Comm.local(world, 0)
    dbuf = torch.zeros(world * stride, dtype=torch.uint8, device="cuda")
    host = torch.zeros(world * stride, dtype=torch.uint8, pin_memory=True)
    xs = GEN.generate_all(SEED, world, count, dtype)
    hv = host.numpy()
    for r in range(world):
        hv[r * stride: r * stride + count * es] = xs[r].view(np.uint8)
    for _ in range(2):
        G.allreduce_exec_host(plan, comm, dbuf, host.data_ptr(), count, dtype)
    torch.cuda.synchronize()
    comm.async_error()
    oplan, _ = GT.gentree(T.parse_topology(single_switch(world)), count, es, force=force)
    want = SM.simulate(oplan, SM.simulate(oplan, xs, dtype), dtype)
    for r in range(world):
        got = hv[r * stride: r * stride + count * es].view(np.float32 if dtype == "f32" else np.uint16)
        assert_bits_equal(got, want[r], dtype, f"rank {r}")


@pytest.mark.parametrize("flatsteps", ["1", "0"])
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_multi_step_kernels(flatsteps, dtype, monkeypatch):
    """Emulated multi-step plans run on the step-table kernel and its per-rank flags; the A/B
    option AR_FLATSTEPS=1 runs them on ar_flatsteps_kernel (every step's ops of all ranks over
    every SM, grid barriers between steps) — both with the plan's bits: every kind, ragged
    sizes, SUM and AVG, back-to-back calls (the barrier words must be back at zero), specials."""
    monkeypatch.setenv("AR_FLATSTEPS", flatsteps)
    kern = "ar_flatsteps_kernel" if flatsteps == "1" else "ar_exec_kernel"
    for force in ("ring", "rhd", "hcps:4,2", "hcps:2,2,2"):
        for count in (8 * 4096 + 7, 1000003):
            run_emulated(single_switch(8), 8, count, dtype, force=force, calls=2, expect_kernel=kern)
        run_emulated(single_switch(8), 8, 300001, dtype, force=force, red="avg", expect_kernel=kern)
    run_emulated(single_switch(8), 8, 300001, dtype, force="ring", mode="specials", expect_kernel=kern)
    for world in (3, 5):
        run_emulated(single_switch(world), world, 200003, dtype, force="ring", expect_kernel=kern)
    c1 = T.two_level_doc([2, 2], T.TABLE5["root_sw"], T.TABLE5["middle_sw"], T.TABLE5["server"])
    run_emulated(c1, 4, 100003, dtype, expect_kernel=kern)          # C1's two-level GenTree plan
