"""GPU parity of the MULTI-PROCESS communicator path, driven from one process on one GPU.

The driver's GPU tests run on a single B200, where the torchrun tests (tests/test_gpu_multi.py)
cannot run.  Here `world` communicators are created with ar_comm_create (one per rank, the
same object a process per GPU would hold), their buffers are exchanged with
ar_comm_register / ar_comm_open_peers (same-process peers are mapped by raw pointer instead of
CUDA IPC — the only difference from the cross-process path), and every rank's kernel is
launched on its own stream with world × CTAs ≤ the SM count so all ranks' persistent kernels
are resident together.  This exercises exactly the code the multi-GPU path runs: the
step-table kernel with system-scope (.sys) release/acquire flags, dynamic tiles of CPS-shaped
plans over the comm path, the push protocol, and the one-shot small-message kernel
(ar_ll_kernel) — checked bit-for-bit against the CPU oracle (north star).
"""
import os

import numpy as np
import pytest

from tests.gpu_util import assert_bits_equal, cuda_ok

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
SEED = GEN.config_seed(7)


def single_switch(world):
    return T.single_switch_doc(world, {"alpha": 3e-6, "beta": 4 / 900e9, "epsilon": 0.0, "w_t": 9},
                               {"gamma": 0.0, "delta": 4 / 6.54e12})


class SameProcess:
    """`world` multi-process communicators living in this process on cuda:0."""

    def __init__(self, world, nbytes, env=None):
        self.world = world
        old = {}
        env = dict(env or {})
        env.setdefault("AR_FLAG_TIMEOUT_MS", "8000")   # a residency problem errors out, never hangs
        for k, v in env.items():
            old[k] = os.environ.get(k)
            os.environ[k] = v
        try:
            self.comms = [G.Comm.create(r, world, 0) for r in range(world)]
        finally:
            for k, v in old.items():
                if v is None:
                    os.environ.pop(k, None)
                else:
                    os.environ[k] = v
        nsm = torch.cuda.get_device_properties(0).multi_processor_count
        for c in self.comms:
            c.set_ctas(nsm // world)     # all ranks' persistent kernels resident together
        self.bufs = [torch.zeros(nbytes, dtype=torch.uint8, device="cuda") for _ in range(world)]
        blobs = [c.export(b) for c, b in zip(self.comms, self.bufs)]
        for c in self.comms:
            c.open_peers(blobs)
        self.streams = [torch.cuda.Stream() for _ in range(world)]

    def fill(self, count, dtype, mode):
        for r, b in enumerate(self.bufs):
            G.fill_synthetic(b, count, dtype, SEED, r, MODES[mode])
        torch.cuda.synchronize()

    def views(self, count, dtype):
        es = 4 if dtype == "f32" else 2
        out = []
        for b in self.bufs:
            raw = b.cpu().numpy()[: count * es]
            out.append(raw.view(np.float32 if dtype == "f32" else np.uint16).copy())
        return out

    def run(self, plan, count, dtype, op="sum"):
        torch.cuda.synchronize()
        for r in range(self.world):
            G.allreduce_exec(plan, self.comms[r], self.bufs[r], count, dtype, stream=self.streams[r], op=op)
        torch.cuda.synchronize()
        for c in self.comms:
            c.async_error()
        return [c.last_kernel() for c in self.comms]

    def destroy(self):
        for c in self.comms:
            c.destroy()


def oracle_plan(world, count, dtype, force):
    oplan, _ = GT.gentree(T.parse_topology(single_switch(world)), count, 4 if dtype == "f32" else 2, force=force)
    return oplan


def check(sp, world, count, dtype, force, mode="gradient", op="sum", calls=1, expect_kernel=None):
    plan = G.Plan.from_topology(single_switch(world), count, dtype, None, force)
    oplan = oracle_plan(world, count, dtype, force)
    assert plan.to_json() == OP.plan_to_json(oplan, dtype)
    sp.fill(count, dtype, mode)
    want = GEN.generate_all(SEED, world, count, dtype, mode)
    kernels = None
    for _ in range(calls):
        kernels = sp.run(plan, count, dtype, op)
        want = SM.simulate(oplan, want, dtype, op=op)
    got = sp.views(count, dtype)
    for r in range(world):
        assert_bits_equal(got[r], want[r], dtype, f"{force or 'gentree'} rank {r}")
    if expect_kernel:
        assert set(kernels) == {expect_kernel}, kernels
    return got


@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_flag_path_all_kinds(world, dtype):
    """ar_exec_kernel with .sys flags: every plan kind, ragged count (> one-shot cut-off; the
    LL128 path, which would take the CPS-shaped ones, switched off)."""
    count = 1_000_003 if dtype == "f32" else 2_000_003
    sp = SameProcess(world, count * 4, env={"AR_LL128_MAX_KB": "0"})
    try:
        kinds = [None, "cps", "ring", "rb"] + {4: ["rhd", "hcps:2,2"], 8: ["rhd", "hcps:4,2"]}.get(world, ["rhd"])
        for force in kinds:
            check(sp, world, count, dtype, force, expect_kernel="ar_exec_kernel")
    finally:
        sp.destroy()


@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_oneshot_path(world, dtype):
    """ar_ll_kernel (small messages, CPS-shaped plans, up to the LL128 floor): bit-identical to
    the plan's bits."""
    es = 4 if dtype == "f32" else 2
    top = min(60001, G.default_paths(world)["ll128_min"] // es - 1)
    sp = SameProcess(world, 1 << 20)
    try:
        for count in (1, 7, 4093, top):
            check(sp, world, count, dtype, None, expect_kernel="ar_ll_kernel")
        if world > 2:   # multi-step plans never take the one-shot path (at N = 2 Ring ≡ CPS)
            check(sp, world, top, dtype, "ring", expect_kernel="ar_exec_kernel")
    finally:
        sp.destroy()


@pytest.mark.parametrize("mode", ["integer", "specials"])
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_modes_every_path(mode, dtype):
    """±0, subnormals, ±max (overflow), ±inf, NaN and integer-valued inputs through the
    one-shot path, the dynamic-tile CPS step and the multi-step kinds."""
    world = 4
    big = 900_007 if dtype == "f32" else 1_800_007
    for env, cases in (({}, [(30011, None, "ar_ll_kernel"), (big, None, "ar_ll128_kernel"),
                             (big, "ring", "ar_exec_kernel"), (big, "rhd", "ar_exec_kernel"),
                             (big, "hcps:2,2", "ar_exec_kernel"),
                             (big, "rb", "ar_ll128_kernel")]),     # RB's blocks share one order
                       ({"AR_LL128_MAX_KB": "0"}, [(big, None, "ar_exec_kernel")])):
        sp = SameProcess(world, 4 << 20, env=env)
        try:
            for count, force, kern in cases:
                got = check(sp, world, count, dtype, force, mode=mode, expect_kernel=kern)
                if mode == "integer":
                    xs = GEN.generate_all(SEED, world, count, dtype, "integer")
                    ref = sum(GEN.as_f64(x, dtype).astype(np.int64) for x in xs)
                    assert np.array_equal(GEN.as_f64(got[1], dtype).astype(np.int64), ref)
        finally:
            sp.destroy()


def test_avg_and_back_to_back():
    """AVG (reading AV1) on both paths; 3 back-to-back calls alternating the one-shot and the
    flag path on the same communicators (epochs and scratch parity carried across calls)."""
    world = 4
    sp = SameProcess(world, 8 << 20)
    try:
        check(sp, world, 50001, "bf16", None, op="avg", expect_kernel="ar_ll_kernel")
        check(sp, world, 1_500_001, "f32", None, op="avg", expect_kernel="ar_ll128_kernel")
        check(sp, world, 1_500_001, "f32", "ring", op="avg")
        for count in (40001, 1_200_001, 40001):
            check(sp, world, count, "f32", None, calls=3)
    finally:
        sp.destroy()


def test_push_protocol_and_jitter():
    """The push protocol (AR_PUSH_MAX_MB) and randomly delayed flag posts (AR_JITTER_NS)."""
    world = 4
    sp = SameProcess(world, 8 << 20, env={"AR_PUSH_MAX_MB": "16", "AR_LL128_MAX_KB": "0"})
    try:
        check(sp, world, 1_000_003, "f32", None, calls=2, expect_kernel="ar_exec_kernel")
        check(sp, world, 2_000_001, "bf16", None)
    finally:
        sp.destroy()
    sp = SameProcess(world, 8 << 20, env={"AR_JITTER_NS": "20000", "AR_LL_MAX_KB": "0", "AR_LL128_MAX_KB": "0"})
    try:
        for force in (None, "ring", "rhd", "hcps:2,2"):
            check(sp, world, 600_001, "f32", force, calls=2, expect_kernel="ar_exec_kernel")
    finally:
        sp.destroy()


def test_settings_are_checked():
    """The blobs carry the settings every rank must share (ADVICE: CTA count, one-shot
    scratch): a mismatch is refused at open_peers, and the CTA count is frozen afterwards."""
    world = 2
    comms = [G.Comm.create(r, world, 0) for r in range(world)]
    bufs = [torch.zeros(1 << 20, dtype=torch.uint8, device="cuda") for _ in range(world)]
    try:
        comms[0].set_ctas(60)
        comms[1].set_ctas(70)
        blobs = [c.export(b) for c, b in zip(comms, bufs)]
        with pytest.raises(Exception, match="settings"):
            comms[0].open_peers(blobs)
        comms[1].set_ctas(60)
        blobs = [c.export(b) for c, b in zip(comms, bufs)]
        for c in comms:
            c.open_peers(blobs)
        with pytest.raises(Exception, match="set_ctas"):
            comms[0].set_ctas(50)
        comms[0].set_ctas(60)   # unchanged value is fine
    finally:
        for c in comms:
            c.destroy()


def test_open_peers_selects_the_right_registration():
    """Two registrations of the same size: open_peers binds the one whose blob it is given.
    (Above the LL128 ceiling: the flag-free paths read only the local buffer and the
    communicator's own scratch, so they need no registration — only a buffer that holds count
    elements.)"""
    world = 2
    count = G.default_paths(world)["ll128_max"] // 4 + 1001
    comms = [G.Comm.create(r, world, 0) for r in range(world)]
    a = [torch.zeros(count * 4, dtype=torch.uint8, device="cuda") for _ in range(world)]
    b = [torch.zeros(count * 4, dtype=torch.uint8, device="cuda") for _ in range(world)]
    streams = [torch.cuda.Stream() for _ in range(world)]
    try:
        for c in comms:
            c.set_ctas(64)
        blobs_a = [c.export(x) for c, x in zip(comms, a)]
        blobs_b = [c.export(x) for c, x in zip(comms, b)]   # registered last
        for c in comms:
            c.open_peers(blobs_a)                             # must bind a, not b
        for r in range(world):
            G.fill_synthetic(a[r], count, "f32", SEED, r, 0)
        torch.cuda.synchronize()
        plan = G.Plan.from_topology(single_switch(world), count, "f32")
        for r in range(world):
            G.allreduce_exec(plan, comms[r], a[r], stream=streams[r])
        torch.cuda.synchronize()
        for c in comms:
            c.async_error()
        oplan = oracle_plan(world, count, "f32", None)
        want = SM.simulate(oplan, GEN.generate_all(SEED, world, count, "f32"), "f32")
        for r in range(world):
            assert_bits_equal(a[r].cpu().numpy().view(np.float32), want[r], "f32", f"rank {r}")
        with pytest.raises(Exception, match="not registered"):   # b was never opened
            G.allreduce_exec(plan, comms[0], b[0], stream=streams[0])
        # a flag-free path's size (LL128) on a buffer (a 2 MiB pool segment) too small for it
        small = torch.zeros(4096, dtype=torch.uint8, device="cuda")
        with pytest.raises(Exception, match="too small"):
            G.allreduce_exec(G.Plan.from_topology(single_switch(world), 1_000_001, "f32"), comms[0],
                             small[256:], 1_000_001, "f32", stream=streams[0])
        del blobs_b
    finally:
        for c in comms:
            c.destroy()


def test_unverified_plan_is_refused():
    """allreduce_exec refuses a plan that fails symbolic verification (duplicate inputs would
    otherwise overrun the kernel's source table); data-movement plans have their own entry."""
    import json
    world, count = 2, 1024
    bad = {"count": count, "dtype": "f32", "n": world, "steps": [
        {"label": "rs", "phase": "rs", "transfers": [],
         "reduces": [{"block": b, "fan_in": 100, "inputs": [0] * 50 + [1] * 50, "server": b} for b in range(world)]}]}
    plan = G.Plan.from_json(json.dumps(bad))
    assert not plan.is_allreduce
    comm = G.Comm.local(world, 0)
    buf = torch.zeros(G.rank_stride_bytes(count, "f32") * world, dtype=torch.uint8, device="cuda")
    try:
        with pytest.raises(Exception, match="not an AllReduce"):
            G.allreduce_exec(plan, comm, buf)
        with pytest.raises(Exception, match="AR_MAX_RANKS"):
            G.Executor(plan, comm, buf, movement=True)()
        with pytest.raises(ValueError, match="needs"):
            good = G.Plan.from_topology(single_switch(world), count, "f32")
            G.allreduce_exec(good, comm, buf[: count * 4])
    finally:
        comm.destroy()


@pytest.mark.parametrize("world", [2, 3, 4, 8])
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_ll128_path(world, dtype):
    """ar_ll128_kernel (CPS-shaped plans between the LL128 floor and ceiling): the CPS plan's RS
    and AG steps with the flag inside every 128-byte line, over the kernel's own block
    partition (8-byte-multiple blocks, the remainder on the last one — down to a 2- or 4-byte
    partial word) — bit-identical to the plan's Q3 partition; partial last lines; SUM and AVG;
    back-to-back calls alternating with the one-shot and the flag paths on the same
    communicators (epoch parity of both scratch areas); N = 3 (no count is a multiple of N·16
    bytes there at powers of two)."""
    es = 4 if dtype == "f32" else 2
    paths = G.default_paths(world)
    sp = SameProcess(world, 16 << 20)
    unit = world * 16 // es                        # equal blocks starting on 16-byte boundaries
    try:
        top = min(16 << 20, paths["ll128_max"]) // es
        sizes = [(2 << 20) // es // unit * unit, 2_000_000 // unit * unit, top - unit]
        ragged = [(1 << 20) // es + 1, 1_000_003 if dtype == "f32" else 2_000_003, top - 1,
                  paths["ll128_min"] // es + 3]
        for count in sizes + ragged:
            check(sp, world, count, dtype, None, expect_kernel="ar_ll128_kernel")
        check(sp, world, sizes[1], dtype, None, op="avg", expect_kernel="ar_ll128_kernel")
        check(sp, world, ragged[1], dtype, None, op="avg", expect_kernel="ar_ll128_kernel")
        for count, kern in ((sizes[0], "ar_ll128_kernel"), (4093, "ar_ll_kernel"), (sizes[0] + 1, "ar_ll128_kernel"),
                            (ragged[0], "ar_ll128_kernel"), (sizes[1], "ar_ll128_kernel"),
                            (sizes[1], "ar_ll128_kernel")):
            check(sp, world, count, dtype, None, calls=2, expect_kernel=kern)
        for mode in ("integer", "specials"):
            check(sp, world, sizes[1], dtype, None, mode=mode, expect_kernel="ar_ll128_kernel")
            check(sp, world, ragged[1], dtype, None, mode=mode, expect_kernel="ar_ll128_kernel")
        if world > 2:   # multi-step plans never take it
            check(sp, world, sizes[0], dtype, "ring", expect_kernel="ar_exec_kernel")
    finally:
        sp.destroy()


@pytest.mark.parametrize("nproc,R", [(2, 4), (4, 2), (2, 8)])
def test_multi_level_same_process(nproc, R):
    """Multi-level execution (SURVEY §8(f) NEXT #3, config C5's "8 ranks per GPU", C1's
    two-level tree): `nproc` communicators from ar_comm_create_multi, each hosting R
    consecutive ranks in one buffer, living in this process on cuda:0 — the code path of one
    process per GPU (system-scope flags, per-process flag-page blocks, peers' rank slots at
    peer_base + (r mod R)·stride), with same-process peers mapped by raw pointer.  The GenTree
    plan of the two-level tree (leaf level among a process's ranks, root level across
    processes) and forced flat kinds that mix hosted and peer ranks inside every step; SUM then
    AVG; bit-exact against the oracle on every rank."""
    world = nproc * R
    nsm = torch.cuda.get_device_properties(0).multi_processor_count
    old = os.environ.get("AR_FLAG_TIMEOUT_MS")
    os.environ["AR_FLAG_TIMEOUT_MS"] = "8000"
    try:
        comms = [G.Comm.create_multi(p, nproc, R, 0) for p in range(nproc)]
    finally:
        if old is None:
            os.environ.pop("AR_FLAG_TIMEOUT_MS", None)
        else:
            os.environ["AR_FLAG_TIMEOUT_MS"] = old
    try:
        for c in comms:
            c.set_ctas(max(1, nsm // world))   # every hosted rank of every process resident at once
        nvl = {"alpha": 1e-5, "beta": 4.0 / 770e9, "epsilon": 0.0, "w_t": 9}
        hbm = {"alpha": 3e-6, "beta": 4.0 / 3000e9, "epsilon": 0.0, "w_t": 64}
        server = {"gamma": 0.0, "delta": 4.0 / 6.5e12}
        tree = T.two_level_doc([R] * nproc, nvl, hbm, server)
        flat = T.single_switch_doc(world, nvl, server)
        streams = [torch.cuda.Stream() for _ in range(nproc)]
        for dtype in ("f32", "bf16"):
            es = 4 if dtype == "f32" else 2
            for count in (world * 1024 + 7, 1 << 18):
                stride = G.rank_stride_bytes(count, dtype)
                bufs = [torch.zeros(stride * R, dtype=torch.uint8, device="cuda") for _ in range(nproc)]
                blobs = [c.export(b) for c, b in zip(comms, bufs)]
                for c in comms:
                    c.open_peers(blobs)
                for doc, force in ((tree, None), (flat, "cps"), (flat, "ring")):
                    for p in range(nproc):
                        for i in range(R):
                            G.fill_synthetic(bufs[p].data_ptr() + i * stride, count, dtype, SEED, p * R + i, 0)
                    plan = G.Plan.from_topology(doc, count, dtype, None, force)
                    oplan, _ = GT.gentree(T.parse_topology(doc), count, es, force=force)
                    assert plan.to_json() == OP.plan_to_json(oplan, dtype)
                    torch.cuda.synchronize()
                    for op in ("sum", "avg"):
                        for p in range(nproc):
                            G.allreduce_exec(plan, comms[p], bufs[p], count, dtype, stream=streams[p], op=op)
                    torch.cuda.synchronize()
                    for c in comms:
                        c.async_error()
                        assert c.last_kernel() == "ar_exec_kernel"
                    xs = GEN.generate_all(SEED, world, count, dtype)
                    want = SM.simulate(oplan, SM.simulate(oplan, xs, dtype), dtype, op="avg")
                    for p in range(nproc):
                        host = bufs[p].cpu().numpy()
                        for i in range(R):
                            got = host[i * stride: i * stride + count * es].view(
                                np.float32 if dtype == "f32" else np.uint16)
                            assert_bits_equal(got, want[p * R + i], dtype,
                                              f"{force or 'tree'} {dtype} count={count} rank {p * R + i}")
    finally:
        for c in comms:
            c.destroy()


@pytest.mark.parametrize("world", [2, 3, 4, 8])
def test_path_choice_follows_the_cutoffs(world):
    """The executor's path for CPS-shaped plans follows the communicator's cut-offs
    (ar_comm_get_paths = ar_default_paths by default): LL128 in (ll128_min, ll128_max] — any
    count, ahead of the one-shot path — one-shot up to oneshot_max otherwise,
    the step-table kernel above; every path with the plan's bits."""
    paths = G.default_paths(world)
    sp = SameProcess(world, paths["ll128_max"] + (1 << 20))
    try:
        assert sp.comms[0].paths() == paths
        unit = world * 4                                   # fp32: blocks of whole 16-byte vectors
        lo, hi = paths["ll128_min"] // 4 // unit * unit, paths["ll128_max"] // 4 // unit * unit
        cases = [(lo, "ar_ll_kernel"),                     # at the floor: one-shot
                 (lo + unit, "ar_ll128_kernel"),           # just above: LL128
                 (lo + unit + 1, "ar_ll128_kernel"),       # ragged blocks: LL128 (its own partition)
                 (lo - 3, "ar_ll_kernel"),                 # ragged below the floor: one-shot
                 (hi, "ar_ll128_kernel"),                  # the ceiling
                 (hi + unit, "ar_exec_kernel")]            # above it
        for count, kern in cases:
            check(sp, world, count, "f32", None, expect_kernel=kern)
    finally:
        sp.destroy()
