"""Worker for tests/test_gpu_multi.py: one process per GPU (torchrun), real IPC peer maps
over NVLink.  Every rank checks its own output bit-for-bit against the CPU oracle run on
all ranks' (deterministic) inputs.  Exit code 0 = all cases bit-exact."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2409_04202_b200 as G  # noqa: E402
from oracle import gentree as GT  # noqa: E402
from oracle import plans as OP  # noqa: E402
from oracle import simulate as SM  # noqa: E402
from oracle import topology as T  # noqa: E402
from synth import generator as GEN  # noqa: E402
from tests.gpu_util import assert_bits_equal, cps_path_kernel  # noqa: E402


def main():
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    comm = G.Comm.create(rank, world, local)
    doc = T.single_switch_doc(world, {"alpha": 3e-6, "beta": 4 / 900e9, "epsilon": 0.0, "w_t": 9},
                              {"gamma": 0.0, "delta": 4 / 6.54e12})
    kinds = [None, "cps", "ring", "rb"]
    if world & (world - 1) == 0:
        kinds.append("rhd")
    if world == 4:
        kinds.append("hcps:2,2")
    if world == 8:
        kinds += ["hcps:4,2", "hcps:2,4", "hcps:2,2,2"]
    cases = [(doc, k) for k in kinds]
    # NEXT #3: multi-level trees executed across GPUs — C1's 2x2 tree on 4 GPUs (P:1034,
    # Table 5 rows), a 2x4 tree and a rearranging cross-DC tree on 8
    tl = lambda sizes: T.two_level_doc(sizes, T.TABLE5["root_sw"], T.TABLE5["middle_sw"], T.TABLE5["server"])
    if world == 4:
        cases.append((tl([2, 2]), None))
    if world == 8:
        from tests.topologies import cross_dc
        cases += [(tl([4, 4]), None), (tl([3, 5]), None), (cross_dc(2, 2, 2, 2), None)]
    seed = GEN.config_seed(2)
    keep = []
    failures = 0
    for dtype in ("f32", "bf16"):
        es = 4 if dtype == "f32" else 2
        for count in (1, world * 4096 + 5, world * 4 * 40000, 1 << 20, 3_000_001):
            buf = torch.zeros(max(16, count * es), dtype=torch.uint8, device="cuda")
            keep.append(buf)
            comm.register(buf)
            for doc_i, force in cases:
                topo = T.parse_topology(doc_i)
                G.fill_synthetic(buf, count, dtype, seed, rank, 0)
                plan = G.Plan.from_topology(doc_i, count, dtype, None, force)
                oplan, _ = GT.gentree(topo, count, es, force=force)
                assert plan.to_json() == OP.plan_to_json(oplan, dtype)
                # second call: AVG on ring/default plans (reading AV1), SUM otherwise
                op2 = "avg" if force in (None, "ring") else "sum"
                G.allreduce_exec(plan, comm, buf)
                G.allreduce_exec(plan, comm, buf, op=op2)
                torch.cuda.synchronize()
                comm.async_error()
                xs = GEN.generate_all(seed, world, count, dtype)
                want = SM.simulate(oplan, SM.simulate(oplan, xs, dtype), dtype, op=op2)[rank]
                got = buf.cpu().numpy()[: count * es].view(np.float32 if dtype == "f32" else np.uint16)
                try:
                    assert_bits_equal(got, want, dtype, f"rank {rank} {dtype} count={count} plan={force}")
                except AssertionError as e:
                    print(e, flush=True)
                    failures += 1
                dist.barrier()
    # bench.py's N > 1 workload at full size (bf16, 256 MiB per rank, GenTree plan, the launch
    # configuration bench times): EVERY element of this rank's buffer vs the oracle
    count = 128 * 1024 * 1024
    buf = torch.empty(count * 2, dtype=torch.uint8, device="cuda")
    comm.register(buf)
    G.fill_synthetic(buf, count, "bf16", seed + 3, rank, 0)
    plan = G.Plan.from_topology(doc, count, "bf16")
    oplan, _ = GT.gentree(T.parse_topology(doc), count, 2)
    torch.cuda.synchronize()
    dist.barrier()
    G.allreduce_exec(plan, comm, buf)
    torch.cuda.synchronize()
    comm.async_error()
    want = SM.simulate(oplan, GEN.generate_all(seed + 3, world, count, "bf16"), "bf16")[rank]
    got = buf.cpu().numpy().view(np.uint16)
    try:
        assert_bits_equal(got, want, "bf16", f"rank {rank} full-size full buffer")
    except AssertionError as e:
        print(e, flush=True)
        failures += 1
    del want, got
    del buf
    dist.barrier()

    # end to end from pinned host memory (chunked natural-CPS sub-plans on interior pointers
    # of the registered buffer; allreduce_exec_host)
    for dtype in ("f32", "bf16"):
        es = 4 if dtype == "f32" else 2
        count = (9 << 20) // es + 333
        buf = torch.zeros(count * es + 16, dtype=torch.uint8, device="cuda")
        keep.append(buf)
        comm.register(buf)
        host = torch.zeros(count * es, dtype=torch.uint8, pin_memory=True)
        xs = GEN.generate_all(seed + 2, world, count, dtype)
        host.numpy()[:] = xs[rank].view(np.uint8)
        plan = G.Plan.from_topology(doc, count, dtype, None, None)
        oplan, _ = GT.gentree(T.parse_topology(doc), count, es)
        dist.barrier()
        G.allreduce_exec_host(plan, comm, buf, host.data_ptr(), count, dtype)
        torch.cuda.synchronize()
        comm.async_error()
        want = SM.simulate(oplan, xs, dtype)[rank]
        got = host.numpy().view(np.float32 if dtype == "f32" else np.uint16)
        try:
            assert_bits_equal(got, want, dtype, f"rank {rank} {dtype} host end-to-end")
        except AssertionError as e:
            print(e, flush=True)
            failures += 1
        dist.barrier()

    # back-to-back small calls without host syncs: the one-shot low-latency path (double-
    # buffered scratch, epoch-tagged lines) interleaved with the flag-protocol path
    # (3001 elements: one-shot path; 600_001: push protocol; ring: flag protocol)
    for dtype, count in (("f32", 3001), ("bf16", 3001), ("f32", 600_001), ("bf16", 600_001)):
        es = 4 if dtype == "f32" else 2
        buf = torch.zeros(count * es + 16, dtype=torch.uint8, device="cuda")
        keep.append(buf)
        comm.register(buf)
        topo = T.parse_topology(doc)
        pc = G.Plan.from_topology(doc, count, dtype, None, "cps")
        pr = G.Plan.from_topology(doc, count, dtype, None, "ring")
        oc, _ = GT.gentree(topo, count, es, force="cps")
        orr, _ = GT.gentree(topo, count, es, force="ring")
        seq = ["cps"] * 6 + ["ring"] + ["cps"] * 5 + ["ring", "cps"]
        G.fill_synthetic(buf, count, dtype, seed + 1, rank, 0)
        torch.cuda.synchronize()
        dist.barrier()
        for k in seq:
            G.allreduce_exec(pc if k == "cps" else pr, comm, buf)
        torch.cuda.synchronize()
        comm.async_error()
        want = GEN.generate_all(seed + 1, world, count, dtype)
        for k in seq:
            want = SM.simulate(oc if k == "cps" else orr, want, dtype)
        got = buf.cpu().numpy()[: count * es].view(np.float32 if dtype == "f32" else np.uint16)
        try:
            assert_bits_equal(got, want[rank], dtype, f"rank {rank} {dtype} count={count} back-to-back calls")
        except AssertionError as e:
            print(e, flush=True)
            failures += 1
        dist.barrier()
    # the one-shot cut-off is settable (ar_comm_set_oneshot_max): off, then raised to 2x
    default_cut = G.default_paths(world)["oneshot_max"]
    assert comm.paths()["oneshot_max"] == default_cut
    for cut, count in ((0, 3001), (2 * default_cut, (2 * default_cut) // 4 - 100)):
        comm.set_oneshot_max(cut)
        buf = torch.zeros(count * 4 + 16, dtype=torch.uint8, device="cuda")
        keep.append(buf)
        comm.register(buf)
        G.fill_synthetic(buf, count, "f32", seed + 4, rank, 0)
        plan = G.Plan.from_topology(doc, count, "f32")
        oplan, _ = GT.gentree(T.parse_topology(doc), count, 4)
        torch.cuda.synchronize()
        dist.barrier()
        G.allreduce_exec(plan, comm, buf)
        torch.cuda.synchronize()
        comm.async_error()
        expect = cps_path_kernel(comm.paths(), count, 4, world)   # LL128 precedes the one-shot path
        want = SM.simulate(oplan, GEN.generate_all(seed + 4, world, count, "f32"), "f32")[rank]
        got = buf.cpu().numpy()[: count * 4].view(np.float32)
        try:
            assert comm.last_kernel() == expect, comm.last_kernel()
            assert_bits_equal(got, want, "f32", f"rank {rank} one-shot cut-off {cut}")
        except AssertionError as e:
            print(e, flush=True)
            failures += 1
        dist.barrier()
    comm.set_oneshot_max(default_cut)
    dist.barrier()
    comm.destroy()
    dist.destroy_process_group()
    if rank == 0:
        print(f"mp_worker world={world}: {'OK' if failures == 0 else f'{failures} FAILURES'}", flush=True)
    sys.exit(1 if failures else 0)


if __name__ == "__main__":
    main()
