"""Probe: one CPS AllReduce split between the LL128 two-shot kernel and the step-table kernel,
running side by side (torchrun, N GPUs, fp32).

    AR_LL128_MAX_KB=... python -m torch.distributed.run --nproc-per-node N tools/ll128_exec_split.py

For a message of S bytes and a share x, the first x·S bytes (a natural-CPS sub-plan on the
registered buffer's first elements: equal 16-byte-aligned blocks, so the LL128 path takes it)
and the remaining bytes (one element fewer than a multiple of N, so the step-table kernel
takes it; same bits — a CPS element's sum does not depend on the block partition) are issued
on two streams after one event; the time is until both finished (CUDA events, max over ranks,
median of 20).  The step-table kernel's fixed per-call cost (entry and exit flag rounds,
≈ 15 µs) can then overlap the LL128 kernel's data movement.  A measurement probe.
"""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2409_04202_b200 as G  # noqa: E402
from tools.harness import doc  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    comm = G.Comm.create(rank, world, local)
    ctas = int(os.environ.get("SPLIT_EXEC_CTAS", "0"))
    if ctas:
        comm.set_ctas(ctas)
    sizes = [int(s) for s in os.environ.get("SPLIT_SIZES", " ".join(str(m << 20) for m in (32, 64, 128, 256))).split()]
    shares = [float(x) for x in os.environ.get("SPLIT_SHARES", "0 0.1 0.2 0.3 0.4 0.5 1").split()]
    maxb = max(sizes)
    buf = torch.empty(maxb + 64, dtype=torch.uint8, device="cuda")
    comm.register(buf)
    paths = comm.paths()
    sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
    unit = world * 4               # fp32 elements: equal blocks of whole 16-byte vectors
    for nbytes in sizes:
        count = nbytes // 4
        for x in shares:
            c1 = int(count * x) // unit * unit
            c2 = count - c1
            if 0 < c2 < count and c2 % world == 0:
                c2 -= 1                # ragged: the step-table kernel, not LL128
            p1 = G.Plan.from_topology(doc(world), c1, "f32") if c1 else None
            p2 = G.Plan.from_topology(doc(world), c2, "f32") if c2 else None
            e1 = G.Executor(p1, comm, buf, stream=sa) if p1 else None
            e2 = G.Executor(p2, comm, buf.data_ptr() + c1 * 4, stream=sb) if p2 else None

            def once():
                ev = torch.cuda.Event()
                ev.record()
                sa.wait_event(ev)
                sb.wait_event(ev)
                if e1:
                    e1()
                if e2:
                    e2()
                torch.cuda.current_stream().wait_stream(sa)
                torch.cuda.current_stream().wait_stream(sb)

            def refill():
                G.fill_synthetic(buf, c1 + c2, "f32", 11, rank, 0)

            refill()
            for _ in range(5):
                once()
            kernels = comm.last_kernel()
            torch.cuda.synchronize()
            dist.barrier()
            reps = 20
            evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
            for i in range(reps):
                if i % 8 == 0:
                    refill()
                evs[i][0].record()
                once()
                evs[i][1].record()
            torch.cuda.synchronize()
            ts = torch.tensor([a.elapsed_time(b) / 1e3 for a, b in evs], dtype=torch.float64, device="cuda")
            dist.all_reduce(ts, op=dist.ReduceOp.MAX)
            ts = ts.cpu().tolist()
            comm.async_error()
            t = statistics.median(ts)
            if rank == 0:
                print(json.dumps({"tool": "ll128_exec_split", "n": world, "bytes": nbytes, "ll128_share": x,
                                  "ll128_bytes": c1 * 4, "exec_bytes": c2 * 4, "exec_ctas": ctas or "auto",
                                  "ll128_ctas": os.environ.get("AR_LL128_CTAS", "auto"), "paths": paths,
                                  "last_kernel": kernels, "t_med": t, "t_min": min(ts),
                                  "busbw_med": (c1 + c2) * 4 / t * 2 * (world - 1) / world / 1e9}), flush=True)
    comm.destroy()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
