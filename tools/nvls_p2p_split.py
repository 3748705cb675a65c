"""Probe: do the NVLS kernel and the P2P executor share NVLink capacity, or does running them
side by side on disjoint parts of one AllReduce move more bytes per second than either alone?
(torchrun, N GPUs, fp32)

    python -m torch.distributed.run --nproc-per-node N tools/nvls_p2p_split.py

For a message of S bytes and a share x, the first x·S bytes are reduced by the NVLS kernel
(multicast buffer, its 16 CTAs, stream A) and the rest by the GenTree plan on the P2P executor
(IPC-registered buffer, 148 − 16 CTAs so both kernels are resident, stream B); both start
after one event and the time is until both finished (CUDA events, max over ranks, median of
the repetitions).  busbw counts S.  A measurement probe: it answers whether a split NVLS + P2P
plan kind could pass either path's ceiling; nothing on the product path uses it.
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
    nsm = torch.cuda.get_device_properties(local).multi_processor_count
    nv_ctas = int(os.environ.get("AR_NVLS_CTAS", "16"))
    comm = G.Comm.create(rank, world, local)
    comm.set_ctas(nsm - nv_ctas)
    sizes = [int(s) for s in os.environ.get("SPLIT_SIZES", str(256 << 20) + " " + str(1 << 30)).split()]
    shares = [float(x) for x in os.environ.get("SPLIT_SHARES", "0 0.2 0.3 0.4 0.5 0.6 0.7 1").split()]
    maxb = max(sizes)
    buf = torch.empty(maxb, dtype=torch.uint8, device="cuda")
    comm.register(buf)
    nv = G.Nvls(maxb, local)
    sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
    unit = world * 1024
    for nbytes in sizes:
        count = nbytes // 4
        for x in shares:
            c_nv = int(count * x) // unit * unit
            c_pp = count - c_nv
            plan = G.Plan.from_topology(doc(world), c_pp, "f32") if c_pp else None
            ex = G.Executor(plan, comm, buf, stream=sb) if plan else None

            def once():
                ev = torch.cuda.Event()
                ev.record()
                sa.wait_event(ev)
                sb.wait_event(ev)
                if c_nv:
                    nv.allreduce(c_nv, "f32", stream=sa)
                if ex:
                    ex()
                torch.cuda.current_stream().wait_stream(sa)
                torch.cuda.current_stream().wait_stream(sb)

            G.fill_synthetic(buf, max(c_pp, 1), "f32", 11, rank, 0)
            G.fill_synthetic(nv.ptr, max(c_nv, 1), "f32", 11, rank, 0)
            for _ in range(5):
                once()
            torch.cuda.synchronize()
            dist.barrier()
            reps = 20
            evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
            for i in range(reps):
                if i % 8 == 0:   # keep the in-place sums finite
                    G.fill_synthetic(buf, max(c_pp, 1), "f32", 11, rank, 0)
                    G.fill_synthetic(nv.ptr, max(c_nv, 1), "f32", 11, rank, 0)
                evs[i][0].record()
                once()
                evs[i][1].record()
            torch.cuda.synchronize()
            ts = torch.tensor([a.elapsed_time(b) / 1e3 for a, b in evs], dtype=torch.float64, device="cuda")
            dist.all_reduce(ts, op=dist.ReduceOp.MAX)
            ts = ts.cpu().tolist()
            comm.async_error()
            nv.async_error()
            t = statistics.median(ts)
            if rank == 0:
                print(json.dumps({"tool": "nvls_p2p_split", "n": world, "bytes": nbytes, "nvls_share": x,
                                  "nvls_bytes": c_nv * 4, "p2p_bytes": c_pp * 4, "p2p_ctas": nsm - nv_ctas,
                                  "nvls_ctas": nv_ctas, "t_med": t, "t_min": min(ts),
                                  "busbw_med": nbytes / t * 2 * (world - 1) / world / 1e9}), flush=True)
    nv.destroy()
    comm.destroy()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
