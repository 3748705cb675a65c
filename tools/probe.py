"""GPU probes for tuning and for the GenModel fit (C3-i local fan-in, Eq. 6).

    python tools/probe.py fanin            # local k-way reduce sweep, 150M-float vectors
    python tools/probe.py emu [--ctas ..]  # emulated R-rank AllReduce timing at one size
    python tools/probe.py copy             # torch copy bandwidth (sanity vs MEASURED_PEAKS)
    python tools/probe.py nvpull           # k-way reduce body over NVLink, one process, 2 GPUs
    python tools/probe.py nvflat           # the executor's bulk-copy body over NVLink (VMM split buffer)
Prints one JSON object per measurement.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2409_04202_b200 as G  # noqa: E402


def timeit(fn, reps=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / 1e3)
    ts.sort()
    return ts[len(ts) // 2], sum(ts) / len(ts), ts[0]


def fanin(args):
    count = args.count
    es = 4 if args.dtype == "f32" else 2
    bufs = [torch.empty(count * es, dtype=torch.uint8, device="cuda") for _ in range(args.kmax + 1)]
    for i, b in enumerate(bufs):
        G.fill_synthetic(b, count, args.dtype, 7, i, 0)
    for k in range(1, args.kmax + 1):
        med, mean, mn = timeit(lambda: G.local_reduce(bufs[:k], bufs[-1], count, args.dtype))
        S = count * es
        print(json.dumps({"probe": "fanin", "k": k, "dtype": args.dtype, "count": count, "t_med": med,
                          "t_mean": mean, "t_min": mn, "hbm_gbs": (k + 1) * S / med / 1e9,
                          "per_add_ms": med / max(k - 1, 1) * 1e3}), flush=True)


def emu(args):
    world, count, dtype = args.ranks, args.count, args.dtype
    params = G.params(3e-6, 1 / 900e9, 0.0, 1 / 6.54e12, 0.0, 9)
    plan = G.Plan.single_switch(world, count, dtype, params, args.force)
    comm = G.Comm.local(world, 0)
    for ctas in args.ctas:
        comm.set_ctas(ctas)
        stride = G.rank_stride_bytes(count, dtype)
        buf = torch.empty(world * stride, dtype=torch.uint8, device="cuda")
        for r in range(world):
            G.fill_synthetic(buf.data_ptr() + r * stride, count, dtype, 7, r, 0)
        med, mean, mn = timeit(lambda: G.allreduce_exec(plan, comm, buf), reps=args.reps)
        es = 4 if dtype == "f32" else 2
        S = count * es
        print(json.dumps({"probe": "emu", "ranks": world, "ctas": ctas, "plan": plan.report()[-1]["chosen"],
                          "dtype": dtype, "bytes": S, "pad": os.environ.get("AR_EMU_STRIDE_PAD", "0"),
                          "t_med": med, "t_min": mn, "busbw": S / med * 2 * (world - 1) / world / 1e9,
                          "hbm_gbs": 2 * world * S / med / 1e9}), flush=True)
        del buf


def trace(args):
    """Per-phase in-kernel timing (globaltimer) of one call, emulated ranks."""
    import numpy as np
    world, count, dtype = args.ranks, args.count, args.dtype
    plan = G.Plan.single_switch(world, count, dtype, G.params(3e-6, 1 / 900e9, 0.0, 1 / 6.54e12, 0.0, 9),
                                args.force)
    comm = G.Comm.local(world, 0)
    if args.ctas[0]:
        comm.set_ctas(args.ctas[0])
    stride = G.rank_stride_bytes(count, dtype)
    buf = torch.empty(world * stride, dtype=torch.uint8, device="cuda")
    ex = G.Executor(plan, comm, buf)
    for _ in range(5):
        ex()
    comm.set_trace(True)
    ex = G.Executor(plan, comm, buf)
    ex()
    tr = comm.read_trace().astype(np.int64)
    low = plan.lowering()
    nst = len(low["ranks"][0]["steps"])
    t0 = tr[:, :, 0].min()
    rows = []
    ctas = args.ctas[0] or tr.shape[1]
    for si in range(nst):
        w, o, n = (tr[:, :ctas, 1 + 3 * si] - t0, tr[:, :ctas, 2 + 3 * si] - t0, tr[:, :ctas, 3 + 3 * si] - t0)
        rows.append({"step": si, "slot": low["ranks"][0]["steps"][si]["slot"],
                     "wait_done_us": [float(np.median(w)) / 1e3, float(w.max()) / 1e3],
                     "ops_done_us": [float(np.median(o)) / 1e3, float(o.max()) / 1e3],
                     "notify_done_us": [float(np.median(n)) / 1e3, float(n.max()) / 1e3]})
    end = tr[:, :ctas, -1] - t0
    start = tr[:, :ctas, 0] - t0
    print(json.dumps({"probe": "trace", "plan": plan.report()[-1]["chosen"], "ranks": world, "count": count,
                      "start_spread_us": float(start.max()) / 1e3, "end_us": [float(np.median(end)) / 1e3,
                                                                             float(end.max()) / 1e3],
                      "steps": rows}), flush=True)
    # host cost of one call (no sync)
    import time
    comm.set_trace(False)
    ex = G.Executor(plan, comm, buf)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(200):
        ex()
    host = (time.perf_counter() - t) / 200
    torch.cuda.synchronize()
    print(json.dumps({"probe": "host_call_us", "us": host * 1e6}), flush=True)


def hunt(args):
    """Repeat calls with tracing until one is slow; dump where that call waited."""
    import time

    import numpy as np
    world, count, dtype = args.ranks, args.count, args.dtype
    plan = G.Plan.single_switch(world, count, dtype, G.params(3e-6, 1 / 900e9, 0.0, 1 / 6.54e12, 0.0, 9),
                                args.force)
    comm = G.Comm.local(world, 0)
    stride = G.rank_stride_bytes(count, dtype)
    buf = torch.empty(world * stride, dtype=torch.uint8, device="cuda")
    comm.set_trace(True)
    ex = G.Executor(plan, comm, buf)
    low = plan.lowering()
    for it in range(args.reps):
        t = time.perf_counter()
        ex()
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
        if dt > 0.05:
            tr = comm.read_trace().astype(np.int64)
            t0 = tr[:, :, 0].min()
            nst = [len(rk["steps"]) for rk in low["ranks"]]
            print(json.dumps({"probe": "hunt", "iter": it, "call_s": dt}), flush=True)
            for r in range(world):
                for c in range(tr.shape[1]):
                    row = [(tr[r, c, 1 + 3 * i] - t0) / 1e3 for i in range(nst[r])]
                    if max(row) > 10000:
                        slow = int(np.argmax(np.array(row) > 10000))
                        st = low["ranks"][r]["steps"][slow]
                        print(json.dumps({"rank": r, "cta": c, "step": slow, "slot": st["slot"],
                                          "waits": st["waits"], "wait_done_us": row}), flush=True)
                        break
            try:
                comm.async_error()
            except Exception as e:
                print(json.dumps({"error": str(e)}))
            return
    print(json.dumps({"probe": "hunt", "iters": args.reps, "result": "no slow call"}))


def copy(args):
    n = 1 << 30
    a = torch.empty(n, dtype=torch.bfloat16, device="cuda")
    b = torch.empty_like(a)
    med, mean, mn = timeit(lambda: b.copy_(a))
    print(json.dumps({"probe": "copy", "gbs": 2 * n * 2 / mn / 1e9, "gbs_med": 2 * n * 2 / med / 1e9}), flush=True)


def nvpull(args):
    """The k-way reduction body (local_reduce_kernel: 16-byte loads, fp32 accumulation, one
    read / one write per element) launched on GPU0 with operands in GPU1's HBM through peer
    access — one process and no flags, so ncu can replay it and read the NVLink counters
    (nvlrx__bytes / nvltx__bytes) that the multi-rank kernel cannot be profiled for.
    pull: out = local + remote (NVLink rx = S);  push: out(remote) = local + local (tx = S);
    pullpush: out(remote) = local + remote (rx = tx = S: the fused CPS step's pattern at N = 2)."""
    from cuda.bindings import runtime as rt
    assert torch.cuda.device_count() >= 2, "nvpull needs 2 GPUs"
    for d, p in ((0, 1), (1, 0)):
        torch.cuda.set_device(d)
        err, = rt.cudaDeviceEnablePeerAccess(p, 0)
        assert err in (rt.cudaError_t.cudaSuccess, rt.cudaError_t.cudaErrorPeerAccessAlreadyEnabled), err
    torch.cuda.set_device(0)
    count, es = args.count, 4
    S = count * es
    l0 = torch.empty(S, dtype=torch.uint8, device="cuda:0")
    l1 = torch.empty(S, dtype=torch.uint8, device="cuda:0")
    lo = torch.empty(S, dtype=torch.uint8, device="cuda:0")
    r0 = torch.empty(S, dtype=torch.uint8, device="cuda:1")
    ro = torch.empty(S, dtype=torch.uint8, device="cuda:1")
    for i, b in enumerate((l0, l1, r0)):
        with torch.cuda.device(b.device):
            G.fill_synthetic(b, count, "f32", 7, i, 0)
    torch.cuda.synchronize(1)
    cases = {"pull": ([l0, r0], lo, S, 0), "push": ([l0, l1], ro, 0, S), "pullpush": ([l0, r0], ro, S, S)}
    for name in args.cases:
        ins, out, rx, tx = cases[name]
        med, mean, mn = timeit(lambda: G.local_reduce(ins, out, count, "f32"), reps=args.reps)
        print(json.dumps({"probe": "nvpull", "case": name, "bytes_per_vector": S, "nvlink_rx_bytes": rx,
                          "nvlink_tx_bytes": tx, "t_med": med, "t_min": mn,
                          "nvlink_gbs_per_direction": max(rx, tx) / med / 1e9}), flush=True)


def _split_buffer(ranks_on, stride):
    """One contiguous virtual range of len(ranks_on) rank slots, slot r backed by physical HBM
    on GPU ranks_on[r] (CUDA VMM), readable and writable from both GPUs."""
    from cuda.bindings import driver as cu

    def ok(r):
        assert r[0] == cu.CUresult.CUDA_SUCCESS, r
        return r[1] if len(r) == 2 else r[1:]
    ok(cu.cuInit(0) + (None,))
    props = []
    for d in (0, 1):
        pr = cu.CUmemAllocationProp()
        pr.type = cu.CUmemAllocationType.CU_MEM_ALLOCATION_TYPE_PINNED
        pr.location.type = cu.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
        pr.location.id = d
        props.append(pr)
    gran = ok(cu.cuMemGetAllocationGranularity(
        props[0], cu.CUmemAllocationGranularity_flags.CU_MEM_ALLOC_GRANULARITY_RECOMMENDED))
    assert stride % gran == 0, (stride, gran)
    total = stride * len(ranks_on)
    va = ok(cu.cuMemAddressReserve(total, gran, 0, 0))
    for r, d in enumerate(ranks_on):
        h = ok(cu.cuMemCreate(stride, props[d], 0))
        ok(cu.cuMemMap(int(va) + r * stride, stride, 0, h, 0) + (None,))
    descs = []
    for d in (0, 1):
        ad = cu.CUmemAccessDesc()
        ad.location.type = cu.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
        ad.location.id = d
        ad.flags = cu.CUmemAccess_flags.CU_MEM_ACCESS_FLAGS_PROT_READWRITE
        descs.append(ad)
    ok(cu.cuMemSetAccess(va, total, descs, 2) + (None,))
    return int(va)


def nvflat(args):
    """The executor's production body (bulk-copy pipeline, ar_flat_kernel) with rank slots split
    across two GPUs: ranks 0..R/2-1 in GPU0's HBM, the rest in GPU1's, one VMM range, the kernel
    on GPU0.  Every element of a GPU1 rank is read over NVLink and its result written back over
    NVLink (rx = tx = R/2·S per call), the pull → add → push pattern of the fused CPS step; one
    process and no flags, so ncu can read nvlrx/nvltx for the real body."""
    assert torch.cuda.device_count() >= 2, "nvflat needs 2 GPUs"
    torch.cuda.set_device(0)
    world, count, dtype = args.ranks, args.count, args.dtype
    stride = G.rank_stride_bytes(count, dtype)
    on = [0] * (world // 2) + [1] * (world - world // 2)
    base = _split_buffer(on, stride)
    for r in range(world):
        with torch.cuda.device(on[r]):
            G.fill_synthetic(base + r * stride, count, dtype, 7, r, 0)
        torch.cuda.synchronize(on[r])
    params = G.params(3e-6, 1 / 900e9, 0.0, 1 / 6.54e12, 0.0, 9)
    plan = G.Plan.single_switch(world, count, dtype, params, "cps")
    comm = G.Comm.local(world, 0)
    S = count * (2 if dtype == "bf16" else 4)
    remote = sum(on) * S
    med, mean, mn = timeit(lambda: G.allreduce_exec(plan, comm, base), reps=args.reps)
    print(json.dumps({"probe": "nvflat", "kernel": comm.last_kernel(), "ranks": world, "ranks_on_gpu1": sum(on),
                      "dtype": dtype, "bytes_per_rank": S, "nvlink_rx_bytes": remote, "nvlink_tx_bytes": remote,
                      "t_med": med, "t_min": mn, "nvlink_gbs_per_direction": remote / med / 1e9,
                      "busbw_equiv": S * 2 * (world - 1) / world / med / 1e9}), flush=True)
    comm.destroy()


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("what")
    ap.add_argument("--count", type=int, default=150_000_000)
    ap.add_argument("--dtype", default="f32")
    ap.add_argument("--kmax", type=int, default=8)
    ap.add_argument("--ranks", type=int, default=8)
    ap.add_argument("--ctas", type=int, nargs="*", default=[0])
    ap.add_argument("--force", default=None)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--cases", nargs="*", default=["pull", "push", "pullpush"])
    a = ap.parse_args()
    torch.cuda.set_device(0)
    {"fanin": fanin, "emu": emu, "copy": copy, "trace": trace, "hunt": hunt, "nvpull": nvpull, "nvflat": nvflat}[a.what](a)
