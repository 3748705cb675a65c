"""GPU probes for tuning and for the GenModel fit (C3-i local fan-in, Eq. 6).

    python tools/probe.py fanin            # local k-way reduce sweep, 150M-float vectors
    python tools/probe.py emu [--ctas ..]  # emulated R-rank AllReduce timing at one size
    python tools/probe.py copy             # torch copy bandwidth (sanity vs MEASURED_PEAKS)
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
    a = ap.parse_args()
    torch.cuda.set_device(0)
    {"fanin": fanin, "emu": emu, "copy": copy, "trace": trace, "hunt": hunt}[a.what](a)
