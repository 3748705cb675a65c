#!/usr/bin/env python
"""GenModel measurement harness (configs C2, C3, C4) — JSONL on stdout.

Multi-GPU (torchrun, one process per GPU; rank 0 prints):
    torchrun --nproc-per-node N tools/harness.py sweep  [--dtype f32] [--plans "gentree;cps;ring"]
        C2: busbw vs size 64 KiB..1 GiB for our plans and NCCL all_reduce on the same box
    torchrun --nproc-per-node N tools/harness.py cps
        C3-iii: CPS AllReduce times at this N for the §3.4 fit (run for N = 2..max)
Single GPU, emulated ranks (all ranks of a plan in one launch, "8 ranks/GPU"):
    python tools/harness.py emu-sweep --ranks 8
    python tools/harness.py emu-cps   --max-ranks 8
    python tools/harness.py fanin                           (C3-i, Eq. 6 local fan-in)

Timing modes (--timing, comma list):
  eager — CUDA events around every call, 5 warm-up calls, inputs refilled from the seeded
          generator every 8 calls outside the events; includes host launch overhead
  graph — `reps` calls captured in one CUDA graph (ours: the kernel has no per-call host
          argument; NCCL: graph-captured all_reduce), replayed once, time / reps: device time
Multi-GPU times are the max over ranks.  Mean and median are reported (the paper uses the
mean; reading Q20).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2409_04202_b200 as G  # noqa: E402

NOMINAL = {"alpha": 3e-6, "beta": 1 / 900e9, "gamma": 0.0, "delta": 1 / 6.54e12, "epsilon": 0.0, "w_t": 9}
SIZES = [1 << k for k in range(16, 31)]       # 64 KiB .. 1 GiB


def tree_doc(groups, mid_link, leaf_link, compute):
    """Topology document (SPEC format): root switch -> len(groups) middle switches -> servers."""
    nodes = [{"id": "R", "kind": "switch", "parent": None, "uplink": None}]
    k = 0
    for g, cnt in enumerate(groups):
        nodes.append({"id": f"M{g}", "kind": "switch", "parent": "R", "uplink": dict(mid_link)})
        for _ in range(cnt):
            nodes.append({"id": f"s{k}", "kind": "server", "parent": f"M{g}", "uplink": dict(leaf_link),
                          "compute": dict(compute)})
            k += 1
    return json.dumps({"nodes": nodes})


def flat_doc(world, link, compute):
    nodes = [{"id": "sw", "kind": "switch", "parent": None, "uplink": None}]
    nodes += [{"id": f"s{i}", "kind": "server", "parent": "sw", "uplink": dict(link), "compute": dict(compute)}
              for i in range(world)]
    return json.dumps({"nodes": nodes})


def doc(world, p=NOMINAL):
    nodes = [{"id": "sw", "kind": "switch", "parent": None, "uplink": None}]
    for i in range(world):
        nodes.append({"id": f"s{i}", "kind": "server", "parent": "sw",
                      "uplink": {"alpha": p["alpha"], "beta": p["beta"] * 4, "epsilon": p["epsilon"] * 4,
                                 "w_t": int(p["w_t"])},
                      "compute": {"gamma": p["gamma"] * 4, "delta": p["delta"] * 4}})
    return json.dumps({"nodes": nodes})


def fitted(name):
    """A GenModel fit committed under profiles/ (tools/fit_report.py --install)."""
    with open(os.path.join(ROOT, "profiles", name)) as f:
        return json.load(f)


def kinds_for(world, plans):
    out = []
    for k in plans.split(";"):
        if k == "rhd" and world & (world - 1):
            continue
        if k.startswith("hcps:"):
            prod = 1
            for x in k[5:].split(","):
                prod *= int(x)
            if prod != world:
                continue
        out.append(k)
    return out


def reps_for(nbytes):
    return 50 if nbytes <= 64 << 20 else 20


class Timer:
    def __init__(self, dist):
        self.dist = dist

    def _sync(self):
        torch.cuda.synchronize()
        if self.dist:
            self.dist.barrier()

    def _max(self, ts):
        t = torch.tensor(ts, dtype=torch.float64, device="cuda")
        if self.dist:
            self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return t.cpu().tolist()

    def run(self, make, reps, refill, mode):
        """make() -> callable issuing one AllReduce on the current stream."""
        if mode == "eager":
            fn = make()
            for _ in range(5):
                fn()
            refill()
            self._sync()
            evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
            for i in range(reps):
                if i and i % 8 == 0:
                    refill()
                evs[i][0].record()
                fn()
                evs[i][1].record()
            torch.cuda.synchronize()
            ts = self._max([a.elapsed_time(b) / 1e3 for a, b in evs])
            return {"t_mean": statistics.mean(ts), "t_med": statistics.median(ts), "t_min": min(ts),
                    "reps": reps, "timing": "eager"}
        # graph
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            fn = make()
            for _ in range(3):
                fn()
        torch.cuda.current_stream().wait_stream(s)
        self._sync()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            fn = make()
            for _ in range(reps):
                fn()
        self._sync()
        g.replay()
        refill()
        self._sync()
        ts = []
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) / 1e3 / reps)
            refill()
            self._sync()
        ts = self._max(ts)
        del g
        return {"t_mean": statistics.mean(ts), "t_med": statistics.median(ts), "t_min": min(ts), "reps": reps,
                "timing": "graph"}


def busbw(nbytes, n, t):
    return nbytes / t * 2 * (n - 1) / n / 1e9


def emit(rank, row):
    if rank == 0:
        print(json.dumps(row), flush=True)


def multi(args):
    import torch.distributed as dist
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    comm = G.Comm.create(rank, world, local)
    if args.ctas:
        comm.set_ctas(args.ctas)
    es = 4 if args.dtype == "f32" else 2
    tdt = torch.float32 if args.dtype == "f32" else torch.bfloat16
    sizes = args.sizes or SIZES
    if args.mode == "cps":
        sizes = [1 << 20, 1 << 22, 1 << 24, 1 << 26, 1 << 28]
    buf = torch.empty(max(sizes), dtype=torch.uint8, device="cuda")
    timer = Timer(dist)
    modes = args.timing.split(",")
    nvls_buf = [None]
    for nbytes in sizes:
        count = nbytes // es
        view = buf[:nbytes]
        comm.register(view)

        def refill():
            G.fill_synthetic(view, count, args.dtype, 11, rank, 0)

        plans = ["cps"] if args.mode == "cps" else ([] if args.plans == "none" else kinds_for(world, args.plans))
        for k in plans:
            if k == "nvls":     # in-switch reduction (NEXT #1), its own multicast-bound buffer
                if nvls_buf[0] is None:
                    nvls_buf[0] = G.Nvls(max(sizes), local)
                nv = nvls_buf[0]

                def nv_refill():
                    G.fill_synthetic(nv.ptr, count, args.dtype, 11, rank, 0)

                for mode in modes:
                    r = timer.run(lambda: (lambda: nv.allreduce(count, args.dtype)), reps_for(nbytes), nv_refill,
                                  mode)
                    emit(rank, {"mode": args.mode, "impl": "ours", "plan": "nvls", "chosen": "nvls", "n": world,
                                "bytes": nbytes, "dtype": args.dtype, **r,
                                "busbw_med": busbw(nbytes, world, r["t_med"]),
                                "busbw_mean": busbw(nbytes, world, r["t_mean"])})
                nv.async_error()
                continue
            if k == "gentree+nvls":
                # GenTree with the NVLS kind as a candidate (gentree_plan_nvls, reading NV1) under
                # the committed B200 fits; an NVLS pick runs through allreduce_exec on the
                # attached multicast buffer, a plan pick on the IPC-registered one
                fp, fn = fitted("genmodel_params.json"), fitted("genmodel_params_nvls.json")
                fo = fitted("genmodel_fit_oneshot_graph.json")
                fl = fitted("genmodel_fit_ll128_graph.json")
                fl = fl.get("per_n", {}).get(str(world), fl)   # the row fitted at this rank count
                paths = comm.paths()   # the path the executor takes decides the plan-side row
                plan = G.Plan.from_topology_nvls(doc(world), count, args.dtype,
                                                 G.params(fp["alpha"], fp["beta"], fp["gamma"], fp["delta"],
                                                          fp["epsilon"], int(fp["w_t"])),
                                                 G.params(alpha=fn["alpha"], beta=fn["beta"]),
                                                 G.params(alpha=fo["alpha"], beta=fo["beta"]), paths["oneshot_max"],
                                                 G.params(alpha=fl["alpha"], beta=fl["beta"]), paths["ll128_max"],
                                                 paths["ll128_min"])
                target, fill_fn = view, refill
                if plan.switch_reduce:
                    if nvls_buf[0] is None:
                        nvls_buf[0] = G.Nvls(max(sizes), local)
                    nv = nvls_buf[0]
                    comm.attach_nvls(nv)
                    target = nv.ptr

                    def fill_fn():
                        G.fill_synthetic(nv.ptr, count, args.dtype, 11, rank, 0)
                for mode in modes:
                    r = timer.run(lambda: G.Executor(plan, comm, target), reps_for(nbytes), fill_fn, mode)
                    emit(rank, {"mode": args.mode, "impl": "ours", "plan": k, "chosen": plan.report()[-1]["chosen"],
                                "n": world, "bytes": nbytes, "dtype": args.dtype, "ctas": args.ctas or "auto", **r,
                                "busbw_med": busbw(nbytes, world, r["t_med"]),
                                "busbw_mean": busbw(nbytes, world, r["t_mean"])})
                continue
            plan = G.Plan.from_topology(doc(world), count, args.dtype, None, None if k == "gentree" else k)
            for mode in modes:
                r = timer.run(lambda: G.Executor(plan, comm, view), reps_for(nbytes), refill, mode)
                emit(rank, {"mode": args.mode, "impl": "ours", "plan": k, "chosen": plan.report()[-1]["chosen"],
                            "n": world, "bytes": nbytes, "dtype": args.dtype, "ctas": args.ctas or "auto", **r,
                            "busbw_med": busbw(nbytes, world, r["t_med"]),
                            "busbw_mean": busbw(nbytes, world, r["t_mean"])})
        if args.mode == "sweep" and not args.no_nccl:
            t = view.view(tdt)
            for mode in modes:
                r = timer.run(lambda: (lambda: dist.all_reduce(t)), reps_for(nbytes), refill, mode)
                label = os.environ.get("NCCL_ALGO") or ("nvls_off" if os.environ.get("NCCL_NVLS_ENABLE") == "0"
                                                        else "default")
                emit(rank, {"mode": "sweep", "impl": "nccl", "plan": label,
                            "n": world, "bytes": nbytes, "dtype": args.dtype, **r,
                            "busbw_med": busbw(nbytes, world, r["t_med"]),
                            "busbw_mean": busbw(nbytes, world, r["t_mean"]),
                            "nccl_version": ".".join(map(str, torch.cuda.nccl.version()))})
    comm.async_error()
    dist.barrier()
    comm.destroy()
    dist.destroy_process_group()


def probe_plan(kind, n, x, count, dtype):
    """Data-movement plans for the C3-ii fan-in tests (reading Q22) in canonical
    plan JSON: ONE step in which the x ranks 0..x-1 exchange concurrently (the incast pattern:
    every receiver has x-1 simultaneous senders).  Block b of the `count`-element buffer has
    the plan's block size (n blocks).

    x-to-x push  : every rank r < x writes its block r into every other rank of the group
    x-to-x pull  : every rank r < x reduces block r from all x ranks of the group (CPS's RS
                   step: one op reading the x-1 peers concurrently)
    x-to-1 push  : ranks 1..x-1 write their block into rank 0
    x-to-1 pull  : rank 0 reduces block 0 from ranks 0..x-1 (one receiver, x-1 senders)
    The pull variants are the reduce kernel's access pattern, the push ones the AllGather's."""
    size = lambda b: count // n + (1 if b < count % n else 0)
    red, tr = [], []
    if kind == "push":
        tr = [{"block": r, "dst": d, "size": size(r), "src": r} for r in range(x) for d in range(x) if d != r]
        label, phase = f"push{x}to{x}", "ag"
    elif kind == "pull":
        red = [{"block": r, "fan_in": x, "inputs": list(range(x)), "server": r} for r in range(x)]
        label, phase = f"pull{x}to{x}", "rs"
    elif kind == "push1":
        tr = [{"block": r, "dst": 0, "size": size(r), "src": r} for r in range(1, x)]
        label, phase = f"push{x}to1", "ag"
    elif kind == "pull1":
        red = [{"block": 0, "fan_in": x, "inputs": list(range(x)), "server": 0}]
        label, phase = f"pull{x}to1", "rs"
    else:
        raise ValueError(kind)
    return json.dumps({"count": count, "dtype": dtype, "n": n,
                       "steps": [{"label": label, "phase": phase, "reduces": red, "transfers": tr}]})


def p2p(args):
    """C3-ii: x-to-x full-mesh and x-to-1 fan-in over NVLink, push and pull, for
    x = 2..N.  Every receiver gets a fixed total of S bytes (--sizes, default the paper's
    20 M floats = 80 MB) from its x-1 senders; without incast T(x) = α + Sβ is flat in
    x, a rise beyond w_t is the incast slope ε."""
    import torch.distributed as dist
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    comm = G.Comm.create(rank, world, local)
    es = 4 if args.dtype == "f32" else 2
    sizes = args.sizes or [80_000_000, 1 << 28]
    # receiver total S = (x-1) blocks of count/world elements -> count = world*S/((x-1)*es)
    cap = max(world * S // es * es for S in sizes) + 4096
    buf = torch.empty(cap, dtype=torch.uint8, device="cuda")
    timer = Timer(dist)
    for S in sizes:
        for x in range(2, world + 1):
            count = world * S // ((x - 1) * es)
            view = buf[: count * es]
            comm.register(view)
            for kind in ("push", "pull", "push1", "pull1"):
                if kind in ("push1", "pull1") and x == 2:
                    continue   # same as x-to-x at x = 2
                plan = G.Plan.from_json(probe_plan(kind, world, x, count, args.dtype))
                r = timer.run(lambda: G.Executor(plan, comm, view, movement=True), 20, lambda: None, "graph")
                recv = (x - 1) * (count // world) * es
                emit(rank, {"mode": "p2p", "kind": kind, "pattern": {"push": "x-to-x push", "pull": "x-to-x pull",
                                                                      "push1": "x-to-1 push", "pull1": "x-to-1 pull"}[kind],
                            "n": world, "x": x, "recv_bytes": recv, **r,
                            "gbs_per_receiver": recv / r["t_med"] / 1e9})
    comm.async_error()
    dist.barrier()
    comm.destroy()
    dist.destroy_process_group()


def nccl_algo(args):
    """Log the algorithm/protocol NCCL picks for all_reduce at each size (run with
    NCCL_DEBUG=INFO NCCL_DEBUG_SUBSYS=TUNING NCCL_DEBUG_FILE=...): one call per size."""
    import torch.distributed as dist
    rank = int(os.environ["RANK"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    tdt = torch.float32 if args.dtype == "f32" else torch.bfloat16
    es = 4 if args.dtype == "f32" else 2
    for nbytes in args.sizes or SIZES:
        t = torch.ones(nbytes // es, dtype=tdt, device="cuda")
        dist.all_reduce(t)
        torch.cuda.synchronize()
        emit(rank, {"mode": "nccl-algo", "bytes": nbytes, "dtype": args.dtype,
                    "NCCL_ALGO": os.environ.get("NCCL_ALGO", "unset"),
                    "NCCL_NVLS_ENABLE": os.environ.get("NCCL_NVLS_ENABLE", "unset")})
    dist.barrier()
    dist.destroy_process_group()


def fanin_ag(args):
    """C3-iv ("concurrent memory traffic"): the Eq. 6 local fan-in reduce of k
    vectors on GPU 0, alone and while GPU 1 streams an AllGather-like copy into
    GPU 0's HBM over NVLink (copy engine, peer writes), to test whether the memory term stays
    additive (the model sums the terms of a step).  One process, two GPUs."""
    import torch.cuda as tc
    assert tc.device_count() >= 2, "needs 2 GPUs"
    count = args.count
    es = 4 if args.dtype == "f32" else 2
    torch.cuda.set_device(0)
    bufs = [torch.empty(count * es, dtype=torch.uint8, device="cuda:0") for _ in range(args.kmax + 1)]
    for i, b in enumerate(bufs):
        G.fill_synthetic(b, count, args.dtype, 7, i, 0)
    land = torch.empty(1 << 30, dtype=torch.uint8, device="cuda:0")          # AG destination on GPU 0
    src = torch.empty(1 << 30, dtype=torch.uint8, device="cuda:1")
    src.fill_(1)
    s1 = torch.cuda.Stream(device="cuda:1")
    torch.cuda.synchronize(0)
    torch.cuda.synchronize(1)

    def time_reduce(k, reps=20):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(reps + 1)]
        ev[0].record()
        for i in range(reps):
            G.local_reduce(bufs[:k], bufs[-1], count, args.dtype)
            ev[i + 1].record()
        torch.cuda.synchronize(0)
        ts = [ev[i].elapsed_time(ev[i + 1]) / 1e3 for i in range(reps)]
        return statistics.median(ts), statistics.mean(ts)

    def ag_rate(ncopies):
        with torch.cuda.stream(s1):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s1)
            for _ in range(ncopies):
                land.copy_(src, non_blocking=True)
            e1.record(s1)
        return e0, e1

    for _ in range(3):
        G.local_reduce(bufs[:2], bufs[-1], count, args.dtype)
    ag_rate(2)                       # warm-up: the first peer copy sets up the mapping
    torch.cuda.synchronize(1)
    e0, e1 = ag_rate(8)
    torch.cuda.synchronize(1)
    ag_alone = 8 * (1 << 30) / (e0.elapsed_time(e1) / 1e3) / 1e9
    for k in range(2, args.kmax + 1):
        t_alone, m_alone = time_reduce(k)
        reps = 20
        # enough AG traffic queued to cover the whole timed region
        ncopies = int(1.5 * reps * t_alone * ag_alone * 1e9 / (1 << 30)) + 4
        e0, e1 = ag_rate(ncopies)
        time.sleep(0.002)
        t_conc, m_conc = time_reduce(k, reps)
        torch.cuda.synchronize(1)
        ag_gbs = ncopies * (1 << 30) / (e0.elapsed_time(e1) / 1e3) / 1e9
        emit(0, {"mode": "fanin-ag", "k": k, "count": count, "dtype": args.dtype,
                 "t_med_alone": t_alone, "t_med_with_ag": t_conc, "t_mean_alone": m_alone, "t_mean_with_ag": m_conc,
                 "hbm_bytes": (k + 1) * count * es,
                 "hbm_gbs_alone": (k + 1) * count * es / t_alone / 1e9,
                 "hbm_gbs_with_ag": (k + 1) * count * es / t_conc / 1e9,
                 "ag_gbs_alone": ag_alone, "ag_gbs_during": ag_gbs,
                 "ag_covers_timed_region": bool(ncopies * (1 << 30) / (ag_gbs * 1e9) >= reps * t_conc)})


def mtrace(args):
    """Per-phase in-kernel timeline of one call on N GPUs (rank 0's CTAs; globaltimer ns)."""
    import numpy as np
    import torch.distributed as dist
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    comm = G.Comm.create(rank, world, local)
    if args.ctas:
        comm.set_ctas(args.ctas)
    es = 4 if args.dtype == "f32" else 2
    for nbytes in args.sizes or [1 << 20]:
        count = nbytes // es
        buf = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
        comm.register(buf)
        for k in kinds_for(world, args.plans):
            plan = G.Plan.from_topology(doc(world), count, args.dtype, None, None if k == "gentree" else k)
            ex = G.Executor(plan, comm, buf)
            for _ in range(5):
                ex()
            torch.cuda.synchronize()
            comm.set_trace(True)
            ex = G.Executor(plan, comm, buf)
            dist.barrier()
            for _ in range(args.steady):    # back-to-back calls: the trace keeps the last one
                ex()
            ex()
            tr = comm.read_trace().astype(np.int64)[0]
            comm.set_trace(False)
            if args.steady:
                # every rank's phases of the same (last) call on one clock: %globaltimer
                allt = [None] * world
                dist.all_gather_object(allt, tr.tolist())
                if rank == 0:
                    g0 = min(min(x[0] for x in a_ if x[-1] > 0) for a_ in allt)
                    for q, a_ in enumerate(allt):
                        a_ = np.array(a_)
                        u = [c for c in range(a_.shape[0]) if a_[c, -1] > 0]
                        med = lambda j: round(float(np.median([(a_[c, j] - g0) / 1e3 for c in u])), 2)
                        nst2 = len(plan.lowering()["ranks"][q]["steps"])
                        spread = lambda j: [round(float(f([(a_[c, j] - g0) / 1e3 for c in u])), 2)
                                            for f in (np.min, np.median, np.max)]
                        print(json.dumps({"mode": "mtrace-steady", "rank": q, "bytes": nbytes, "start": med(0),
                                          "steps": [[med(1 + 3 * i), med(2 + 3 * i), med(3 + 3 * i)]
                                                    for i in range(nst2)], "end": med(-1),
                                          "cta_spread_min_med_max": {
                                              "start": spread(0), "end": spread(-1),
                                              "steps": [[spread(1 + 3 * i), spread(2 + 3 * i), spread(3 + 3 * i)]
                                                        for i in range(nst2)]}}), flush=True)
            nst = len(plan.lowering()["ranks"][rank]["steps"])
            t0 = tr[:, 0].min()
            C = comm_ctas = tr.shape[0]
            used = [c for c in range(C) if tr[c, -1] > 0]
            rows = []
            for si in range(nst):
                ph = [np.median([(tr[c, 1 + 3 * si + j] - t0) / 1e3 for c in used]) for j in range(3)]
                rows.append([si] + [round(x, 2) for x in ph])
            end = np.median([(tr[c, -1] - t0) / 1e3 for c in used])
            emit(rank, {"mode": "mtrace", "plan": k, "n": world, "bytes": nbytes, "ctas": len(used),
                        "steps_wait_ops_notify_us": rows, "end_us": round(float(end), 2)})
    comm.async_error()
    dist.barrier()
    comm.destroy()
    dist.destroy_process_group()


def emu(args):
    torch.cuda.set_device(0)
    es = 4 if args.dtype == "f32" else 2
    timer = Timer(None)
    modes = args.timing.split(",")
    worlds = list(range(2, args.max_ranks + 1)) if args.mode == "emu-cps" else [args.ranks]
    sizes = args.sizes or ([1 << 20, 1 << 22, 1 << 24, 1 << 26, 1 << 28] if args.mode == "emu-cps"
                           else [s for s in SIZES if s * args.ranks <= (8 << 30)])
    for world in worlds:
        comm = G.Comm.local(world, 0)
        plans = ["cps"] if args.mode == "emu-cps" else kinds_for(world, args.plans)
        for nbytes in sizes:
            count = nbytes // es
            stride = G.rank_stride_bytes(count, args.dtype)
            buf = torch.empty(world * stride, dtype=torch.uint8, device="cuda")

            def refill():
                for r in range(world):
                    G.fill_synthetic(buf.data_ptr() + r * stride, count, args.dtype, 11, r, 0)

            for k in plans:
                plan = G.Plan.from_topology(doc(world), count, args.dtype, None, None if k == "gentree" else k)
                for mode in modes:
                    r = timer.run(lambda: G.Executor(plan, comm, buf), reps_for(nbytes), refill, mode)
                    emit(0, {"mode": args.mode, "impl": "ours", "plan": k, "chosen": plan.report()[-1]["chosen"],
                             "n": world, "bytes": nbytes, "dtype": args.dtype, "emulated": True, **r,
                             "busbw_med": busbw(nbytes, world, r["t_med"]),
                             "hbm_gbs_med": 2 * world * nbytes / r["t_med"] / 1e9})
            del buf
        comm.async_error()
        comm.destroy()


def hybrid(args):
    """NEXT #3: R = --ranks ranks per GPU across the torchrun processes (ar_comm_create_multi);
    plans: GenTree on the two-level tree (leaves = one GPU's ranks, root over NVLink) and
    forced flat kinds over all N*R ranks."""
    import torch.distributed as dist
    proc = int(os.environ["RANK"])
    nproc = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", proc))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    R = args.ranks
    world = nproc * R
    comm = G.Comm.create_multi(proc, nproc, R, local)
    es = 4 if args.dtype == "f32" else 2
    nvl = {"alpha": 1e-5, "beta": 4.0 / 770e9, "epsilon": 0.0, "w_t": 9}
    hbm = {"alpha": 3e-6, "beta": 4.0 / 3000e9, "epsilon": 0.0, "w_t": 64}
    server = {"gamma": 0.0, "delta": 4.0 / 6.5e12}
    tree = tree_doc([R] * nproc, nvl, hbm, server)
    flat = flat_doc(world, nvl, server)
    timer = Timer(dist)
    modes = args.timing.split(",")
    sizes = args.sizes or [1 << 20, 1 << 22, 1 << 24, 1 << 26, 1 << 28]
    for nbytes in sizes:
        count = nbytes // es
        stride = G.rank_stride_bytes(count, args.dtype)
        buf = torch.empty(R * stride, dtype=torch.uint8, device="cuda")
        comm.register(buf)

        def refill():
            for i in range(R):
                G.fill_synthetic(buf.data_ptr() + i * stride, count, args.dtype, 11, proc * R + i, 0)

        for name, d, force in (("tree", tree, None), ("cps", flat, "cps"), ("ring", flat, "ring")):
            if name not in args.plans.split(";"):
                continue
            plan = G.Plan.from_topology(d, count, args.dtype, None, force)
            for mode in modes:
                r = timer.run(lambda: G.Executor(plan, comm, buf), reps_for(nbytes), refill, mode)
                emit(proc, {"mode": "hybrid", "impl": "ours", "plan": name, "chosen": plan.report()[-1]["chosen"],
                            "n": world, "gpus": nproc, "ranks_per_gpu": R, "bytes": nbytes, "dtype": args.dtype,
                            **r, "busbw_med": busbw(nbytes, world, r["t_med"])})
        del buf
    comm.async_error()
    dist.barrier()
    comm.destroy()
    dist.destroy_process_group()


def fanin(args):
    """C3-i: k-way local reduce of 150M-float vectors, Eq. 6."""
    torch.cuda.set_device(0)
    count = args.count
    es = 4 if args.dtype == "f32" else 2
    bufs = [torch.empty(count * es, dtype=torch.uint8, device="cuda") for _ in range(args.kmax + 1)]
    for i, b in enumerate(bufs):
        G.fill_synthetic(b, count, args.dtype, 7, i, 0)
    timer = Timer(None)
    for k in range(2, args.kmax + 1):
        r = timer.run(lambda: (lambda: G.local_reduce(bufs[:k], bufs[-1], count, args.dtype)), 20,
                      lambda: None, "eager")
        emit(0, {"mode": "fanin", "k": k, "count": count, "dtype": args.dtype, **r,
                 "t_per_add_med": r["t_med"] / (k - 1),
                 "hbm_gbs_med": (k + 1) * count * es / r["t_med"] / 1e9})


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("mode", choices=["sweep", "cps", "emu-sweep", "emu-cps", "fanin", "fanin-ag", "p2p", "mtrace",
                                     "hybrid", "nccl-algo"])
    ap.add_argument("--dtype", default="f32")
    ap.add_argument("--plans", default="gentree;cps;ring;rhd;rb;hcps:2,2;hcps:4,2;hcps:2,4;hcps:2,2,2",
                    help="';'-separated plan kinds")
    ap.add_argument("--timing", default="eager,graph")
    ap.add_argument("--ranks", type=int, default=8)
    ap.add_argument("--max-ranks", type=int, default=8)
    ap.add_argument("--sizes", type=int, nargs="*", default=None)
    ap.add_argument("--count", type=int, default=150_000_000)
    ap.add_argument("--kmax", type=int, default=8)
    ap.add_argument("--no-nccl", action="store_true")
    ap.add_argument("--ctas", type=int, default=0, help="CTAs per rank (0 = the comm's default)")
    ap.add_argument("--steady", type=int, default=0, help="mtrace: back-to-back calls before the traced one")
    a = ap.parse_args()
    if a.mode in ("sweep", "cps"):
        multi(a)
    elif a.mode == "mtrace":
        mtrace(a)
    elif a.mode == "hybrid":
        hybrid(a)
    elif a.mode == "p2p":
        p2p(a)
    elif a.mode == "fanin":
        fanin(a)
    elif a.mode == "fanin-ag":
        fanin_ag(a)
    elif a.mode == "nccl-algo":
        nccl_algo(a)
    else:
        emu(a)
