#!/usr/bin/env python
"""Benchmark of the GenTree-plan AllReduce hot path (arXiv 2409.04202) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Metric (BASELINE.json): AllReduce busbw (GB/s) = S/t * 2(R-1)/R for S bytes per rank and R
ranks (nccl-tests convention); plus the GenModel prediction error of the executed plan.

Workload (config C4 of BASELINE.json, "bf16, 256 MB buffer, GenTree plan through one
executor"):
  * N = 1 (default): R = 8 ranks emulated on one B200 ("8 ranks/GPU", config C5's mode) —
    one cooperative launch of the step-table kernel moves every rank's 256 MiB through HBM;
  * N > 1 (torchrun, one process per GPU): R = N ranks, peer buffers mapped with CUDA IPC,
    the kernel pulls/pushes over NVLink 5 (NVSwitch).  NCCL all_reduce on the same buffer is
    timed alongside for comparison.
A "step" is one full AllReduce (all SURVEY §8(a) rows) of the 256 MiB buffer.  Inputs are
synthetic gradient-shaped data from the seeded generator (DESIGN.md input recipe), resident
in HBM; the working set (>= 256 MiB per GPU) exceeds the 126 MB L2, so no flush is needed.

Only the cpu_baseline leg and --impl reference execute the CPU oracle (oracle/).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

MIB = 1 << 20


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--dtype", choices=["bf16", "f32"], default="bf16")
    ap.add_argument("--mib", type=int, default=256, help="MiB per rank")
    ap.add_argument("--ranks", type=int, default=8, help="emulated ranks when --gpus 1")
    ap.add_argument("--force", default=None, help="plan kind instead of GenTree (cps, ring, rhd, rb, hcps:a,b)")
    ap.add_argument("--ctas", type=int, default=0)
    ap.add_argument("--cpu-timing-plan", action="store_true",
                    help="run SURVEY §8(d)'s CPU-oracle timing plan (C1, C2, C4 data simulation; C1/C5 plan "
                         "generation, oracle and library) pinned to one core, print JSONL, exit")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-nccl", action="store_true")
    ap.add_argument("--no-nvls", action="store_true")
    ap.add_argument("--cpu-sample-mib", type=float, default=64.0, help="oracle sample per rank (MiB)")
    return ap.parse_args()


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return pk.get("hbm_gbs", 6650.0), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


NVLINK_PEAK_GBS = 770.0   # measured peer copy per direction (B200_PROFILING.md)


NOMINAL = {"alpha": 3e-6, "beta": 1 / 900e9, "gamma": 0.0, "delta": 1 / 6.54e12, "epsilon": 0.0, "w_t": 9}


def fitted_params(emulated=False):
    """B200 GenModel fit committed under profiles/ (tools/fit_report.py --install): NVLink
    ranks (genmodel_params.json) or emulated ranks sharing one GPU's HBM."""
    path = os.path.join(ROOT, "profiles", "genmodel_params_emulated.json" if emulated else "genmodel_params.json")
    if os.path.exists(path):
        with open(path) as f:
            return json.load(f)
    return None


def model_params(world=None, emulated=False):
    """GenModel parameters (per byte) used to select the plan.  The B200 fit is used only for
    worlds it was fitted on (its incast threshold w_t and slope ε are not identifiable beyond
    the largest measured n); otherwise nominal B200 values (α 3 µs,
    β 1/900 GB/s, δ 1/6.54 TB/s, no incast below 9)."""
    if emulated:
        # emulated ranks share one GPU's HBM: their fit (reading A6e, used for the prediction
        # below) has no link term, and a topology link needs β > 0 — plan selection therefore
        # uses the nominal B200 values; both give CPS (δ-optimal, fewest steps) on one switch
        return dict(NOMINAL), "nominal (emulated ranks; the shared-HBM fit has no link term)"
    p = fitted_params(emulated)
    if p is not None and (world is None or world <= p.get("n_max_fit", 0)):
        return p, "fitted (%s)" % p.get("source", "profiles")
    return dict(NOMINAL), "nominal (fit covers n <= %s)" % (p.get("n_max_fit") if p else "-")


def single_switch_doc(world, p):
    from_float = 4.0
    nodes = [{"id": "sw", "kind": "switch", "parent": None, "uplink": None}]
    for i in range(world):
        nodes.append({"id": f"s{i}", "kind": "server", "parent": "sw",
                      "uplink": {"alpha": p["alpha"], "beta": p["beta"] * from_float,
                                 "epsilon": p["epsilon"] * from_float, "w_t": int(p["w_t"])},
                      "compute": {"gamma": p["gamma"] * from_float, "delta": p["delta"] * from_float}})
    return json.dumps({"nodes": nodes})


class ClockSampler:
    """SM clocks + throttle reasons sampled DURING the timed region: an NVML thread polls every
    ~2 ms between start() and stop() (the timed region of a 256 MiB step lasts only ~10-15 ms,
    shorter than nvidia-smi's 100 ms period); nvidia-smi is the fallback."""
    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4}

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.err = None

    def start(self):
        import threading
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
        except Exception as e:   # no NVML: nvidia-smi one-shot queries in the thread
            h, self.max_mhz, self.err = None, None, str(e)[:80]
        self.stop_flag = False

        def poll():
            while not self.stop_flag:
                try:
                    if h is not None:
                        sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                        rs = getattr(pynvml, "nvmlDeviceGetCurrentClocksEventReasons",
                                     getattr(pynvml, "nvmlDeviceGetCurrentClocksThrottleReasons", None))(h)
                        pw = pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0
                    else:
                        out = subprocess.run(["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm",
                                              "--format=csv,noheader,nounits"], capture_output=True, text=True).stdout
                        sm, mx = (int(x) for x in out.strip().split(","))
                        self.max_mhz, rs, pw = mx, 0, 0.0
                    self.rows.append((sm, rs, pw))
                except Exception as e:
                    self.err = str(e)[:80]
                time.sleep(0.002)

        self.t = threading.Thread(target=poll, daemon=True)
        self.t.start()
        t0 = time.time()
        while not self.rows and time.time() - t0 < 3.0:   # sampling is live before timing starts
            time.sleep(0.001)
        self.rows.clear()

    def stop(self):
        self.stop_flag = True
        self.t.join(timeout=5)
        rows = self.rows
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["no samples: " + str(self.err)]}
        reasons = sorted({k for _, rs, _ in rows for k, bit in self.REASONS.items() if rs & bit})
        return {"sm_mhz": statistics.median(r[0] for r in rows), "sm_max_mhz": self.max_mhz, "reasons": reasons,
                "samples": len(rows), "power_w_max": round(max(r[2] for r in rows), 1), "source": "nvml, 2 ms"}


def busbw(bytes_per_rank, ranks, seconds):
    return bytes_per_rank / seconds * 2 * (ranks - 1) / ranks / 1e9


# ----------------------------------------------------------------------------- CPU oracle legs

def oracle_sample(world, dtype, count, force, p):
    """The oracle's plan and seeded inputs for a bounded sample (built once, outside the timing)."""
    from oracle import genmodel as OG
    from oracle import gentree as GT
    from oracle import topology as T
    from synth import generator as GEN
    t = T.parse_topology(single_switch_doc(world, p))
    op = OG.Params(p["alpha"], p["beta"], p["gamma"], p["delta"], p["epsilon"], int(p["w_t"]))
    plan, _ = GT.gentree(t, count, 2 if dtype == "bf16" else 4, params=op, force=force)
    return plan, GEN.generate_all(GEN.config_seed(4), world, count, dtype)


def oracle_step_time(sample, dtype):
    """One step of the oracle (as it stands): its step-by-step simulation of the plan on the
    sample (simulate copies its inputs, so the sample can be reused)."""
    from oracle import simulate as SM
    plan, xs = sample
    t0 = time.perf_counter()
    SM.simulate(plan, xs, dtype)
    return time.perf_counter() - t0


def oracle_sample_time(world, dtype, count, force, p):
    """The oracle (as it stands) simulating the same plan kind on a bounded sample."""
    return oracle_step_time(oracle_sample(world, dtype, count, force, p), dtype)


def host_info():
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"cpu_model": model, "cpu_count": os.cpu_count()}


def pinned_one_core(fn):
    """Run fn() with this process pinned to one core (the oracle's numpy adds are serial;
    pinning makes `cores: 1` a fact, not an assumption), then restore the affinity."""
    old = os.sched_getaffinity(0)
    core = min(old)
    os.sched_setaffinity(0, {core})
    try:
        return fn(), core
    finally:
        os.sched_setaffinity(0, old)


def cpu_baseline(world, dtype, sample_mib, force, p):
    es = 2 if dtype == "bf16" else 4
    count = int(sample_mib * MIB) // es
    secs, core = pinned_one_core(lambda: oracle_sample_time(world, dtype, count, force, p))
    return {"value": round(busbw(count * es, world, secs), 4), "unit": "GB/s", "cores": 1, "kind": "oracle",
            "pinned_core": core, **host_info(),
            "sample": f"{world} ranks x {count} {dtype} elements ({sample_mib:g} MiB/rank), same plan kind, "
                      f"numpy single-threaded step-by-step simulation pinned to one core; {secs:.2f} s per "
                      f"AllReduce (the full 256 MiB workload and the C1/C2/C4 plan: "
                      f"profiles/round2/cpu_oracle_timing.jsonl)"}


def arm_config(args, n, world, chosen, p_src):
    """The `config` both arms report (the reference arm times the oracle on the same one)."""
    es = 2 if args.dtype == "bf16" else 4
    dbytes = (world if n == 1 else 1) * (args.mib * MIB // es) * es
    return {"workload": (f"C4: GenTree-plan AllReduce, {args.dtype}, {args.mib} MiB per rank, "
                         + (f"{world} ranks emulated on 1 GPU (8 ranks/GPU, C5 mode)" if n == 1
                            else f"{n} ranks = {n} GPUs over NVLink/NVSwitch")),
            "ranks": world, "bytes_per_rank": args.mib * MIB, "plan": chosen,
            "plan_source": args.force or f"GenTree with {p_src} GenModel params",
            "l2": f"working set {dbytes / MIB:.0f} MiB per GPU > 126 MB L2 (no flush needed)",
            "ctas_per_rank": args.ctas or "auto"}


def run_reference(args):
    """--impl reference: the CPU oracle timed as the reference arm (rank 0 only)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    n = args.gpus
    world = args.ranks if n == 1 else n
    p, p_src = model_params(world, emulated=n == 1)
    es = 2 if args.dtype == "bf16" else 4
    # every one of the --warmup W + --steps K steps simulates the whole plan on a bounded sample;
    # the sample shrinks as K + W grows so the run stays within a few minutes (1.4 s per step at
    # 64 MiB per rank x 8 ranks on the GPU box's host: K + W <= 16 keeps the full sample)
    calls = max(1, args.steps) + max(0, args.warmup)
    sample_mib = args.cpu_sample_mib * min(1.0, 16.0 / calls)
    count = max(world * 64, int(sample_mib * MIB) // es // 256 * 256)
    from oracle import gentree as GT
    from oracle import topology as T
    from oracle import genmodel as OG
    op = OG.Params(p["alpha"], p["beta"], p["gamma"], p["delta"], p["epsilon"], int(p["w_t"]))
    _, reps = GT.gentree(T.parse_topology(single_switch_doc(world, p)), args.mib * MIB // es, es, params=op,
                         force=args.force)
    chosen = reps[-1].chosen
    sample = oracle_sample(world, args.dtype, count, args.force, p)
    def run():
        for _ in range(max(0, args.warmup)):
            oracle_step_time(sample, args.dtype)
        return [oracle_step_time(sample, args.dtype) for _ in range(max(1, args.steps))]
    times, core = pinned_one_core(run)
    t = sum(times) / len(times)
    v = busbw(count * es, world, t)
    line = {"impl": "reference", "metric": "allreduce_busbw", "value": round(v, 4), "unit": "GB/s",
            "n_gpus": n, "steps": len(times), "warmup": max(0, args.warmup), "ms_per_step": round(t * 1e3, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": args.dtype,
            "data": "synthetic",
            "config": arm_config(args, n, world, chosen, p_src),
            "note": (f"the reference arm is the CPU oracle (no reference implementation exists); it runs the "
                     f"same {len(times)} timed steps after {max(0, args.warmup)} warm-up as the GPU arm, each on a "
                     f"bounded sample ({count * es / MIB:g} MiB per rank) so the run ends in minutes"),
            "cpu_baseline": {"value": round(v, 4), "unit": "GB/s", "cores": 1, "kind": "oracle",
                             "pinned_core": core, **host_info(),
                             "sample": f"each step: the oracle's step-by-step simulation of the same plan on a "
                                       f"bounded sample, {world} ranks x {count} {args.dtype} elements "
                                       f"({count * es / MIB:g} MiB/rank), numpy single-threaded"},
            "e2e": {"value": round(v, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    emit(line)


# ----------------------------------------------------------------------------- GPU arm

def cpu_timing_plan(core=0, reps=2):
    """SURVEY §8(d) / BASELINE.md §6 CPU-oracle timing plan (the cpu_baseline leg, widened): the
    oracle as it stands, pinned to ONE core, on the BASELINE.json configs — JSONL on stdout.

      C1  4 ranks, 1 MiB fp32 per rank, GenTree plan on the 2-level tree (Table 5 links): plan
          generation + step-by-step simulation + GenModel prediction
      C2  8 ranks, fp32, 16 MiB and 256 MiB per rank, GenTree plan (CPS) on one switch
      C4  8 ranks, bf16, 256 MiB per rank (bench.py's workload), GenTree plan (CPS)
      plan generation (host µs): the oracle's GenTree and the library's gentree_plan, and the
          GenModel evaluation of the plan (oracle predict_plan, library genmodel_predict_executed),
          on C1 and on C5 (64 ranks = 8 x 8, 2-level tree) at 1e7 / 3.2e7 / 1e8 / 3.2e8 floats
    Input generation is outside every timing."""
    import platform
    os.sched_setaffinity(0, {core})          # one core (numpy's elementwise adds are serial)
    from oracle import gentree as GT
    from oracle import simulate as SM
    from oracle import topology as T
    from synth import generator as GEN
    import paper_2409_04202_b200 as G
    host = {**host_info(), "pinned_core": core, "cores": 1, "python": platform.python_version()}
    nominal = {"alpha": 3e-6, "beta": 4 / 900e9, "epsilon": 0.0, "w_t": 9}
    comp = {"gamma": 0.0, "delta": 4 / 6.54e12}
    c1 = T.two_level_doc([2, 2], T.TABLE5["root_sw"], T.TABLE5["middle_sw"], T.TABLE5["server"])
    cases = [("C1", c1, 4, MIB, "f32"),
             ("C2", T.single_switch_doc(8, nominal, comp), 8, 16 * MIB, "f32"),
             ("C2", T.single_switch_doc(8, nominal, comp), 8, 256 * MIB, "f32"),
             ("C4", T.single_switch_doc(8, nominal, comp), 8, 256 * MIB, "bf16")]
    for cfg, doc, n, nbytes, dtype in cases:
        es = 4 if dtype == "f32" else 2
        count = nbytes // es
        topo = T.parse_topology(doc)
        t0 = time.perf_counter()
        plan, _ = GT.gentree(topo, count, es)
        t_plan = time.perf_counter() - t0
        t0 = time.perf_counter()
        pred = GT.predict_plan(topo, plan, es)["total"]
        t_pred = time.perf_counter() - t0
        xs = GEN.generate_all(GEN.config_seed(4), n, count, dtype)
        sims = []
        for _ in range(reps):
            t0 = time.perf_counter()
            SM.simulate(plan, xs, dtype)
            sims.append(time.perf_counter() - t0)
        t_sim = min(sims)
        emit({"config": cfg, "ranks": n, "bytes_per_rank": nbytes, "dtype": dtype, "plan_steps": len(plan.steps),
              "t_plan_s": t_plan, "t_predict_s": t_pred, "t_simulate_s": t_sim, "t_simulate_all_s": sims,
              "oracle_busbw_gbs": busbw(nbytes, n, t_sim), "genmodel_pred_s": pred, **host})
        del xs
    c5 = T.two_level_doc([8] * 8, T.TABLE5["root_sw"], T.TABLE5["middle_sw"], T.TABLE5["server"])
    for cfg, doc, n in (("C1", c1, 4), ("C5", c5, 64)):
        topo = T.parse_topology(doc)
        for floats in (10 ** 7, 32 * 10 ** 6, 10 ** 8, 32 * 10 ** 7):
            row = {"config": cfg + "-plan", "ranks": n, "floats": floats}
            for side in ("oracle", "library"):
                ts, tp = [], []
                for _ in range(max(1, reps)):
                    t0 = time.perf_counter()
                    if side == "oracle":
                        plan, rep = GT.gentree(topo, floats, 4)
                    else:
                        lp = G.Plan.from_topology(doc, floats, "f32")
                    ts.append(time.perf_counter() - t0)
                    t0 = time.perf_counter()
                    if side == "oracle":
                        GT.predict_plan(topo, plan, 4)
                    else:
                        lp.predict()
                    tp.append(time.perf_counter() - t0)
                row[f"{side}_gentree_us"] = min(ts) * 1e6
                row[f"{side}_predict_us"] = min(tp) * 1e6
            row["chosen"] = [r["chosen"] for r in lp.report()]
            emit({**row, **host})


_JSON_OUT = None


def emit(line):
    """The one JSON line on stdout (everything else — e.g. NCCL's C-level version banner — was
    moved to stderr by keep_stdout_for_json)."""
    out = _JSON_OUT or sys.stdout
    out.write(json.dumps(line) + "\n")
    out.flush()


def keep_stdout_for_json():
    """Reserve the process's stdout for the JSON line: keep a duplicate of fd 1 for emit() and
    point fd 1 at stderr, so libraries printing to stdout (NCCL prints its version there) cannot
    add lines the driver would have to skip."""
    global _JSON_OUT
    sys.stdout.flush()
    _JSON_OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)


def main():
    args = parse_args()
    keep_stdout_for_json()
    if args.cpu_timing_plan:
        cpu_timing_plan()
        return
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    import paper_2409_04202_b200 as G

    n = args.gpus
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if n > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        assert dist.get_world_size() == n
    else:
        torch.cuda.set_device(0)
    dev = torch.cuda.current_device()
    es = 2 if args.dtype == "bf16" else 4
    nbytes = args.mib * MIB
    count = nbytes // es
    world = args.ranks if n == 1 else n
    p, p_src = model_params(world, emulated=n == 1)
    plan = G.Plan.from_topology(single_switch_doc(world, p), count, args.dtype, None, args.force)
    chosen = plan.report()[-1]["chosen"]
    # a6: GenModel prediction of the executed plan with the B200 fit of this machine kind
    # (N = 1: all ranks share one GPU's HBM — reading A6e, genmodel_predict_executed_shared;
    # N > 1: reading A6x).  Both fits use CPS rows only and never the bench's own point (the
    # emulated fit uses 2..7 ranks, the NVLink fit leaves out the 256 MiB rows), so the
    # prediction below is held out; the fit's validation summary is carried into the line.
    fp = fitted_params(emulated=n == 1) or NOMINAL
    pred_src = ("fitted " + fp["source"]) if "source" in fp else "nominal"
    if chosen != "cps" and "step_table_row" in fp:
        # a multi-step plan runs as dependent steps on the step-table kernel: that path's row
        fp = {**fp["step_table_row"], "validation": fp.get("validation")}
        pred_src += " (step-table kernel row)"
    gp = G.params(fp["alpha"], fp["beta"], fp["gamma"], fp["delta"], fp["epsilon"], int(fp["w_t"]))
    pred = (plan.predict_executed_shared(gp) if n == 1 else plan.predict_executed(gp))["total"]
    seed = 0x240904202 ^ 4
    stream = torch.cuda.current_stream()

    if n == 1:
        comm = G.Comm.local(world, dev)
        stride = G.rank_stride_bytes(count, args.dtype)
        buf = torch.empty(world * stride, dtype=torch.uint8, device="cuda")
        for r in range(world):
            G.fill_synthetic(buf.data_ptr() + r * stride, count, args.dtype, seed, r, 0)
        dbytes = world * stride
    else:
        comm = G.Comm.create(rank, n, dev)
        if args.ctas:   # agreed at registration (ar_comm_open_peers checks it)
            comm.set_ctas(args.ctas)
        buf = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
        G.fill_synthetic(buf, count, args.dtype, seed, rank, 0)
        comm.register(buf)
        dbytes = nbytes
    if args.ctas and n == 1:
        comm.set_ctas(args.ctas)
    torch.cuda.synchronize()

    def barrier():
        if dist is not None:
            dist.barrier()

    def refill():   # keep magnitudes bounded (in-place sums grow x world per call)
        if n == 1:
            for r in range(world):
                G.fill_synthetic(buf.data_ptr() + r * stride, count, args.dtype, seed, r, 0)
        else:
            G.fill_synthetic(buf, count, args.dtype, seed, rank, 0)

    for _ in range(args.warmup):
        G.allreduce_exec(plan, comm, buf)
    refill()
    torch.cuda.synchronize()
    comm.async_error()
    barrier()
    clocks = ClockSampler(dev)
    clocks.start()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    torch.cuda.synchronize()
    barrier()
    ev[0].record(stream)
    for i in range(args.steps):
        G.allreduce_exec(plan, comm, buf)
        ev[i + 1].record(stream)
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    comm.async_error()
    launches = args.steps * comm.last_launch_count()
    per_step = [ev[i].elapsed_time(ev[i + 1]) / 1e3 for i in range(args.steps)]
    total = ev[0].elapsed_time(ev[-1]) / 1e3
    if dist is not None:
        tt = torch.tensor([total], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        total = float(tt.item())
    t_step = total / args.steps
    value = busbw(nbytes, world, t_step)

    # roofline of the dominant (only) kernel: launch duration = the step's event interval
    kern_t = statistics.mean(per_step)
    if n == 1:
        hbm_peak, hbm_src = load_peaks()
        # the plan's HBM bytes, all ranks sharing one HBM (reading A6e's D: every op's k reads and
        # one write per destination): 2·R·S for CPS (every rank buffer read once, written once),
        # (5R − 6)·S for Ring, …
        alg_bytes = int(plan.predict_executed_shared(G.params(0.0, 1e-30, 0.0, 1.0, 0.0, 9))["memory"])
        achieved = alg_bytes / kern_t / 1e9
        roof = {"kernel": comm.last_kernel(), "bound": "hbm", "achieved": round(achieved, 1), "peak": hbm_peak,
                "unit": "GB/s",
                "frac": round(achieved / hbm_peak, 4), "traffic": None,
                "algorithmic_bytes_per_launch": alg_bytes, "peak_source": hbm_src}
        # DRAM traffic per launch from the committed ncu --set full capture of this config
        try:
            with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
                tr = json.load(f).get(f"emulated:r{world}:{args.dtype}:{nbytes}:{chosen}")
            if tr and not args.ctas and tr.get("kernel", "ar_exec_kernel") == comm.last_kernel():
                roof["traffic"] = tr["traffic_bytes_per_launch"]
                roof["traffic_source"] = tr["source"]
        except (OSError, ValueError):
            pass
    else:
        wire = 2 * (n - 1) * nbytes / n          # Eq. 2: bytes per direction per GPU
        achieved = wire / kern_t / 1e9
        roof = {"kernel": comm.last_kernel(), "bound": "nvlink", "achieved": round(achieved, 1),
                "peak": NVLINK_PEAK_GBS, "unit": "GB/s",
                "frac": round(achieved / NVLINK_PEAK_GBS, 4), "traffic": None,
                "algorithmic_bytes_per_launch": int(wire),
                "peak_source": "measured peer copy per direction (B200_PROFILING.md)",
                "nominal_peak": 900.0, "frac_nominal": round(achieved / 900.0, 4),
                # NVLink wire bytes per user byte of the pull -> add -> push step, from ncu's
                # nvltx/nvlrx counters (profiles/README.md: writes 1.269, read responses 1.148,
                # read requests 0.221 per byte read): (1.269 + 1.148 + 0.221) / 2 = 1.319 per
                # direction, so 900 GB/s of wire carries at most 682 GB/s of user data
                "wire_per_user_byte": 1.319, "wire_user_ceiling": round(900.0 / 1.319, 1),
                "frac_wire_ceiling": round(achieved / (900.0 / 1.319), 4)}

    # NVLS in-switch reduction (NEXT #1 plan kind, not a GenTree candidate), same size (N > 1)
    nvls = None
    if dist is not None and not args.no_nvls:
        try:
            nv = G.Nvls(nbytes, dev)
            G.fill_synthetic(nv.ptr, count, args.dtype, seed, rank, 0)
            for _ in range(args.warmup):
                nv.allreduce(count, args.dtype)
            torch.cuda.synchronize()
            barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(args.steps):
                nv.allreduce(count, args.dtype)
            e1.record(stream)
            torch.cuda.synchronize()
            nv.async_error()
            tt = torch.tensor([e0.elapsed_time(e1) / 1e3 / args.steps], dtype=torch.float64, device="cuda")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            nvls = {"busbw": round(busbw(nbytes, n, float(tt.item())), 2),
                    "ms_per_step": round(float(tt.item()) * 1e3, 4),
                    "note": "multimem.ld_reduce/st through the NVSwitch; switch-chosen summation order"}
            npath = os.path.join(ROOT, "profiles", "genmodel_params_nvls.json")
            if os.path.exists(npath):   # GenModel's plan-vs-NVLS choice (NEXT #1 row, reading NV1)
                nj = json.load(open(npath))
                c = plan.choose_nvls(gp, G.params(alpha=nj["alpha"], beta=nj["beta"]))
                nvls["genmodel"] = {"use_nvls": c["use_nvls"], "t_plan_ms": round(c["t_plan"] * 1e3, 4),
                                    "t_nvls_ms": round(c["t_nvls"] * 1e3, 4), "params": nj["source"]}
            nv.destroy()
        except Exception as e:   # multicast unavailable: report, do not fail the bench
            nvls = {"unavailable": str(e)[:200]}

    # NCCL on the same data size (N > 1), three variants (the config's Ring
    # comparator, NCCL's default choice, and NVLS disabled).  NCCL reads NCCL_ALGO when a
    # communicator is initialised, so each variant is its own process group, created and
    # initialised (first collective) while NCCL_ALGO is set; "^NVLS,NVLSTree" excludes the
    # NVSwitch algorithms without touching the process-wide NCCL_NVLS_ENABLE parameter.
    nccl = None
    if dist is not None and not args.no_nccl:
        t = torch.empty(count, dtype=torch.bfloat16 if args.dtype == "bf16" else torch.float32, device="cuda")
        t.normal_()
        nccl = {"version": ".".join(map(str, torch.cuda.nccl.version()))}
        for key, algo in (("default", None), ("ring", "Ring"), ("nvls_off", "^NVLS,NVLSTree")):
            old = os.environ.get("NCCL_ALGO")
            try:
                if algo is not None:
                    os.environ["NCCL_ALGO"] = algo
                grp = dist.new_group(list(range(n)), backend="nccl") if algo is not None else None
                for _ in range(max(1, args.warmup)):
                    dist.all_reduce(t, group=grp)
                torch.cuda.synchronize()
            finally:
                if old is None:
                    os.environ.pop("NCCL_ALGO", None)
                else:
                    os.environ["NCCL_ALGO"] = old
            barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(args.steps):
                dist.all_reduce(t, group=grp)
            e1.record(stream)
            torch.cuda.synchronize()
            tt = torch.tensor([e0.elapsed_time(e1) / 1e3 / args.steps], dtype=torch.float64, device="cuda")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            nccl[key] = {"busbw": round(busbw(nbytes, n, float(tt.item())), 2),
                         "ms_per_step": round(float(tt.item()) * 1e3, 4), "NCCL_ALGO": algo or "unset"}
        del t

    # end to end through the C-ABI from pinned host memory
    e2e = None
    if not args.no_e2e:
        host = torch.empty(dbytes, dtype=torch.uint8, pin_memory=True)
        host.copy_(buf)
        k = max(1, min(args.steps, 5))
        G.allreduce_exec_host(plan, comm, buf, host.data_ptr(), count, args.dtype)
        torch.cuda.synchronize()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(k):
            G.allreduce_exec_host(plan, comm, buf, host.data_ptr(), count, args.dtype)
        e1.record(stream)
        torch.cuda.synchronize()
        te = e0.elapsed_time(e1) / 1e3 / k
        if dist is not None:
            tt = torch.tensor([te], dtype=torch.float64, device="cuda")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            te = float(tt.item())
        e2e = {"value": round(busbw(nbytes, world, te), 4), "unit": "GB/s",
               "h2d_bytes_per_step": dbytes * (n if n > 1 else 1), "d2h_bytes_per_step": dbytes * (n if n > 1 else 1),
               "ms_per_step": round(te * 1e3, 3), "steps": k}
        comm.async_error()

    if rank != 0:
        if dist is not None:
            dist.barrier()
            dist.destroy_process_group()
        return
    cpu = None
    if not args.no_cpu_baseline:
        cpu = cpu_baseline(world, args.dtype, args.cpu_sample_mib, args.force, p)
    line = {
        "metric": "allreduce_busbw", "value": round(value, 2), "unit": "GB/s", "n_gpus": n,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(t_step * 1e3, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": args.dtype,
        "data": "synthetic",
        "config": arm_config(args, n, world, chosen, p_src),
        "roofline": roof,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": launches,
        "gpu_launches_note": f"one launch of {comm.last_kernel()} per step (per process)",
        "clocks": clk,
        "genmodel": {"predicted_ms": round(pred * 1e3, 4), "measured_ms": round(t_step * 1e3, 4),
                     "pred_err": round(abs(pred - t_step) / t_step, 4), "params": pred_src,
                     "bench_point_in_fit": False,
                     "model": ("GenModel of the executed steps, all ranks sharing one HBM (reading A6e)" if n == 1
                               else "GenModel of the executed (fused, full-duplex) steps (reading A6x)"),
                     "validation_held_out": fp.get("validation")},
        # busbw (nccl-tests) is a per-rank figure: the bus bandwidth every rank sustains, which a
        # bandwidth-optimal AllReduce keeps flat in the rank count — so `value` is not expected
        # to grow with N.  The job-wide figure is the sum over the ranks.
        "value_semantics": "busbw per rank (nccl-tests: S/t x 2(R-1)/R); not additive over GPUs",
        "aggregate_busbw": {"value": round(value * world, 2), "unit": "GB/s",
                            "note": f"sum over the {world} ranks ({'all on one GPU' if n == 1 else 'one per GPU'})"},
        "busbw_per_step_min_median_max": [round(busbw(nbytes, world, max(per_step)), 2),
                                          round(busbw(nbytes, world, statistics.median(per_step)), 2),
                                          round(busbw(nbytes, world, min(per_step)), 2)],
    }
    if nccl:
        line["nccl"] = nccl
        line["vs_nccl"] = {k: round(value / v["busbw"], 3) for k, v in nccl.items() if isinstance(v, dict)}
    if nvls:
        line["nvls"] = nvls
        g = nvls.get("genmodel")
        if g is not None and "busbw" in nvls and args.dtype == "f32" and not args.force:
            # GenTree with the NVLS kind as a candidate (reading NV1, fp32 only: bit-exact there):
            # GenModel's pick and the busbw this run measured for the picked path
            line["gentree_incl_nvls"] = {"pick": "nvls" if g["use_nvls"] else chosen,
                                         "busbw": nvls["busbw"] if g["use_nvls"] else round(value, 2),
                                         "unit": "GB/s"}
    emit(line)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
