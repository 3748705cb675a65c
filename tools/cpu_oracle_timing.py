#!/usr/bin/env python
"""SURVEY §8(d) CPU-oracle timing plan: the oracle (as it stands, never tuned) timed on this
host, pinned to ONE core, on the BASELINE.json configs — JSONL on stdout.

    python tools/cpu_oracle_timing.py [--core 0]

  C1  4 ranks, 1 MiB fp32 per rank, GenTree plan on the 2-level tree (Table 5 links):
      plan generation + step-by-step simulation + GenModel prediction
  C2  8 ranks, fp32, 16 MiB and 256 MiB per rank, GenTree plan (CPS) on one switch
  C4  8 ranks, bf16, 256 MiB per rank (bench.py's workload), GenTree plan (CPS)
Each row: seconds per AllReduce (plan build and simulation separately), the busbw the
oracle reaches, the CPU model and os.cpu_count(), and the core it was pinned to.
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

MIB = 1 << 20


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--core", type=int, default=0)
    ap.add_argument("--reps", type=int, default=2)
    a = ap.parse_args()
    os.sched_setaffinity(0, {a.core})          # one core (numpy's elementwise adds are serial)
    from oracle import genmodel as OG
    from oracle import gentree as GT
    from oracle import simulate as SM
    from oracle import topology as T
    from synth import generator as GEN
    host = {"cpu_model": cpu_model(), "cpu_count": os.cpu_count(), "pinned_core": a.core, "cores": 1,
            "python": platform.python_version()}
    nominal = {"alpha": 3e-6, "beta": 4 / 900e9, "epsilon": 0.0, "w_t": 9}
    comp = {"gamma": 0.0, "delta": 4 / 6.54e12}
    cases = [
        ("C1", T.two_level_doc([2, 2], T.TABLE5["root_sw"], T.TABLE5["middle_sw"], T.TABLE5["server"]), 4,
         MIB, "f32"),
        ("C2", T.single_switch_doc(8, nominal, comp), 8, 16 * MIB, "f32"),
        ("C2", T.single_switch_doc(8, nominal, comp), 8, 256 * MIB, "f32"),
        ("C4", T.single_switch_doc(8, nominal, comp), 8, 256 * MIB, "bf16"),
    ]
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
        for _ in range(a.reps):
            t0 = time.perf_counter()
            SM.simulate(plan, xs, dtype)
            sims.append(time.perf_counter() - t0)
        t_sim = min(sims)
        busbw = nbytes / t_sim * 2 * (n - 1) / n / 1e9
        print(json.dumps({"config": cfg, "ranks": n, "bytes_per_rank": nbytes, "dtype": dtype,
                          "plan_steps": len(plan.steps), "t_plan_s": t_plan, "t_predict_s": t_pred,
                          "t_simulate_s": t_sim, "t_simulate_all_s": sims, "oracle_busbw_gbs": busbw,
                          "genmodel_pred_s": pred, **host}), flush=True)
        del xs


if __name__ == "__main__":
    main()
