"""Small single-GPU workload for compute-sanitizer (memcheck / racecheck / synccheck):
every plan kind on 4 and 8 emulated ranks, fp32 and bf16, ragged sizes, SUM and AVG, through
the step-table kernel, the flat kernel and local_reduce; results checked against the oracle.

    compute-sanitizer --tool memcheck python tests/sanitize_probe.py

(compute-sanitizer is closed on the round-1 GPU pool; the probe alone runs every path once
with bounded waits and oracle checks.)
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2409_04202_b200 as G  # noqa: E402
from oracle import gentree as GT  # noqa: E402
from oracle import simulate as SM  # noqa: E402
from oracle import topology as T  # noqa: E402
from synth import generator as GEN  # noqa: E402


def main():
    torch.cuda.set_device(0)
    bad = 0
    for world, kinds in ((4, [None, "ring", "rhd", "rb", "hcps:2,2"]), (8, [None, "ring", "hcps:4,2"])):
        doc = T.single_switch_doc(world, {"alpha": 3e-6, "beta": 4 / 900e9, "epsilon": 0.0, "w_t": 9},
                                  {"gamma": 0.0, "delta": 4 / 6.54e12})
        comm = G.Comm.local(world, 0)
        for dtype in ("f32", "bf16"):
            es = 4 if dtype == "f32" else 2
            count = 4099 * world + 3
            stride = G.rank_stride_bytes(count, dtype)
            for kind in kinds:
                for op in ("sum", "avg"):
                    buf = torch.zeros(world * stride, dtype=torch.uint8, device="cuda")
                    for r in range(world):
                        G.fill_synthetic(buf.data_ptr() + r * stride, count, dtype, 5, r, 0)
                    plan = G.Plan.from_topology(doc, count, dtype, None, kind)
                    G.allreduce_exec(plan, comm, buf, op=op)
                    torch.cuda.synchronize()
                    comm.async_error()
                    oplan, _ = GT.gentree(T.parse_topology(doc), count, es, force=kind)
                    want = SM.simulate(oplan, GEN.generate_all(5, world, count, dtype), dtype, op=op)
                    host = buf.cpu().numpy()
                    for r in range(world):
                        got = host[r * stride: r * stride + count * es].view(np.uint32 if es == 4 else np.uint16)
                        w = want[r].view(np.uint32) if es == 4 else want[r]
                        bad += int(not np.array_equal(got, w))
        comm.destroy()
    ins = [torch.zeros(4096 * 4, dtype=torch.uint8, device="cuda") for _ in range(3)]
    out = torch.zeros(4096 * 4, dtype=torch.uint8, device="cuda")
    G.local_reduce(ins, out, 4096, "f32")
    torch.cuda.synchronize()
    print(f"sanitize_probe: {'OK' if bad == 0 else f'{bad} mismatches'}", flush=True)
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
