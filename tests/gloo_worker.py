"""Worker of tests/test_gloo_multiproc.py (CPU, gloo): builds plans and their device step
tables through the C-ABI and all-gathers them; rank 0 writes the gathered objects to
argv[2] as JSON."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch.distributed as dist  # noqa: E402

import paper_2409_04202_b200 as G  # noqa: E402
from oracle import topology as T  # noqa: E402


def main():
    world_of_plan, out = int(sys.argv[1]), sys.argv[2]
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    doc = T.single_switch_doc(world_of_plan, {"alpha": 3e-6, "beta": 4 / 900e9, "epsilon": 0.0, "w_t": 9},
                              {"gamma": 0.0, "delta": 4 / 6.54e12})
    res = []
    kinds = [None, "ring", "rhd", "rb"] + (["hcps:2,2"] if world_of_plan == 4 else [])
    for force in kinds:
        plan = G.Plan.from_topology(doc, 12345, "bf16", None, force)
        allv = [None] * world
        dist.all_gather_object(allv, {"plan": plan.to_json(), "low": plan.lowering()})
        res.append(allv)
    dist.barrier()
    dist.destroy_process_group()
    if rank == 0:
        with open(out, "w") as f:
            json.dump(res, f)


if __name__ == "__main__":
    main()
