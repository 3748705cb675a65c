"""Worker for the multi-level execution test (SURVEY §8(f) NEXT #3, config C5's "8 ranks per
GPU" across GPUs): one process per GPU, each hosting R consecutive ranks
(ar_comm_create_multi).  The GenTree plan of a two-level tree whose leaves are the R ranks of
one GPU moves its leaf-level data inside HBM and its root level over NVLink; forced flat
kinds (CPS, Ring) mix local and remote peers inside every step.  Every hosted rank's buffer
must be bit-exact against the CPU oracle.  Exit code 0 = all cases bit-exact.

    torchrun --nproc-per-node N tests/mp_hybrid_worker.py [R]
"""
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
from tests.gpu_util import assert_bits_equal  # noqa: E402


def main():
    proc = int(os.environ["RANK"])
    nproc = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", proc))
    R = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    world = nproc * R
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    comm = G.Comm.create_multi(proc, nproc, R, local)
    nvl = {"alpha": 1e-5, "beta": 4.0 / 770e9, "epsilon": 0.0, "w_t": 9}       # root: NVLink
    hbm = {"alpha": 3e-6, "beta": 4.0 / 3000e9, "epsilon": 0.0, "w_t": 64}     # leaves: HBM
    server = {"gamma": 0.0, "delta": 4.0 / 6.5e12}
    tree = T.two_level_doc([R] * nproc, nvl, hbm, server)
    flat = T.single_switch_doc(world, nvl, server)
    cases = [(tree, None), (flat, "cps"), (flat, "ring")]
    seed = GEN.config_seed(5)
    failures = 0
    keep = []
    for dtype in ("f32", "bf16"):
        es = 4 if dtype == "f32" else 2
        for count in (world * 1024 + 7, 1 << 20):
            stride = G.rank_stride_bytes(count, dtype)
            buf = torch.zeros(stride * R, dtype=torch.uint8, device="cuda")
            keep.append(buf)
            comm.register(buf)
            for ci, (doc, force) in enumerate(cases):
                for i in range(R):
                    G.fill_synthetic(buf.data_ptr() + i * stride, count, dtype, seed, proc * R + i, 0)
                plan = G.Plan.from_topology(doc, count, dtype, None, force)
                oplan, _ = GT.gentree(T.parse_topology(doc), count, es, force=force)
                assert plan.to_json() == OP.plan_to_json(oplan, dtype)
                torch.cuda.synchronize()
                dist.barrier()
                G.allreduce_exec(plan, comm, buf)
                G.allreduce_exec(plan, comm, buf, op="avg")
                torch.cuda.synchronize()
                comm.async_error()
                xs = GEN.generate_all(seed, world, count, dtype)
                want = SM.simulate(oplan, SM.simulate(oplan, xs, dtype), dtype, op="avg")
                host = buf.cpu().numpy()
                for i in range(R):
                    got = host[i * stride: i * stride + count * es].view(np.float32 if dtype == "f32" else np.uint16)
                    try:
                        assert_bits_equal(got, want[proc * R + i], dtype,
                                          f"rank {proc * R + i} {dtype} count={count} case={ci}")
                    except AssertionError as e:
                        print(e, flush=True)
                        failures += 1
                dist.barrier()
    dist.barrier()
    comm.destroy()
    dist.destroy_process_group()
    if proc == 0:
        print(f"hybrid_worker nproc={nproc} R={R}: {'OK' if failures == 0 else f'{failures} FAILURES'}", flush=True)
    sys.exit(1 if failures else 0)


if __name__ == "__main__":
    main()
