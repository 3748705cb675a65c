"""Worker for the NVLS tests (torchrun, one process per GPU).  Integer-valued inputs must give
the exact sum (any summation order is exact for them); fp32 gradient-shaped inputs must be
BIT-EXACT against the oracle's correctly rounded sum (reading NV2: the switch rounds the exact
sum once); bf16 gradient-shaped inputs must be within the north star's norm-wise bound of the
float64 sum (1e-2; reading Q21 — the switch's bf16 rounding is not RNE at ties); every rank
must hold identical bits (the switch multicasts one result)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2409_04202_b200 as G  # noqa: E402
from oracle import exactsum as XS  # noqa: E402
from oracle import simulate as SM  # noqa: E402
from synth import generator as GEN  # noqa: E402


def main():
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    nbytes = 64 << 20
    nv = G.Nvls(nbytes, local)
    seed = GEN.config_seed(3)
    failures = 0
    for dtype in ("f32", "bf16"):
        es = 4 if dtype == "f32" else 2
        for count in (world * 16 // es, world * 4096, (nbytes // es) // (world * 8) * world * 8):
            for mode, mid in (("integer", 1), ("gradient", 0)):
                G.fill_synthetic(nv.ptr, count, dtype, seed, rank, mid)
                torch.cuda.synchronize()
                dist.barrier()
                nv.allreduce(count, dtype)
                torch.cuda.synchronize()
                nv.async_error()
                got = nv.tensor[: count * es].cpu().numpy().view(np.float32 if dtype == "f32" else np.uint16)
                xs = GEN.generate_all(seed, world, count, dtype, mode)
                ref = SM.exact_sum_f64(xs, dtype)
                g64 = got.astype(np.float64) if dtype == "f32" else SM.bf16_bits_to_f32(got).astype(np.float64)
                if mode == "integer":
                    ok = np.array_equal(g64, ref)
                elif dtype == "f32":   # rank 0 checks the bits; the others' equality is `same` below
                    ok = True
                    if rank == 0:
                        want = np.concatenate([XS.correctly_rounded_sum_f32(
                            [np.asarray(x[c0:c0 + (1 << 21)]).view(np.float32) for x in xs])
                            for c0 in range(0, count, 1 << 21)])
                        ok = np.array_equal(got.view(np.uint32), want.view(np.uint32))
                    if not ok:
                        print(f"rank {rank} f32 count={count}: {int(np.sum(got.view(np.uint32) != want.view(np.uint32)))} "
                              f"elements differ from the correctly rounded sum", flush=True)
                else:
                    err = SM.normwise_rel_err(got, ref, dtype)
                    ok = err <= (1e-6 if dtype == "f32" else 1e-2)
                allv = [None] * world
                dist.all_gather_object(allv, got[:4096].tobytes())
                same = all(a == allv[0] for a in allv)
                if not (ok and same):
                    print(f"rank {rank} FAIL {dtype} {mode} count={count} ok={ok} same={same}", flush=True)
                    failures += 1
    # NVLS as a GenTree plan kind (gentree_plan_nvls / force "nvls"): allreduce_exec on a
    # communicator with the NVLS buffer attached, ragged fp32 counts (vectors split evenly over
    # the ranks, scalar tail on the last rank), checked bit-for-bit against oracle.simulate of
    # the oracle's NVLS plan (= the correctly rounded sum, reading NV2) on every rank
    from oracle import gentree as GT
    from oracle import genmodel as OG
    from oracle import topology as T
    doc = T.single_switch_doc(world, {"alpha": 3e-6, "beta": 4 / 900e9, "epsilon": 0.0, "w_t": 9},
                              {"gamma": 0.0, "delta": 4 / 6.54e12})
    pp = G.params(9.4e-6, 1.465e-12, 0.0, 0.0, 0.0, 4)
    nvp = G.params(5.7e-6, 0.9e-12, 0.0, 0.0, 0.0, 1)    # NVLS row cheaper: the min-GenModel pick is NVLS
    comm = G.Comm.create(rank, world, local)
    comm.attach_nvls(nv)
    for count in (1, 3, world * 4 + 1, 1000003, (nbytes // 4) - 5):
        plan = G.Plan.from_topology_nvls(doc, count, "f32", pp, nvp)
        oplan, _ = GT.gentree_nvls(T.parse_topology(doc), count, 4, OG.Params(9.4e-6, 1.465e-12, 0, 0, 0, 4),
                                   OG.Params(5.7e-6, 0.9e-12, 0, 0, 0, 1))
        ok = plan.switch_reduce and oplan.switch_reduce
        G.fill_synthetic(nv.ptr, count, "f32", seed, rank, 0)
        torch.cuda.synchronize()
        dist.barrier()
        G.allreduce_exec(plan, comm, nv.ptr)
        torch.cuda.synchronize()
        comm.async_error()
        ok = ok and comm.last_kernel() == "nvls_kernel"
        got = nv.tensor[: count * 4].cpu().numpy().view(np.uint32)
        if rank in (0, world - 1):
            xs = GEN.generate_all(seed, world, count, "f32")
            want = np.concatenate([SM.simulate(type(oplan)(world, min(1 << 21, count - c0), oplan.steps[:0], True),
                                               [x[c0:c0 + (1 << 21)] for x in xs], "f32")[rank]
                                   for c0 in range(0, count, 1 << 21)])
            if not np.array_equal(got, want.view(np.uint32)):
                ok = False
                print(f"rank {rank} nvls plan count={count}: {int(np.sum(got != want.view(np.uint32)))} differ", flush=True)
        allv = [None] * world
        dist.all_gather_object(allv, got[-4096:].tobytes())
        if not (ok and all(a == allv[0] for a in allv)):
            print(f"rank {rank} FAIL nvls plan count={count}", flush=True)
            failures += 1
        if count in (world * 4 + 1, 1000003):   # AVG: the rounded sum / N, one RNE division
            G.fill_synthetic(nv.ptr, count, "f32", seed, rank, 0)
            torch.cuda.synchronize()
            dist.barrier()
            G.allreduce_exec(plan, comm, nv.ptr, op="avg")
            torch.cuda.synchronize()
            comm.async_error()
            got = nv.tensor[: count * 4].cpu().numpy().view(np.uint32)
            xs = GEN.generate_all(seed, world, count, "f32")
            want = SM.simulate(type(oplan)(world, count, oplan.steps[:0], True), xs, "f32", op="avg")[rank]
            if not np.array_equal(got, want.view(np.uint32)):
                print(f"rank {rank} FAIL nvls AVG count={count}: {int(np.sum(got != want.view(np.uint32)))} differ",
                      flush=True)
                failures += 1
    comm.destroy()
    dist.barrier()
    nv.destroy()
    dist.destroy_process_group()
    if rank == 0:
        print(f"nvls_worker world={world}: {'OK' if failures == 0 else f'{failures} FAILURES'}", flush=True)
    sys.exit(1 if failures else 0)


if __name__ == "__main__":
    main()
