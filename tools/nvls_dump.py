"""Dump what the NVSwitch returns for bf16 multimem.ld_reduce, for offline analysis (torchrun).

    python -m torch.distributed.run --nproc-per-node N tools/nvls_dump.py OUTDIR

For bf16 with fp32 accumulation in the switch (`acc::f32`, the NVLS kernel's default) and with
bf16 accumulation (AR_NVLS_BF16_ACC=bf16), on gradient-shaped and adversarial inputs
(tools/nvls_order.py's generators), rank 0 writes OUTDIR/nvls_bf16_n{N}.npz holding every
rank's input bits and the result bits.  tools/nvls_bf16_fit.py then tests rounding hypotheses
against the dump on the CPU.  A measurement tool; nothing on the product path depends on it.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2409_04202_b200 as G  # noqa: E402
from synth import generator as GEN  # noqa: E402
from tools.nvls_order import adversarial, f32_to_bf16_rne  # noqa: E402


def main():
    out_dir = sys.argv[1]
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    count = 1 << 20
    seed = GEN.config_seed(12)
    arrays = {}
    for acc in ("f32", "bf16"):
        if acc == "bf16":
            os.environ["AR_NVLS_BF16_ACC"] = "bf16"
        nv = G.Nvls(count * 2, local)
        os.environ.pop("AR_NVLS_BF16_ACC", None)
        for kind in ("gradient", "adversarial"):
            if kind == "adversarial":
                adv = adversarial(seed, world, count, "bf16")
                xs = [f32_to_bf16_rne(a) for a in adv]
                nv.tensor[: count * 2].copy_(torch.from_numpy(xs[rank].view(np.uint8).copy()))
            else:
                xs = [np.asarray(x).view(np.uint16) for x in GEN.generate_all(seed, world, count, "bf16", "gradient")]
                G.fill_synthetic(nv.ptr, count, "bf16", seed, rank, 0)
            torch.cuda.synchronize()
            dist.barrier()
            nv.allreduce(count, "bf16")
            torch.cuda.synchronize()
            nv.async_error()
            got = nv.tensor[: count * 2].cpu().numpy().copy().view(np.uint16)
            if rank == 0:
                arrays[f"{acc}_{kind}_inputs"] = np.stack(xs)
                arrays[f"{acc}_{kind}_result"] = got
            dist.barrier()
        nv.destroy()
    if rank == 0:
        os.makedirs(out_dir, exist_ok=True)
        np.savez_compressed(os.path.join(out_dir, f"nvls_bf16_n{world}.npz"), **arrays)
        print(f"nvls_dump world={world}: wrote {len(arrays)} arrays", flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
