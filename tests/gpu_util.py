"""Helpers shared by the GPU tests (no method arithmetic here)."""
from __future__ import annotations

import numpy as np


def cuda_ok() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def emulated_buffer(world: int, count: int, dtype: str, seed: int, mode: int = 0):
    """Device buffer holding `world` rank buffers (stride = ar_rank_stride_bytes), filled with
    the synthetic generator on the device (ar_fill_synthetic)."""
    import torch

    import paper_2409_04202_b200 as G
    stride = G.rank_stride_bytes(count, dtype)
    buf = torch.zeros(world * stride, dtype=torch.uint8, device="cuda")
    for r in range(world):
        G.fill_synthetic(buf.data_ptr() + r * stride, count, dtype, seed, r, mode)
    return buf, stride


def rank_views(buf, world: int, count: int, dtype: str, stride: int) -> list:
    """Host copies of each rank's buffer: float32 arrays or uint16 bf16 bit arrays."""
    host = buf.cpu().numpy()
    es = 4 if dtype == "f32" else 2
    out = []
    for r in range(world):
        raw = host[r * stride: r * stride + count * es]
        out.append(raw.view(np.float32 if dtype == "f32" else np.uint16).copy())
    return out


def assert_bits_equal(got: np.ndarray, want: np.ndarray, dtype: str, what: str = ""):
    """Bitwise equality; NaNs compared by isnan only (payloads are not part of the contract)."""
    if dtype == "f32":
        g, w = got.view(np.uint32), want.view(np.uint32)
        gn, wn = np.isnan(got), np.isnan(want)
    else:
        g, w = got, want
        gn = ((got & 0x7F80) == 0x7F80) & ((got & 0x7F) != 0)
        wn = ((want & 0x7F80) == 0x7F80) & ((want & 0x7F) != 0)
    if not np.array_equal(gn, wn):
        i = int(np.nonzero(gn != wn)[0][0])
        raise AssertionError(f"{what}: NaN mismatch at {i}")
    ok = (g == w) | gn
    if not ok.all():
        i = int(np.nonzero(~ok)[0][0])
        raise AssertionError(f"{what}: first mismatch at element {i}: got {int(g[i]):#x} want {int(w[i]):#x} "
                             f"({int((~ok).sum())} mismatches)")


def cps_path_kernel(paths: dict, count: int, es: int, world: int) -> str:
    """The kernel the executor picks for a CPS-shaped plan on a one-rank-per-GPU communicator
    with these cut-offs (ar_comm_get_paths; 8-byte-aligned buffer): the LL128 kernel in
    (ll128_min, ll128_max] for N <= 8, else the one-shot kernel up to oneshot_max, else the
    step-table kernel."""
    nbytes = count * es
    if world <= 8 and paths["ll128_max"] and paths["ll128_min"] < nbytes <= paths["ll128_max"] and nbytes >= 8 * world:
        return "ar_ll128_kernel"
    if nbytes <= paths["oneshot_max"]:
        return "ar_ll_kernel"
    return "ar_exec_kernel"
