"""Seeded synthetic AllReduce inputs — the ONE module shared by the oracle and the CUDA path.

This module holds none of the method's arithmetic (no sums, no rounding of sums, no
plans).  It only produces per-rank input vectors from a counter-based generator so
that the CPU oracle (`oracle/`) and the GPU path (which has its own, independent CUDA
implementation of the same generator, `ar_fill_synthetic` in the C-ABI library) see
bit-identical inputs without copying data between them.

Generator G(seed, rank, i):

    z  = splitmix64(seed * 0x9E3779B97F4A7C15  ^  (rank << 48)  ^  i)
    e  = 7 + splitmix64(seed ^ 0xA5A5 ^ (i >> 16)) % 12      # per-64Ki-element "layer" scale,
                                                              # shared by all ranks
    fp32 : m = ((z >> 40) & 0xFFFFFF) - 0x800000   (24-bit signed)   x = m * 2^-(23+e)
    bf16 : m = ((z >> 56) & 0xFF)     - 0x80       ( 8-bit signed)   x = m * 2^-(7+e)

Both are exact in their storage type (|m| fits the significand), zero-mean, and the
per-layer scale spans ~3.5 decades: "gradient-shaped" data.  The paper's data content is
unspecified beyond "float" (§3 "Experimental Settings").

Modes:
  "gradient"  — the recipe above (default, used by bench and parity tests)
  "integer"   — x = m with m uniform in [-2^10, 2^10] (fp32) or [-2^5, 2^5] (bf16): every
                partial sum of <=64 (fp32) / <=8 (bf16) ranks is exact, so any plan's
                output must equal the int64 sum (order-independent pin).
  "specials"  — a fixed cycle of IEEE special values (±0, subnormals, ±max, ±inf, NaN)
                mixed with gradient values.
"""
from __future__ import annotations

import numpy as np

MASK64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15
SEED_BASE = 0x240904202

F32 = "f32"
BF16 = "bf16"
DTYPES = (F32, BF16)
MODES = ("gradient", "integer", "specials")
MODE_ID = {"gradient": 0, "integer": 1, "specials": 2}

# fp32 bit patterns cycled through by mode "specials" (every 8th element is special)
SPECIALS_F32 = np.array(
    [0x00000000, 0x80000000, 0x00000001, 0x807FFFFF, 0x7F7FFFFF, 0xFF7FFFFF,
     0x7F800000, 0xFF800000, 0x7FC00000, 0x00800000, 0x80000010, 0x3F800000],
    dtype=np.uint32)
SPECIALS_BF16 = np.array(
    [0x0000, 0x8000, 0x0001, 0x807F, 0x7F7F, 0xFF7F,
     0x7F80, 0xFF80, 0x7FC0, 0x0080, 0x8010, 0x3F80],
    dtype=np.uint16)


def config_seed(config_id: int) -> int:
    """seed = 0x240904202 ^ config_id (recorded in every bench row)."""
    return (SEED_BASE ^ int(config_id)) & MASK64


def _splitmix64(x: np.ndarray) -> np.ndarray:
    """Vectorised SplitMix64 finaliser on uint64 arrays (wrapping arithmetic)."""
    with np.errstate(over="ignore"):
        x = x + np.uint64(GOLDEN)
        z = x
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def splitmix64_scalar(x: int) -> int:
    """Scalar reference of the same finaliser (used by tests of this module)."""
    x = (x + GOLDEN) & MASK64
    z = x
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


def generate(seed: int, rank: int, count: int, dtype: str = F32, mode: str = "gradient",
             start: int = 0) -> np.ndarray:
    """Rank `rank`'s input elements [start, start+count).

    Returns float32 values for dtype "f32" and the uint16 bit patterns for "bf16".
    """
    if dtype not in DTYPES:
        raise ValueError(f"dtype must be one of {DTYPES}")
    if mode not in MODES:
        raise ValueError(f"mode must be one of {MODES}")
    i = np.arange(start, start + count, dtype=np.uint64)
    with np.errstate(over="ignore"):
        key = np.uint64((seed * GOLDEN) & MASK64) ^ np.uint64((rank << 48) & MASK64)
    z = _splitmix64(key ^ i)
    if mode == "integer":
        if dtype == F32:
            m = (z % np.uint64(2049)).astype(np.int64) - 1024
            return m.astype(np.float32)
        m = (z % np.uint64(65)).astype(np.int64) - 32
        return (m.astype(np.float32).view(np.uint32) >> np.uint32(16)).astype(np.uint16)
    layer = _splitmix64(np.uint64(seed ^ 0xA5A5) ^ (i >> np.uint64(16)))
    e = (layer % np.uint64(12)).astype(np.int32) + 7
    if dtype == F32:
        m = ((z >> np.uint64(40)) & np.uint64(0xFFFFFF)).astype(np.int64) - 0x800000
        x = np.ldexp(m.astype(np.float64), -(23 + e)).astype(np.float32)  # exact
        out = x
        if mode == "specials":
            bits = out.view(np.uint32).copy()
            sel = (i % np.uint64(8)) == 0
            idx = ((i // np.uint64(8)) % np.uint64(len(SPECIALS_F32))).astype(np.int64)
            bits[sel] = SPECIALS_F32[idx[sel]]
            out = bits.view(np.float32)
        return out
    m = ((z >> np.uint64(56)) & np.uint64(0xFF)).astype(np.int64) - 0x80
    x = np.ldexp(m.astype(np.float64), -(7 + e)).astype(np.float32)  # exact, low 16 bits zero
    bits = (x.view(np.uint32) >> np.uint32(16)).astype(np.uint16)
    if mode == "specials":
        sel = (i % np.uint64(8)) == 0
        idx = ((i // np.uint64(8)) % np.uint64(len(SPECIALS_BF16))).astype(np.int64)
        bits[sel] = SPECIALS_BF16[idx[sel]]
    return bits


def generate_all(seed: int, world: int, count: int, dtype: str = F32,
                 mode: str = "gradient") -> list[np.ndarray]:
    """Inputs of all `world` ranks."""
    return [generate(seed, r, count, dtype, mode) for r in range(world)]


def as_f64(x: np.ndarray, dtype: str) -> np.ndarray:
    """Exact widening of stored values to float64 (bf16 bits -> value)."""
    if dtype == F32:
        return x.astype(np.float64)
    return (x.astype(np.uint32) << np.uint32(16)).view(np.float32).astype(np.float64)
