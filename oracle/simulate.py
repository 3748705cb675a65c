"""Step-by-step data simulation of a plan (oracle; test infrastructure only).

Follows the plan semantics of `oracle.plans` literally:
  * RS Reduce(server r, block b, inputs I):  acc = x[I0][b] (widened to fp32);
    acc = acc + x[Ij][b] for j = 1..k-1, one IEEE binary32 round-to-nearest-even add per
    element, left to right (reading Q1; numpy float32 elementwise add has no FMA and no
    re-association); bf16 data is widened exactly and rounded to bf16 (RNE) once, when the
    partial is stored (reading Q2).  A one-input Reduce is a raw bit move.
  * AG Transfer(src, dst, b): raw bit copy.
  * op "avg" (reading AV1): the Reduce(s) of block b in the
    last RS step that reduces b divide the fp32 sum by N (one correctly rounded IEEE binary32
    division) before the store's rounding; a one-input Reduce there widens, divides, stores.
Every step's hazard-freedom is checked first (`check_step_hazards`), so applying its ops in
any order is equivalent to the concurrent semantics.

`simulate_scalar` is an independent brute-force re-implementation (dict of Python lists,
binary32 rounding through `struct`) used only to pin `simulate` on tiny cases.
"""
from __future__ import annotations

import struct

import numpy as np

from .plans import Plan, block_offset, block_size, check_step_hazards


def bf16_bits_to_f32(u16: np.ndarray) -> np.ndarray:
    return (u16.astype(np.uint32) << np.uint32(16)).view(np.float32)


def f32_to_bf16_rne(x: np.ndarray) -> np.ndarray:
    """Round binary32 to bfloat16, ties to even; NaN -> quiet NaN keeping the sign."""
    u = x.view(np.uint32).astype(np.uint64)
    rounded = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)
    nan = np.isnan(x)
    if nan.any():
        sign = ((u >> 16) & 0x8000).astype(np.uint16)
        rounded = np.where(nan, np.uint16(0x7FC0) | sign, rounded)
    return rounded.astype(np.uint16)


def last_rs_step(plan: Plan) -> dict:
    """block -> index of the last RS step that has a Reduce writing it (reading AV1)."""
    last = {}
    for i, st in enumerate(plan.steps):
        if st.phase == "rs":
            for rd in st.reduces:
                last[rd.block] = i
    return last


def simulate(plan: Plan, inputs: list, dtype: str, op: str = "sum") -> list:
    """Run `plan` on per-rank inputs (float32 arrays, or uint16 bf16 bit arrays).
    Returns the per-rank output buffers (new arrays)."""
    n, count = plan.n, plan.count
    if op not in ("sum", "avg"):
        raise ValueError(op)
    if plan.switch_reduce:
        # NVLS plan (reading NV2): every element is the correctly rounded fp32 sum of the
        # ranks' inputs, on every rank (the switch reduces each element once); AVG (reading
        # AV1 on this kind): that sum divided by N, one IEEE binary32 division (RNE)
        if dtype != "f32":
            raise ValueError("NVLS plans: fp32 only (reading NV2)")
        from .exactsum import correctly_rounded_sum_f32
        out = correctly_rounded_sum_f32(inputs)
        if op == "avg":
            out = (out / np.float32(n)).astype(np.float32)
        return [out.copy() for _ in range(n)]
    last = last_rs_step(plan)
    bufs = [np.array(x, copy=True) for x in inputs]
    for x in bufs:
        if x.shape != (count,):
            raise ValueError("input length != plan count")
    for si, st in enumerate(plan.steps):
        check_step_hazards(st)
        if st.phase == "rs":
            for rd in st.reduces:
                o, sz = block_offset(count, n, rd.block), block_size(count, n, rd.block)
                if sz == 0:
                    continue
                div = op == "avg" and last[rd.block] == si
                if len(rd.inputs) == 1 and not div:
                    bufs[rd.server][o:o + sz] = bufs[rd.inputs[0]][o:o + sz]
                    continue
                if dtype == "f32":
                    acc = bufs[rd.inputs[0]][o:o + sz].astype(np.float32, copy=True)
                    for q in rd.inputs[1:]:
                        acc = acc + bufs[q][o:o + sz]
                    if div:
                        acc = acc / np.float32(n)
                    bufs[rd.server][o:o + sz] = acc
                else:
                    acc = bf16_bits_to_f32(bufs[rd.inputs[0]][o:o + sz]).copy()
                    for q in rd.inputs[1:]:
                        acc = acc + bf16_bits_to_f32(bufs[q][o:o + sz])
                    if div:
                        acc = acc / np.float32(n)
                    bufs[rd.server][o:o + sz] = f32_to_bf16_rne(acc)
        else:
            for t in st.transfers:
                o = block_offset(count, n, t.block)
                bufs[t.dst][o:o + t.size] = bufs[t.src][o:o + t.size]
    return bufs


# ---------------------------------------------------------------- independent brute force

def _f32(v: float) -> float:
    """Round a double to binary32 (RNE).  The double sum of two binary32 values rounded once
    more to binary32 is the correctly rounded binary32 sum (53 >= 2*24 + 2)."""
    if v == v and abs(v) >= 2.0 ** 128 - 2.0 ** 103:   # at/above the overflow midpoint
        return float("inf") if v > 0 else float("-inf")
    return struct.unpack("<f", struct.pack("<f", v))[0]


def _bits_f32(v: float) -> int:
    return struct.unpack("<I", struct.pack("<f", v))[0]


def _bf16_round(v: float) -> int:
    """Scalar RNE to bf16 written independently of f32_to_bf16_rne: choose the nearer of the
    two bf16 neighbours (by exact real distance), ties to the even one."""
    u = _bits_f32(v)
    if v != v:
        return 0x7FC0 | ((u >> 16) & 0x8000)
    lo = u >> 16
    hi = lo + 1
    vlo = struct.unpack("<f", struct.pack("<I", lo << 16))[0]
    if (hi & 0x7F80) == 0x7F80 and (hi & 0x7F) == 0:
        # the neighbour above the largest finite bf16 is "2^128" for rounding purposes
        vhi = 2.0 ** 128 if not (u >> 31) else -(2.0 ** 128)
    else:
        vhi = struct.unpack("<f", struct.pack("<I", (hi & 0xFFFF) << 16))[0]
    if (u & 0xFFFF) == 0:
        return lo
    dlo, dhi = abs(v - vlo), abs(vhi - v)
    if dlo < dhi:
        return lo
    if dhi < dlo:
        return hi & 0xFFFF
    return lo if (lo & 1) == 0 else (hi & 0xFFFF)


def simulate_scalar(plan: Plan, inputs: list, dtype: str, op: str = "sum") -> list:
    """Element-by-element re-implementation for tiny cases (pins `simulate`).  AVG: the
    double quotient of binary32 values rounded once to binary32 is the correctly rounded
    binary32 quotient (53 >= 2*24 + 2)."""
    n, count = plan.n, plan.count
    final = {}
    for i, st in enumerate(plan.steps):
        if st.phase == "rs":
            for rd in st.reduces:
                final[rd.block] = i
    if dtype == "f32":
        bufs = [[float(v) for v in x] for x in inputs]
    else:
        bufs = [[int(v) for v in x] for x in inputs]

    def val(q, e):
        if dtype == "f32":
            return bufs[q][e]
        return struct.unpack("<f", struct.pack("<I", bufs[q][e] << 16))[0]

    for si, st in enumerate(plan.steps):
        new = {}
        if st.phase == "rs":
            for rd in st.reduces:
                o = block_offset(count, n, rd.block)
                div = op == "avg" and final[rd.block] == si
                for e in range(o, o + block_size(count, n, rd.block)):
                    if len(rd.inputs) == 1 and not div:
                        new[(rd.server, e)] = bufs[rd.inputs[0]][e]
                        continue
                    acc = val(rd.inputs[0], e)
                    for q in rd.inputs[1:]:
                        acc = _f32(acc + val(q, e))
                    if div:
                        acc = _f32(acc / n)
                    new[(rd.server, e)] = acc if dtype == "f32" else _bf16_round(acc)
        else:
            for t in st.transfers:
                o = block_offset(count, n, t.block)
                for e in range(o, o + t.size):
                    new[(t.dst, e)] = bufs[t.src][e]
        for (r, e), v in new.items():
            bufs[r][e] = v
    if dtype == "f32":
        return [np.array(b, dtype=np.float32) for b in bufs]
    return [np.array(b, dtype=np.uint16) for b in bufs]


def simulate_at(plan: Plan, idx, values: list, dtype: str, op: str = "sum") -> list:
    """The plan's outputs at selected element indices only (for full-size checks).

    idx: sorted element indices; values[r][k] = rank r's input at idx[k] (float32 values or
    bf16 bit patterns).  Replays every step on just those elements, with the same
    arithmetic as `simulate`.  Returns per-rank arrays of len(idx)."""
    n, count = plan.n, plan.count
    idx = np.asarray(idx, dtype=np.int64)
    bufs = [np.array(v, copy=True) for v in values]
    starts = np.array([block_offset(count, n, b) for b in range(n)], dtype=np.int64)
    blk = np.searchsorted(starts, idx, side="right") - 1
    last = last_rs_step(plan)
    for si, st in enumerate(plan.steps):
        if st.phase == "rs":
            for rd in st.reduces:
                sel = np.nonzero(blk == rd.block)[0]
                if sel.size == 0:
                    continue
                div = op == "avg" and last[rd.block] == si
                if len(rd.inputs) == 1 and not div:
                    bufs[rd.server][sel] = bufs[rd.inputs[0]][sel]
                    continue
                if dtype == "f32":
                    acc = bufs[rd.inputs[0]][sel].astype(np.float32, copy=True)
                    for q in rd.inputs[1:]:
                        acc = acc + bufs[q][sel]
                    if div:
                        acc = acc / np.float32(n)
                    bufs[rd.server][sel] = acc
                else:
                    acc = bf16_bits_to_f32(bufs[rd.inputs[0]][sel]).copy()
                    for q in rd.inputs[1:]:
                        acc = acc + bf16_bits_to_f32(bufs[q][sel])
                    if div:
                        acc = acc / np.float32(n)
                    bufs[rd.server][sel] = f32_to_bf16_rne(acc)
        else:
            for t in st.transfers:
                sel = np.nonzero(blk == t.block)[0]
                if sel.size:
                    bufs[t.dst][sel] = bufs[t.src][sel]
    return bufs


def exact_sum_f64(inputs: list, dtype: str) -> np.ndarray:
    """The plain definition out[e] = sum_q x_q[e], accumulated in float64
    (exact for the generator's inputs up to N=64 ranks only in 'integer' mode; otherwise
    the accuracy reference of reading Q21)."""
    acc = np.zeros(len(inputs[0]), dtype=np.float64)
    for x in inputs:
        acc += (x.astype(np.float64) if dtype == "f32" else
                bf16_bits_to_f32(x).astype(np.float64))
    return acc


def normwise_rel_err(out: np.ndarray, ref: np.ndarray, dtype: str) -> float:
    """Reading Q21: ||y - ref||_2 / ||ref||_2."""
    y = out.astype(np.float64) if dtype == "f32" else bf16_bits_to_f32(out).astype(np.float64)
    den = np.linalg.norm(ref)
    return float(np.linalg.norm(y - ref) / den) if den > 0 else float(np.linalg.norm(y))
