"""Which rounding does the NVSwitch apply to a bf16 multimem.ld_reduce?  (CPU, offline)

    python tools/nvls_bf16_fit.py gpurun_out/nv/nvls_bf16_n4.npz [...]

Reads tools/nvls_dump.py's dumps (every rank's bf16 input bits and the switch's result bits)
and reports, for each (accumulation mode, data) case, the fraction of elements each rounding
hypothesis reproduces bit for bit.  Hypotheses are built from the exact rational sum of the
inputs (float64 where provably exact, Fraction otherwise) and from fixed association orders:

  exact_{rne,rz,rna,rto,rno}   exact sum rounded once to bf16 (ties-to-even, toward zero,
                                ties-away, round-to-odd (sticky), ties-to-odd)
  f32rne_then_{rne,rz,rna}      exact sum rounded to fp32 (RNE), then to bf16
  f32rz_then_{rne,rz,rna}       exact sum truncated to fp32, then to bf16
  seq_{order}_f32_{rne,rz}      sequential fp32 sum in a rank order, then to bf16
  seq_{order}_bf16_rne          every partial rounded to bf16 (RNE) (bf16 accumulation)

Then, over the elements whose exact sum is not a bf16 value, the probability that the switch
rounded AWAY from zero as a function of the sum's position between its two bf16 neighbours
(frac = distance from the toward-zero neighbour in units of the gap): a round-to-nearest unit
gives 0 below 1/2 and 1 above; stochastic rounding gives P(away) rising with frac.

Measurement analysis only; nothing on the product path depends on it.
"""
import json
import sys
from fractions import Fraction

import numpy as np


def bf16_to_f64(u16):
    return (u16.astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def exact_sums(X):
    """Exact Σ over axis 0 of float64 values X (N, n): float64 where every partial is exact,
    else a Fraction (object array entry)."""
    n = X.shape[0]
    nz = X != 0
    ex = np.frexp(X)[1].astype(np.int64)
    emax = np.where(nz, ex, -10 ** 6).max(axis=0)
    emin = np.where(nz, ex, 10 ** 6).min(axis=0)
    need = emax - emin + 8 + int(np.ceil(np.log2(n))) + 1
    exact = (~nz.any(axis=0)) | (need <= 53)
    s = np.zeros(X.shape[1])
    for r in range(n):
        s = s + X[r]
    out = s.astype(object)
    for i in np.nonzero(~exact)[0]:
        out[i] = sum(Fraction(float(v)) for v in X[:, i])
    return out


def round_to(q, mant_bits, mode):
    """Round the exact value q (float or Fraction) to a binary format with `mant_bits`
    significand bits (incl. hidden) and fp32's exponent range; returns a Python float."""
    q = Fraction(q)
    if q == 0:
        return 0.0
    sign = -1 if q < 0 else 1
    a = abs(q)
    k = a.numerator.bit_length() - a.denominator.bit_length()
    if Fraction(2) ** k > a if k >= 0 else Fraction(1, 2 ** -k) > a:
        k -= 1
    e = max(k, -126)
    quantum = Fraction(2) ** (e - mant_bits + 1) if e - mant_bits + 1 >= 0 else Fraction(1, 2 ** (mant_bits - 1 - e))
    m = a / quantum
    qi = m.numerator // m.denominator
    rem = m - qi
    half = Fraction(1, 2)
    if mode == "rne":
        up = rem > half or (rem == half and qi % 2 == 1)
    elif mode == "rz":
        up = False
    elif mode == "rna":
        up = rem >= half
    elif mode == "rno":   # ties to odd
        up = rem > half or (rem == half and qi % 2 == 0)
    elif mode == "rto":   # round to odd (sticky): truncate, set the last bit when inexact
        up = rem != 0 and qi % 2 == 0
    else:
        raise ValueError(mode)
    v = (qi + (1 if up else 0)) * quantum
    if v >= Fraction(2) ** 128:
        return sign * float("inf")
    return sign * float(v)


def f64_to_bf16_bits(v):
    f = np.asarray(v, dtype=np.float64).astype(np.float32)   # exact: v is a bf16 value
    return (f.view(np.uint32) >> 16).astype(np.uint16)


def vec_round(vals, mant_bits, mode):
    return np.array([round_to(v, mant_bits, mode) for v in vals], dtype=np.float64)


def f32_round_array(x, mode):
    """float64 array -> nearest fp32 under mode (vectorised for rne/rz)."""
    f = x.astype(np.float32)   # RNE
    if mode == "rne":
        return f.astype(np.float64)
    # rz: step back toward zero where RNE went away from zero
    away = np.abs(f.astype(np.float64)) > np.abs(x)
    g = f.copy()
    g[away] = np.nextafter(f[away], np.float32(0))
    return g.astype(np.float64)


def bf16_round_array(x, mode):
    """fp32-valued float64 array -> bf16 bits under mode (rne/rz/rna)."""
    u = x.astype(np.float32).view(np.uint32).astype(np.uint64)
    if mode == "rne":
        r = (u + 0x7FFF + ((u >> 16) & 1)) >> 16
    elif mode == "rz":
        r = u >> 16
    else:
        r = (u + 0x8000) >> 16
    return r.astype(np.uint16)


def hypotheses(inp):
    X = bf16_to_f64(inp)          # (N, n) exact
    N = X.shape[0]
    ex = exact_sums(X)
    H = {}
    for mode in ("rne", "rz", "rna", "rto", "rno"):
        H[f"exact_{mode}"] = f64_to_bf16_bits(vec_round(ex, 8, mode))
    f32_rne = np.array([round_to(v, 24, "rne") for v in ex])
    f32_rz = np.array([round_to(v, 24, "rz") for v in ex])
    for m in ("rne", "rz", "rna"):
        H[f"f32rne_then_{m}"] = bf16_round_array(f32_rne, m)
        H[f"f32rz_then_{m}"] = bf16_round_array(f32_rz, m)
    orders = {"asc": list(range(N)), "desc": list(range(N - 1, -1, -1))}
    for s in range(1, N):
        orders[f"rot{s}"] = [(s + i) % N for i in range(N)]
    for name, order in orders.items():
        acc = X[order[0]].astype(np.float32)
        accz = X[order[0]].copy()
        accb = X[order[0]].copy()
        for q in order[1:]:
            acc = (acc + X[q].astype(np.float32)).astype(np.float32)
            accz = f32_round_array(accz + X[q], "rz")    # fp32 partials exact in f64 before rounding
            accb = bf16_to_f64(bf16_round_array(accb + X[q], "rne"))
        H[f"seq_{name}_f32_rne"] = bf16_round_array(acc.astype(np.float64), "rne")
        H[f"seq_{name}_f32_rz"] = bf16_round_array(accz, "rne")
        H[f"seq_{name}_bf16_rne"] = bf16_round_array(accb, "rne")
    if N == 4:
        for a, b, c, d in ((0, 1, 2, 3), (0, 2, 1, 3), (0, 3, 1, 2)):
            p = (X[a].astype(np.float32) + X[b].astype(np.float32)).astype(np.float32)
            q = (X[c].astype(np.float32) + X[d].astype(np.float32)).astype(np.float32)
            H[f"pairs_{a}{b}_{c}{d}_f32_rne"] = bf16_round_array((p + q).astype(np.float64), "rne")
            pb = bf16_to_f64(bf16_round_array(X[a] + X[b], "rne"))
            qb = bf16_to_f64(bf16_round_array(X[c] + X[d], "rne"))
            H[f"pairs_{a}{b}_{c}{d}_bf16_rne"] = bf16_round_array(pb + qb, "rne")
    return H


def away_table(inp, got):
    """P(rounded away from zero | frac) in eighths, plus the ties (frac = 1/2) separately."""
    X = bf16_to_f64(inp)
    ex = exact_sums(X)
    g = bf16_to_f64(got)
    fr, aw = [], []
    for i in range(got.size):
        q = Fraction(ex[i])
        z = Fraction(round_to(q, 8, "rz"))
        if q == z:
            continue
        b = int(np.array([float(z)], dtype=np.float32).view(np.uint32)[0] >> 16)
        nxt = Fraction(float(np.array([(b + 1) << 16], dtype=np.uint32).view(np.float32)[0]))
        fr.append(float((abs(q) - abs(z)) / (abs(nxt) - abs(z))))
        aw.append(bool(g[i] != float(z)))
    fr, aw = np.array(fr), np.array(aw)
    rows = []
    for k in range(8):
        m = (fr >= k / 8) & (fr < (k + 1) / 8)
        if m.any():
            rows.append({"frac": [k / 8, (k + 1) / 8], "n": int(m.sum()), "p_away": round(float(aw[m].mean()), 4)})
    t = fr == 0.5
    return {"inexact": int(fr.size), "bins": rows,
            "ties": {"n": int(t.sum()), "p_away": round(float(aw[t].mean()), 4) if t.any() else None}}


def main():
    for path in sys.argv[1:]:
        d = np.load(path)
        cases = sorted({k.rsplit("_", 1)[0] for k in d.files})
        for case in cases:
            inp, got = d[case + "_inputs"], d[case + "_result"]
            n = min(got.size, 200000)
            inp, got = inp[:, :n], got[:n]
            H = hypotheses(inp)
            match = {k: float(np.mean(v == got)) for k, v in H.items()}
            best = sorted(match.items(), key=lambda kv: -kv[1])[:6]
            bk = best[0][0]
            bad = np.nonzero(H[bk] != got)[0][:5]
            X = bf16_to_f64(inp)
            print(json.dumps({"file": path, "case": case, "world": int(inp.shape[0]), "elements": int(n),
                              "best": best,
                              "best_misses": [{"inputs": [float(x) for x in X[:, i]], "got": int(got[i]),
                                               "best": int(H[bk][i]),
                                               "exact": float(sum(Fraction(float(x)) for x in X[:, i]))}
                                              for i in bad],
                              "p_away_by_frac": away_table(inp[:, :60000], got[:60000])}), flush=True)


if __name__ == "__main__":
    main()
