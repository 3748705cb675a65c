"""Fitting GenModel to a machine (oracle; test infrastructure only).

§3.4: fit from Co-located-PS benchmarks on 2..max communicators; only
(2β + γ) is identifiable ("the ratio of the β-term coefficient to the γ-term coefficient is
always 2"), β can be computed from the bandwidth and γ = (2β+γ) − 2β.  The procedure below
is SPEC's — the paper does not give its solver:

  for each candidate w_t: non-negative least squares for [α, k = 2β+γ, δ, ε] on the CPS
  row of Table 2,  T(n, s) = 2α + ((n−1)s/n)·k + ((n+1)s/n)·δ + max(n − w_t, 0)·(2(n−1)s/n)·ε
  pick the smallest SSE; candidates within a relative 1e-6 (+1e-24 absolute) of the best
  count as tied and the smallest w_t wins (reading F1).
Repeated (n, s) rows are averaged first (the paper reports means).

Eq. 6: T(x) = (x+1)·S·δ + (x−1)·S·γ  ⇒  T(x)/(x−1) = C1·(x+1)/(x−1) + C2 with
C1 = S·δ, C2 = S·γ; `fit_eq6` fits it (least squares, optionally non-negative).
"""
from __future__ import annotations

import numpy as np
from scipy.optimize import nnls

from .genmodel import Params


def cps_design_row(n: int, s: float, w_t: int) -> list:
    return [2.0, (n - 1) * s / n, (n + 1) * s / n, max(n - w_t, 0) * 2.0 * (n - 1) * s / n]


def average_rows(rows):
    acc = {}
    for n, s, t in rows:
        acc.setdefault((int(n), float(s)), []).append(float(t))
    return [(n, s, sum(v) / len(v)) for (n, s), v in sorted(acc.items())]


def fit_params(rows, wt_min: int, wt_max: int):
    """rows: (n, s_bytes, t_seconds).  Returns (alpha, k, delta, epsilon, w_t, sse, scan)."""
    rows = average_rows(rows)
    if len(rows) < 4:
        raise ValueError("underdetermined: need >= 4 distinct (n, s) rows")
    if len({n for n, _, _ in rows}) < 2 or len({s for _, s, _ in rows}) < 2:
        raise ValueError("underdetermined: need >= 2 distinct n and >= 2 distinct s")
    t = np.array([r[2] for r in rows])
    scan = []
    for w_t in range(wt_min, wt_max + 1):
        A = np.array([cps_design_row(n, s, w_t) for n, s, _ in rows])
        # column scaling keeps NNLS well conditioned (s spans decades)
        scale = np.maximum(np.abs(A).max(axis=0), 1e-300)
        x, _ = nnls(A / scale, t)
        x = x / scale
        r = A @ x - t
        scan.append((w_t, float(r @ r), x))
    best = min(v[1] for v in scan)
    tol = best * 1e-6 + 1e-24
    w_t, sse, x = next(v for v in scan if v[1] <= best + tol)
    return {"alpha": float(x[0]), "combined": float(x[1]), "delta": float(x[2]),
            "epsilon": float(x[3]), "w_t": w_t, "sse": sse,
            "scan": [(w, s) for w, s, _ in scan]}


def nvls_design_row(n: int, s: float) -> list:
    """NVLS row of the closed forms (reading NV1): T = 2α + ((n+1)·s/n)·β."""
    return [2.0, (n + 1) * s / n]


def fit_nvls(rows):
    """NNLS for (α, β) of the NVLS row ("α and β fitted in C3").
    rows: (n, s_bytes, t_seconds), repeated (n, s) averaged.  Needs >= 2 distinct rows."""
    rows = average_rows(rows)
    if len(rows) < 2 or len({s for _, s, _ in rows}) < 2:
        raise ValueError("underdetermined: need >= 2 distinct sizes")
    A = np.array([nvls_design_row(n, s) for n, s, _ in rows])
    t = np.array([r[2] for r in rows])
    scale = np.maximum(np.abs(A).max(axis=0), 1e-300)
    x, _ = nnls(A / scale, t)
    x = x / scale
    r = A @ x - t
    return {"alpha": float(x[0]), "beta": float(x[1]), "sse": float(r @ r)}


def fit_row(kind: str, rows):
    """NNLS for (α, β) of a closed-form row's A and B coefficients (the "nvls" and "oneshot"
    rows: their own fitted latency and per-byte link cost, C/D/I absorbed).  rows: (n, s, t)."""
    from .genmodel import closed_form_terms
    rows = average_rows(rows)
    if len(rows) < 2 or len({s for _, s, _ in rows}) < 2:
        raise ValueError("underdetermined: need >= 2 distinct sizes")
    A = []
    for n, s, _ in rows:
        a_, bn, _, _, _, den = closed_form_terms(kind, n, int(s), 1 << 30)
        A.append([float(a_), bn / den])
    A = np.array(A)
    t = np.array([r[2] for r in rows])
    scale = np.maximum(np.abs(A).max(axis=0), 1e-300)
    x, _ = nnls(A / scale, t)
    x = x / scale
    r = A @ x - t
    return {"alpha": float(x[0]), "beta": float(x[1]), "sse": float(r @ r)}


def split_combined(k: float, link_bytes_per_s: float):
    """β from the bandwidth, γ = k − 2β; error if that is negative."""
    beta = 1.0 / link_bytes_per_s
    gamma = k - 2.0 * beta
    if gamma < 0:
        raise ValueError("k < 2β: inconsistent inputs")
    return beta, gamma


def params_from_fit(fit: dict, link_bytes_per_s: float | None = None) -> Params:
    if link_bytes_per_s:
        beta, gamma = split_combined(fit["combined"], link_bytes_per_s)
        return Params(fit["alpha"], beta, gamma, fit["delta"], fit["epsilon"], fit["w_t"])
    return Params(fit["alpha"], 0.0, 0.0, fit["delta"], fit["epsilon"], fit["w_t"],
                  combined=fit["combined"])


def cps_forward(n: int, s: float, alpha, k, delta, eps, w_t) -> float:
    """The CPS row of Table 2 as used by the fit."""
    row = cps_design_row(n, s, w_t)
    return row[0] * alpha + row[1] * k + row[2] * delta + row[3] * eps


def fit_eq6(x, t_per_op, nonneg: bool = False):
    """Fit T(x)/(x−1) = a/(x−1) + b  (a = 2·C1, b = C1 + C2) and return
    (a, b, C1 = S·δ, C2 = S·γ).  Eq. 6 with (x+1)/(x−1) = 1 + 2/(x−1) (reading Q18)."""
    x = np.asarray(x, dtype=float)
    y = np.asarray(t_per_op, dtype=float)
    A = np.stack([1.0 / (x - 1.0), np.ones_like(x)], axis=1)
    if nonneg:
        # parametrise directly in (C1, C2) >= 0: y = C1*(x+1)/(x-1) + C2
        B = np.stack([(x + 1.0) / (x - 1.0), np.ones_like(x)], axis=1)
        (c1, c2), _ = nnls(B, y)
        return 2 * c1, c1 + c2, float(c1), float(c2)
    (a, b), *_ = np.linalg.lstsq(A, y, rcond=None)
    return float(a), float(b), float(a / 2), float(b - a / 2)
