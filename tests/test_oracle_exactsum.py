"""Pins for oracle.exactsum (reading NV2: the NVLS fp32 result is the correctly rounded sum).

Independent of the implementation: the IEEE binary32 add is correctly rounded by definition
(N = 2 must equal numpy's float32 add), the defining property of round-to-nearest-even is
checked directly on the exact rational sum, and hand-worked ties/overflow/zero cases."""
import math
import struct
from fractions import Fraction

import numpy as np
import pytest

from oracle.exactsum import correctly_rounded_sum_f32, round_fraction_to_f32


def f32(x):
    return float(np.float32(x))


def wide_random(rng, n, count, span):
    """Random binary32 values over 2^span binades, both signs, some zeros and subnormals."""
    m = rng.integers(1, 1 << 24, size=(n, count)).astype(np.float64)
    e = rng.integers(-span // 2, span // 2, size=(n, count))
    x = (rng.choice([-1.0, 1.0], size=(n, count)) * m * np.exp2(e - 24)).astype(np.float32)
    x[rng.random((n, count)) < 0.05] = 0
    x[rng.random((n, count)) < 0.02] = np.float32(1e-40) * rng.integers(1, 100)   # subnormal
    return x


def test_two_inputs_equal_ieee_single_add():
    rng = np.random.default_rng(0)
    for span in (4, 40, 200):
        x = wide_random(rng, 2, 20000, span)
        with np.errstate(over="ignore"):
            ieee = (x[0] + x[1]).astype(np.float32)
        got = correctly_rounded_sum_f32([x[0], x[1]])
        both_zero = (ieee == 0) & (got == 0)
        assert np.array_equal(got.view(np.uint32)[~both_zero], ieee.view(np.uint32)[~both_zero]), span
        assert np.all(~np.signbit(got[both_zero]))          # an exactly-zero sum is +0


def _neighbours(r):
    b = struct.unpack("<I", struct.pack("<f", r))[0]
    return [struct.unpack("<f", struct.pack("<I", b + d))[0] for d in (-1, 1)] if r > 0 else []


@pytest.mark.parametrize("n", [3, 4, 8])
def test_nearest_ties_to_even_property(n):
    """r is a binary32 no farther from the exact sum than either neighbour; at a tie, its
    significand is even.  Checked on the exact Fraction sum, element by element."""
    rng = np.random.default_rng(n)
    for span in (6, 60):
        x = wide_random(rng, n, 400, span)
        got = correctly_rounded_sum_f32(list(x))
        for i in range(x.shape[1]):
            exact = sum(Fraction(float(v)) for v in x[:, i])
            r = float(got[i])
            a, ra = abs(exact), abs(r)
            assert math.copysign(1, r) == (math.copysign(1, float(exact)) if exact != 0 else 1)
            d = abs(Fraction(ra) - a)
            for nb in _neighbours(ra):
                dn = abs(Fraction(nb) - a)
                assert d <= dn
                if d == dn:
                    assert struct.unpack("<I", struct.pack("<f", ra))[0] % 2 == 0


def test_hand_cases():
    u = 2.0 ** -24                       # half an ulp of 1.0 in binary32
    cases = [([1.0, u], 1.0),            # tie -> even (1.0)
             ([1.0, u, u], 1.0 + 2 * u),  # exact 1 + 2^-23, whereas ((1 + u) + u) = 1 in binary32
             ([1.0 + 2 * u, u], 1.0 + 4 * u),   # tie, 1 + 2^-23 has an odd significand -> up
             ([1.0, -1.0, u], u),
             ([-0.0, -0.0], 0.0),
             ([3.0 * 2.0 ** 126, 3.0 * 2.0 ** 126], math.inf),
             ([2.0 ** -149, 2.0 ** -149, 2.0 ** -150 * 0], 2.0 ** -148)]
    for xs, want in cases:
        got = float(correctly_rounded_sum_f32([np.array([f32(v)], dtype=np.float32) for v in xs])[0])
        assert got == want and math.copysign(1, got) == math.copysign(1, want), (xs, got, want)
    # the sequential binary32 association differs from it on the second case
    assert f32(f32(1.0 + u) + u) == 1.0


def test_integer_inputs_give_the_integer_sum():
    rng = np.random.default_rng(3)
    x = rng.integers(-(1 << 20), 1 << 20, size=(8, 5000)).astype(np.float32)
    assert np.array_equal(correctly_rounded_sum_f32(list(x)), x.astype(np.int64).sum(axis=0).astype(np.float32))


def test_round_fraction_overflow_and_subnormal():
    assert round_fraction_to_f32(Fraction(2) ** 128) == math.inf
    assert round_fraction_to_f32(-(Fraction(2) ** 128 - Fraction(2) ** 103)) == -math.inf   # tie -> even = 2^128
    assert round_fraction_to_f32(Fraction(2) ** 128 - Fraction(2) ** 103 - 1) == f32(3.4028234663852886e38)
    assert round_fraction_to_f32(Fraction(1, 2 ** 150)) == 0.0                           # tie -> even (0)
    assert round_fraction_to_f32(Fraction(3, 2 ** 151)) == 2.0 ** -149


def test_rejects_non_finite():
    with pytest.raises(ValueError):
        correctly_rounded_sum_f32([np.array([np.inf], np.float32), np.array([1.0], np.float32)])


def test_nvls_avg_is_the_rounded_quotient_of_the_rounded_sum():
    """NVLS AVG (fp32; readings NV2 + AV1): oracle.simulate of a switch_reduce plan with op
    "avg" gives every element as round(round(Σx)/N) — checked element by element against the
    quotient of exact rationals rounded with round_fraction_to_f32 (N = 3, 5: non-powers of two,
    where the division rounds), against Σ × 1/N exactly for N = 4 (a power of two, normal range),
    and N equal inputs average to the input."""
    from oracle import plans as OP
    from oracle import simulate as SM
    rng = np.random.default_rng(7)
    for n in (3, 4, 5):
        count = 3000
        x = wide_random(rng, n, count, 20)
        plan = OP.Plan(n, count, [], True)
        got = SM.simulate(plan, list(x), "f32", op="avg")[0]
        s = correctly_rounded_sum_f32(list(x))
        for i in range(0, count, 7):
            want = round_fraction_to_f32(Fraction(float(s[i])) / n)
            assert struct.pack("<f", got[i]) == struct.pack("<f", want) or (got[i] == 0 and want == 0), (n, i)
        if n == 4:
            normal = np.abs(s) >= np.float32(2.0 ** -124)
            assert np.array_equal(got[normal], (s[normal] * np.float32(0.25)).astype(np.float32))
    same = np.full(64, np.float32(1.375), dtype=np.float32)
    for n in (3, 6):
        got = SM.simulate(OP.Plan(n, 64, [], True), [same] * n, "f32", op="avg")
        assert all(np.array_equal(g, same) for g in got)
