"""Pins for oracle.simulate, oracle.theorems, oracle.fit and synth.generator (CPU only).

Pins: integer-valued inputs make every partial sum exact, so any plan must return the int64
sum (closed form, order independent); an independent scalar simulator (struct-rounded
binary32) must agree bitwise with the numpy one on tiny cases (brute force); summation
order of CPS/Ring written out by hand from P:141/P:143 and Q1; bf16 RNE textbook cases;
Q21 accuracy bounds; A000311 tree counts and Eq. 12-14 / Theorems 1-2 by enumeration;
fig:calc trend lines recovered by the Eq. 6 fit; fit round trips.
"""
import numpy as np
import pytest

from oracle import fit as FT
from oracle import plans as P
from oracle import simulate as SM
from oracle import theorems as TH
from synth import generator as GEN

KINDS8 = ["cps", "ring", "rhd", "rb", "hcps:4,2", "hcps:2,4", "hcps:2,2,2"]


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("kind", KINDS8)
def test_integer_inputs_exact_sum(kind, dtype):
    n, count = 8, 1000
    xs = GEN.generate_all(7, n, count, dtype, "integer")
    plan = P.build_plan(kind, n, count)
    out = SM.simulate(plan, xs, dtype)
    ref = sum(GEN.as_f64(x, dtype).astype(np.int64) for x in xs)
    for r in range(n):
        assert np.array_equal(GEN.as_f64(out[r], dtype).astype(np.int64), ref)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("mode", ["gradient", "specials"])
@pytest.mark.parametrize("kind,n", [("cps", 2), ("cps", 4), ("ring", 3), ("ring", 4),
                                    ("rhd", 4), ("rhd", 3), ("rb", 4), ("hcps:2,2", 4),
                                    ("cps", 3)])
def test_numpy_equals_scalar_bruteforce(kind, n, dtype, mode):
    count = 64 + n - 1
    xs = GEN.generate_all(11, n, count, dtype, mode)
    plan = P.build_plan(kind, n, count)
    a = SM.simulate(plan, xs, dtype)
    b = SM.simulate_scalar(plan, xs, dtype)
    for r in range(n):
        va = a[r].view(np.uint32) if dtype == "f32" else a[r]
        vb = b[r].view(np.uint32) if dtype == "f32" else b[r]
        nan = np.isnan(a[r]) if dtype == "f32" else np.isnan(SM.bf16_bits_to_f32(a[r]))
        assert np.array_equal(va[~nan], vb[~nan])
        nanb = np.isnan(b[r]) if dtype == "f32" else np.isnan(SM.bf16_bits_to_f32(b[r]))
        assert np.array_equal(nan, nanb)


def test_cps_summation_order_by_hand():
    """P:141 + reading Q1: block b = ((x0 + x1) + x2) + x3 in binary32, ascending rank."""
    n, count = 4, 4
    xs = [np.array([1e8, 1.0, -1e8, 3.0], np.float32) for _ in range(n)]
    xs = [np.roll(x, r) for r, x in enumerate(xs)]
    out = SM.simulate(P.build_plan("cps", n, count), xs, "f32")
    for e in range(count):
        acc = np.float32(xs[0][e])
        for q in range(1, n):
            acc = np.float32(acc + xs[q][e])
        assert out[0][e] == acc and out[3][e] == acc


def test_ring_association_by_hand():
    """block b accumulates x_{b-1}, x_b, x_{b+1}, ..., x_{b-2} left to right."""
    n = 5
    rng = np.random.default_rng(3)
    xs = [(rng.standard_normal(n) * 10.0 ** rng.integers(-3, 8, n)).astype(np.float32)
          for _ in range(n)]
    out = SM.simulate(P.build_plan("ring", n, n), xs, "f32")
    for b in range(n):
        order = [(b - 1 + k) % n for k in range(n)]
        acc = np.float32(xs[order[0]][b])
        for q in order[1:]:
            acc = np.float32(acc + xs[q][b])
        assert out[0][b].view(np.uint32) == acc.view(np.uint32)


def test_bf16_rne_textbook():
    cases = {0x3F808000: 0x3F80,   # tie, even stays
             0x3F818000: 0x3F82,   # tie, odd rounds up
             0x3F808001: 0x3F81,   # above half
             0x3F807FFF: 0x3F80,   # below half
             0x7F7FFFFF: 0x7F80,   # overflow to +inf
             0xFF7FFFFF: 0xFF80,
             0x00000001: 0x0000,   # tiny subnormal rounds to +0
             0x80008000: 0x8000,   # -tie at zero, even
             0x7F800000: 0x7F80, 0x00000000: 0x0000}
    x = np.array(list(cases), np.uint32).view(np.float32)
    assert list(SM.f32_to_bf16_rne(x)) == list(cases.values())
    nan = SM.f32_to_bf16_rne(np.array([0xFFC12345], np.uint32).view(np.float32))
    assert np.isnan(SM.bf16_bits_to_f32(nan))[0]


@pytest.mark.parametrize("kind", KINDS8)
def test_accuracy_bounds(kind):
    """North star: rel. error vs float64 <= 1e-6 (fp32) and <= 1e-2 (bf16), norm-wise (Q21)."""
    n, count = 8, 40000
    for dtype, tol in (("f32", 1e-6), ("bf16", 1e-2)):
        xs = GEN.generate_all(GEN.config_seed(4), n, count, dtype)
        out = SM.simulate(P.build_plan(kind, n, count), xs, dtype)
        ref = SM.exact_sum_f64(xs, dtype)
        for r in (0, n - 1):
            assert SM.normwise_rel_err(out[r], ref, dtype) <= tol


@pytest.mark.parametrize("kind", KINDS8)
def test_all_ranks_identical(kind):
    xs = GEN.generate_all(5, 8, 777, "bf16")
    out = SM.simulate(P.build_plan(kind, 8, 777), xs, "bf16")
    assert all(np.array_equal(out[0], o) for o in out)


# ---------------------------------------------------------------- theorems

def test_reduce_tree_counts_a000311():
    assert [len(list(TH.reduce_trees(list(range(n))))) for n in range(2, 7)] == [1, 4, 26, 236, 2752]


@pytest.mark.parametrize("n", range(2, 7))
def test_theorems_bruteforce(n):
    res = TH.check_theorems(n)
    assert res["min_memory"] == (n + 1) / n or float(res["min_memory"]) == (n + 1) / n


# ---------------------------------------------------------------- fitting

def test_eq6_fit_recovers_fig_calc(golden):
    fc = golden["fig_calc"]
    a, b, c1, c2 = FT.fit_eq6(fc["x"], fc["gpu_ms_per_op"])
    assert a == pytest.approx(fc["gpu_trend"]["a"], abs=5e-4)
    assert b == pytest.approx(fc["gpu_trend"]["b"], abs=5e-4)
    a, b, c1, c2 = FT.fit_eq6(fc["x"], fc["cpu_ms_per_op"])
    assert a == pytest.approx(fc["cpu_trend"]["a"], abs=5e-3)
    assert b == pytest.approx(fc["cpu_trend"]["b"], abs=5e-3)
    assert c2 < 0            # reading Q18: the CPU line implies γ < 0


def _rows(alpha, k, delta, eps, wt, noise=0.0, seed=0):
    rng = np.random.default_rng(seed)
    rows = []
    for n in range(2, 17):
        for s in (4e7, 4e8):
            t = FT.cps_forward(n, s, alpha, k, delta, eps, wt)
            rows.append((n, s, t * (1 + noise * rng.standard_normal())))
    return rows


def test_fit_roundtrip_noiseless():
    """Table 5-like params (per byte) recovered exactly from noiseless data."""
    truth = (6.58e-3, 1.34e-9 / 4, 1.87e-10 / 4, 1.22e-10 / 4, 9)
    f = FT.fit_params(_rows(*truth), 2, 16)
    assert f["w_t"] == 9 and f["sse"] < 1e-18
    for key, v in zip(("alpha", "combined", "delta", "epsilon"), truth[:4]):
        assert f[key] == pytest.approx(v, rel=1e-6)


@pytest.mark.slow
def test_fit_noise_1pct():
    """1 % noise, 100 seeds: w_t exact in >= 95; median α and k within 5 %, δ, ε 15 %."""
    truth = (6.58e-3, 1.34e-9 / 4, 1.87e-10 / 4, 1.22e-10 / 4, 9)
    hits, errs = 0, {k: [] for k in ("alpha", "combined", "delta", "epsilon")}
    for seed in range(100):
        f = FT.fit_params(_rows(*truth, noise=0.01, seed=seed), 2, 16)
        hits += f["w_t"] == 9
        for key, v in zip(errs, truth[:4]):
            errs[key].append(abs(f[key] - v) / v)
    assert hits >= 95
    assert np.median(errs["alpha"]) < 0.05 and np.median(errs["combined"]) < 0.05
    assert np.median(errs["delta"]) < 0.15 and np.median(errs["epsilon"]) < 0.15


def test_split_combined(spec_examples):
    e = spec_examples["split_combined"]
    beta, gamma = FT.split_combined(e["k"], 1.0 / e["beta"])
    assert beta == pytest.approx(e["beta"]) and gamma == pytest.approx(e["gamma"], rel=1e-9)
    assert FT.split_combined(2e-9, 1e9)[1] == 0.0
    with pytest.raises(ValueError):
        FT.split_combined(1e-9, 1e9)


def test_fit_underdetermined():
    with pytest.raises(ValueError):
        FT.fit_params([(2, 1e6, 1.0), (3, 1e6, 1.1), (4, 1e6, 1.2), (5, 1e6, 1.3)], 2, 5)


# ---------------------------------------------------------------- input generator

def test_splitmix64_known_value():
    """SplitMix64 with state 0: first output 0xE220A8397B1DCDAF (reference implementation)."""
    assert GEN.splitmix64_scalar(0) == 0xE220A8397B1DCDAF
    v = GEN._splitmix64(np.array([0, 1, 12345], np.uint64))
    assert [int(x) for x in v] == [GEN.splitmix64_scalar(x) for x in (0, 1, 12345)]


def test_generator_properties():
    x = GEN.generate(3, 1, 1 << 17, "f32")
    assert np.all(np.abs(x) < 2.0 ** -7) and abs(float(x.mean())) < 1e-4
    assert np.array_equal(x, GEN.generate(3, 1, 1 << 17, "f32"))
    assert not np.array_equal(x, GEN.generate(3, 2, 1 << 17, "f32"))
    assert np.array_equal(GEN.generate(3, 1, 100, "f32", start=500), x[500:600])
    b = GEN.generate(3, 1, 4096, "bf16")
    f = (b.astype(np.uint32) << 16).view(np.float32)
    assert np.all(np.abs(f) <= 2.0 ** -7)
    ints = GEN.generate(9, 0, 5000, "f32", "integer")
    assert np.all(ints == np.round(ints)) and np.abs(ints).max() <= 1024


# ---------------------------------------------------------------- AVG (NEXT #4, reading AV1)

AVG_CASES = [("cps", 4), ("cps", 3), ("ring", 3), ("ring", 5), ("rhd", 4), ("rhd", 3), ("rb", 4),
             ("hcps:2,2", 4), ("hcps:3,2", 6)]


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("kind,n", AVG_CASES)
def test_avg_numpy_equals_scalar_bruteforce(kind, n, dtype):
    count = 40 + n - 1
    xs = GEN.generate_all(13, n, count, dtype, "gradient")
    plan = P.build_plan(kind, n, count)
    a = SM.simulate(plan, xs, dtype, op="avg")
    b = SM.simulate_scalar(plan, xs, dtype, op="avg")
    for r in range(n):
        va = a[r].view(np.uint32) if dtype == "f32" else a[r]
        vb = b[r].view(np.uint32) if dtype == "f32" else b[r]
        assert np.array_equal(va, vb)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("kind,n", AVG_CASES)
def test_avg_of_identical_inputs_is_the_input(kind, n, dtype):
    """The mean of N equal integer values is that value, exactly, on every rank."""
    count = 50 + n
    x = GEN.generate_all(17, 1, count, dtype, "integer")[0]
    out = SM.simulate(P.build_plan(kind, n, count), [x.copy() for _ in range(n)], dtype, op="avg")
    for r in range(n):
        assert np.array_equal(out[r], x)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("kind", KINDS8)
def test_avg_pow2_is_sum_scaled_once(kind, dtype):
    """N = 8: division by 2^3 is exact and commutes with RNE (no under/overflow here), so the
    AVG result is the SUM result times 1/8 — dividing twice or never would fail."""
    n, count = 8, 333
    xs = GEN.generate_all(19, n, count, dtype, "gradient")
    plan = P.build_plan(kind, n, count)
    s = SM.simulate(plan, xs, dtype)
    a = SM.simulate(plan, xs, dtype, op="avg")
    for r in range(n):
        assert np.array_equal(GEN.as_f64(a[r], dtype), GEN.as_f64(s[r], dtype) / 8)


def test_avg_simulate_at_matches_simulate():
    n, count = 5, 1001
    xs = GEN.generate_all(23, n, count, "bf16", "gradient")
    plan = P.build_plan("ring", n, count)
    full = SM.simulate(plan, xs, "bf16", op="avg")
    idx = np.array([0, 1, 199, 200, 201, 600, 1000])
    part = SM.simulate_at(plan, idx, [x[idx] for x in xs], "bf16", op="avg")
    for r in range(n):
        assert np.array_equal(part[r], full[r][idx])


def test_exact_sum_and_normwise_error_pins():
    """Pins for the accuracy reference (reading Q21), independent of the simulator:
    exact_sum_f64 equals the exact rational sum whenever float64 holds it (fp32 inputs whose
    exponents span < 53 - 24 - log2 N bits: every partial sum exact), checked with Fraction;
    normwise_rel_err on hand values: y = ref·(1 + d) gives |d|; an error orthogonal to ref
    gives ||e|| / ||ref|| (3-4-5 triangle); bf16 bits are widened before the norm; a zero
    reference reports ||y||."""
    from fractions import Fraction
    rng = np.random.default_rng(11)
    xs = [(rng.integers(-2 ** 23, 2 ** 23, 1000) * 2.0 ** rng.integers(-30, -20)).astype(np.float32)
          for _ in range(8)]
    got = SM.exact_sum_f64(xs, "f32")
    for i in range(0, 1000, 37):
        assert Fraction(float(got[i])) == sum(Fraction(float(x[i])) for x in xs)
    ref = np.array([1.0, -2.0, 4.0, 0.5])
    for d in (1e-3, -2.5e-7):
        y = (ref * (1 + d)).astype(np.float32)
        assert SM.normwise_rel_err(y, ref, "f32") == pytest.approx(abs(d), abs=2 ** -23)   # y rounded to fp32
    assert SM.normwise_rel_err(np.array([3.0, 4.0 + 1.0], np.float32), np.array([3.0, 4.0]), "f32") == pytest.approx(0.2)
    assert SM.normwise_rel_err(np.array([3.0, 4.0], np.float32), np.array([3.0, 4.0]), "f32") == 0.0
    bits = np.array([0x3F80, 0x4000], dtype=np.uint16)          # bf16 1.0, 2.0
    assert SM.normwise_rel_err(bits, np.array([1.0, 2.0]), "bf16") == 0.0
    assert SM.normwise_rel_err(bits, np.array([1.0, 1.0]), "bf16") == pytest.approx(1 / np.sqrt(2))
    assert SM.normwise_rel_err(np.array([3.0, 4.0], np.float32), np.zeros(2), "f32") == 5.0
