"""Pins for the oracle's quantiser (a1) -- checked against things other than the oracle itself.

* closed form for integers: v = q*s + r, code = q + [2r > s or (2r == s and q odd)]   (exhaustive)
* exact rationals: Python's round() on a Fraction is round-half-even of the exact quotient
* the invariant |x - code*s| <= eb that the paper's quantiser guarantees for every voxel
* the hand-evaluated worked example in tests/golden/spec_examples.json
"""
import json
import os
from fractions import Fraction

import numpy as np
import pytest

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def test_worked_example_eb2(oracle_mod):
    g = GOLD["quantize_u16_eb2"]
    codes = oracle_mod.quantize(np.array(g["x"], np.uint16), g["eb"])
    assert codes.tolist() == g["codes"]


@pytest.mark.parametrize("s", [1, 2, 3, 4, 5, 6, 7, 8, 10, 12, 16, 100, 255, 1000, 4095, 40000])
def test_u16_exhaustive_integer_closed_form(oracle_mod, s):
    v = np.arange(65536, dtype=np.uint16)
    codes = oracle_mod.quantize(v, s / 2.0).astype(np.int64)
    q, r = np.divmod(v.astype(np.int64), s)
    up = (2 * r > s) | ((2 * r == s) & (q % 2 == 1))
    np.testing.assert_array_equal(codes, q + up)
    # P:348 output contract |Q - D| <= E_abs, here with E_abs = eb = s/2
    assert np.all(np.abs(v.astype(np.int64) * 2 - codes * 2 * s) <= s)


@pytest.mark.parametrize("eb", [0.5, 0.75, 1.25, 2.5, 3.3])
def test_u16_fractional_step_vs_fraction(oracle_mod, eb):
    s = Fraction(float(np.float32(2 * eb)))
    v = np.arange(0, 65536, 7, dtype=np.uint16)
    codes = oracle_mod.quantize(v, eb)
    ref = [round(Fraction(int(a)) / s) for a in v]   # round() on Fraction = half-even, exact
    assert codes.astype(np.int64).tolist() == ref


def _fraction_rne(x, s):
    return round(Fraction(float(x)) / Fraction(float(s)))


def test_f32_random_vs_exact_rational(oracle_mod):
    rng = np.random.default_rng(7)
    x = np.concatenate([rng.normal(0.5, 0.4, 20000), rng.uniform(-3, 3, 20000)]).astype(np.float32)
    for eb in [np.float32(1.3e-3), np.float32(0.01), np.float32(0.37)]:
        s = np.float32(2 * eb)
        codes = oracle_mod.quantize(x, eb)
        ref = [_fraction_rne(a, s) for a in x]
        assert codes.astype(np.int64).tolist() == ref
        err = np.abs(x.astype(np.float64) - codes.astype(np.float64) * np.float64(s))
        assert np.all(err <= np.float64(eb))          # exact: products of fp32 values fit fp64


def test_f32_exact_ties_go_to_even(oracle_mod):
    # x = (k + 1/2) * s exactly representable: s a power of two times a small odd integer
    s = np.float32(0.0078125 * 3)          # 3 * 2^-7
    k = np.arange(-200, 200)
    x = ((k + 0.5) * np.float64(s)).astype(np.float32)
    assert all(Fraction(float(a)) / Fraction(float(s)) == Fraction(int(2 * kk + 1), 2) for a, kk in zip(x, k))
    codes = oracle_mod.quantize(x, s / np.float32(2)).astype(np.int64)
    assert np.all(codes % 2 == 0)
    assert np.all(np.abs(codes - (k + 0.5)) == 0.5)


def test_f32_near_ties_not_rounded_twice(oracle_mod):
    # quotients a hair above/below k+1/2 whose fp32 quotient rounds onto k+1/2 (G-4)
    rng = np.random.default_rng(3)
    s = np.float32(2.6e-3)
    k = rng.integers(-500, 500, 4000)
    base = ((k + 0.5) * np.float64(s)).astype(np.float32)
    x = np.concatenate([np.nextafter(base, np.float32(np.inf)), np.nextafter(base, np.float32(-np.inf)), base])
    codes = oracle_mod.quantize(x, s / np.float32(2)).astype(np.int64)
    ref = [_fraction_rne(a, s) for a in x]
    assert codes.tolist() == ref


def test_range_limits(oracle_mod):
    with pytest.raises(oracle_mod.OracleError):       # |x/s| >= 2^23 rejected (G-4)
        oracle_mod.quantize(np.array([2.0 ** 23], np.float32), 0.5)
    oracle_mod.quantize(np.array([2.0 ** 23 - 1], np.float32), 0.5)
    with pytest.raises(oracle_mod.OracleError):       # u16 codes must fit u16 (G-7)
        oracle_mod.quantize(np.array([65535], np.uint16), 0.25)
    with pytest.raises(oracle_mod.OracleError):       # eb > 0 (G-5)
        oracle_mod.quantize(np.array([1], np.uint16), 0.0)
    with pytest.raises(oracle_mod.OracleError):       # non-finite (G-32)
        oracle_mod.quantize(np.array([np.nan], np.float32), 1.0)


def test_range_and_relative_eb(oracle_mod):
    rng = np.random.default_rng(1)
    x = rng.normal(0, 1, 1000).astype(np.float32)
    assert oracle_mod.value_range(x) == (x.min(), x.max())
    x[17] = np.inf
    with pytest.raises(oracle_mod.OracleError):
        oracle_mod.value_range(x)
    # G-6 example: range [0, 1], rel 1e-3 -> eb = fl32(1e-3)
    assert oracle_mod.resolve_eb(0.0, 1.0, 1e-3) == float(np.float32(1e-3))


def _round_f32(fr):
    """Correctly rounded binary32 (ties to even) of a positive rational, by exact comparison with the
    neighbouring binary32 values."""
    from fractions import Fraction

    f = np.float32(float(fr))
    cands = [np.nextafter(f, np.float32(-np.inf)), f, np.nextafter(f, np.float32(np.inf))]
    dist = [abs(Fraction(float(c)) - fr) for c in cands]
    best = min(dist)
    ties = [c for c, d in zip(cands, dist) if d == best]
    if len(ties) > 1:
        ties = [c for c in ties if int(np.float32(c).view(np.uint32)) % 2 == 0]
    return float(ties[0])


@pytest.mark.parametrize("mn,mx", [(-0.24847662448883057, 1.5229978561401367),
                                   (0.20228619873523712, 0.5688977837562561),
                                   (0.03421112149953842, 1.8453582525253296)])
def test_resolve_eb_is_fp64_then_fp32(oracle_mod, mn, mx):
    """G-6: eb = fl32(rel * (fl64(max) - fl64(min))) with rel = 1e-3 as a binary64 value.  The expected
    value is the exact rational product rounded once to binary32 (Fractions), on ranges where
    evaluating the product in binary32 arithmetic gives a different eb -- so an fp32 implementation
    (or a dropped term) fails here."""
    from fractions import Fraction

    mn32, mx32 = np.float32(mn), np.float32(mx)
    exact = Fraction(1e-3) * (Fraction(float(mx32)) - Fraction(float(mn32)))
    want = _round_f32(exact)
    assert oracle_mod.resolve_eb(float(mn32), float(mx32), 1e-3) == want
    naive = float(np.float32(np.float32(1e-3) * (mx32 - mn32)))
    assert naive != want
