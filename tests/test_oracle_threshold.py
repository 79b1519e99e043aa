"""Pins for the oracle's histogram, Eq.-1 normalisation and Otsu threshold (a2, a3, a4)."""
import json
import os
from fractions import Fraction

import cv2
import numpy as np
import pytest

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def test_histogram_spec_examples_and_bincount(oracle_mod):
    for ex in GOLD["histogram"]:
        h = oracle_mod.hist_u16(np.array(ex["x"], np.uint16))
        exp = np.zeros(65536, np.uint64)
        for k, v in ex["bins"].items():
            exp[int(k)] = v
        np.testing.assert_array_equal(h, exp)
    x = np.random.default_rng(0).integers(0, 65536, 100000).astype(np.uint16)
    h = oracle_mod.hist_u16(x)
    np.testing.assert_array_equal(h, np.bincount(x, minlength=65536))
    assert int(h.sum()) == x.size
    assert oracle_mod.imax_u16(h) == int(x.max())
    assert oracle_mod.imax_u16(np.zeros(65536, np.uint64)) == GOLD["imax_all_zero"]["i_max"]
    h0 = oracle_mod.hist_u16(np.zeros(5, np.uint16))
    assert oracle_mod.imax_u16(h0) == 1


def test_norm8_spec_examples(oracle_mod):
    for ex in GOLD["norm8"]:
        assert oracle_mod.norm8_u16(ex["v"], ex["i_max"]) == ex["norm8"], ex["cite"]


def _half_up(fr):
    """round_half_up of a non-negative Fraction."""
    return int(fr + Fraction(1, 2)) if fr >= 0 else 0


@pytest.mark.parametrize("imax", [1, 2, 255, 256, 1000, 1023, 4095, 40000, 65535])
def test_norm8_u16_exhaustive_vs_fraction(oracle_mod, imax):
    for v in range(0, imax + 1, max(1, imax // 3000)):
        assert oracle_mod.norm8_u16(v, imax) == _half_up(Fraction(255 * v, imax))


def test_norm8_f32_eq1_within_reading(oracle_mod):
    """G-30 evaluates Eq. 1 once in binary64; it must equal exact round-half-up except where the
    exact value sits within binary64 rounding of a half-integer, and must be monotone in x."""
    rng = np.random.default_rng(5)
    for imax in [np.float32(1.0), np.float32(1.2573), np.float32(0.0371)]:
        x = np.sort(rng.uniform(-0.1, float(imax), 20000).astype(np.float32))
        x = np.concatenate([x, [np.float32(0), imax]])
        got = np.array([oracle_mod.norm8_f32(a, imax) for a in x])
        assert got[-1] == 255 and got[-2] == 0
        assert np.all(np.diff(got[:-2]) >= 0)
        for a, g in zip(x, got):
            fr = Fraction(float(a)) * 255 / Fraction(float(imax))
            exact = min(255, _half_up(fr))
            if g != exact:
                assert abs(fr - int(fr) - Fraction(1, 2)) < Fraction(1, 10 ** 12)


def test_hist8_fold_equals_per_voxel_normalisation(oracle_mod):
    rng = np.random.default_rng(11)
    x = np.concatenate([rng.normal(400, 60, 30000), rng.normal(2500, 80, 9000)]).clip(0, 4095).astype(np.uint16)
    h = oracle_mod.hist_u16(x)
    imax = int(x.max())
    table = np.array([_half_up(Fraction(255 * v, imax)) for v in range(imax + 1)])
    np.testing.assert_array_equal(oracle_mod.hist8_from_u16(h, imax), np.bincount(table[x], minlength=256))


def test_hist8_f32_matches_bincount(oracle_mod):
    rng = np.random.default_rng(12)
    x = rng.uniform(-0.05, 1.3, 5000).astype(np.float32)
    imax = float(x.max())
    per = np.array([oracle_mod.norm8_f32(a, imax) for a in x])
    np.testing.assert_array_equal(oracle_mod.hist8_f32(x, imax), np.bincount(per, minlength=256))


def _spikes(d):
    h = np.zeros(256, np.int64)
    for k, v in d.items():
        h[int(k)] = v
    return h


def test_otsu_spec_examples(oracle_mod):
    for ex in GOLD["otsu"]:
        h = _spikes(ex["spikes"])
        if ex["t"] is None:
            with pytest.raises(oracle_mod.Degenerate):
                oracle_mod.otsu2(h)
        else:
            assert oracle_mod.otsu2(h) == ex["t"], ex["cite"]
    with pytest.raises(oracle_mod.Degenerate):
        oracle_mod.otsu2(np.zeros(256, np.int64))


def _dform_argmax(h):
    """An algebraically different statement of the same maximiser: with D = N*s0 - n0*S the
    between-class variance is D^2 / (N^2 n0 n1); compare D_a^2 n0b n1b vs D_b^2 n0a n1a in ints."""
    h = [int(v) for v in h]
    N, S = sum(h), sum(k * v for k, v in enumerate(h))
    best = None
    n0 = s0 = 0
    for t in range(255):
        n0 += h[t]
        s0 += t * h[t]
        n1 = N - n0
        if n0 == 0 or n1 == 0:
            continue
        D = N * s0 - n0 * S
        if best is None or D * D * best[1] > best[0] * n0 * n1:
            best = (D * D, n0 * n1, t)
    return best[2]


def test_otsu_vs_integer_dform_random(oracle_mod):
    rng = np.random.default_rng(21)
    for trial in range(60):
        h = np.zeros(256, np.int64)
        kind = trial % 3
        if kind == 0:
            h[rng.integers(0, 256, 3)] = rng.integers(1, 50, 3)       # sparse: many exact ties
        elif kind == 1:
            h = rng.integers(0, 5, 256)
        else:
            a = rng.normal(rng.uniform(20, 100), 10, 3000)
            b = rng.normal(rng.uniform(140, 230), 15, 1000)
            h = np.bincount(np.clip(np.concatenate([a, b]), 0, 255).astype(int), minlength=256)
        if np.count_nonzero(h) < 2:
            continue
        assert oracle_mod.otsu2(h) == _dform_argmax(h)


def test_otsu_vs_opencv(oracle_mod):
    """cv2.threshold(THRESH_OTSU) returns the smallest maximiser; it is float, so only well-separated
    maxima are compared."""
    rng = np.random.default_rng(4)
    compared = 0
    for trial in range(40):
        a = rng.normal(rng.uniform(20, 90), rng.uniform(5, 20), 4000)
        b = rng.normal(rng.uniform(130, 230), rng.uniform(5, 25), int(rng.integers(500, 4000)))
        img = np.clip(np.concatenate([a, b]), 0, 255).astype(np.uint8).reshape(1, -1)
        h = np.bincount(img.ravel(), minlength=256)
        t = oracle_mod.otsu2(h)
        var = [oracle_mod.otsu.between_class_variance([int(v) for v in h], k) or 0 for k in range(255)]
        top = sorted(set(var))[-2:]
        if len(top) == 2 and (top[1] - top[0]) / top[1] < 1e-9:
            continue
        tcv, _ = cv2.threshold(img, 0, 255, cv2.THRESH_BINARY + cv2.THRESH_OTSU)
        assert t == int(tcv)
        compared += 1
    assert compared > 30


def test_otsu_reflection_and_scale_invariance(oracle_mod):
    rng = np.random.default_rng(9)
    for _ in range(20):
        h = rng.integers(0, 40, 256) * (rng.random(256) < 0.6)
        if np.count_nonzero(h) < 2:
            continue
        t = oracle_mod.otsu2(h)
        assert oracle_mod.otsu2(h * 7) == t
        # reflecting the histogram reflects the unique maximiser
        var = [oracle_mod.otsu.between_class_variance([int(v) for v in h], k) for k in range(255)]
        vmax = max(v for v in var if v is not None)
        if sum(1 for v in var if v == vmax) == 1:
            assert oracle_mod.otsu2(h[::-1]) == 254 - t


def test_binarize_spec_examples(oracle_mod):
    for ex in GOLD["binarize"]:
        m = oracle_mod.binarize(np.array(ex["x"], np.uint16), 255, ex["t"], 0)   # I_max 255: identity norm8
        assert m.tolist() == ex["mask"], ex["cite"]
        low = oracle_mod.binarize(np.array(ex["x"], np.uint16), 255, ex["t"], 1)
        assert low.tolist() == [1 - v for v in ex["mask"]]


def test_binarize_f32_spec_examples_and_edges(oracle_mod):
    """fp32 binarisation (Eq. 2 on Eq. 1's norm8 with round-half-up, G-30), pinned by hand:
    with I_max = 255 norm8 is the identity on integers, so S:182-183 apply to fp32 input; a voxel
    exactly on a norm8 edge (x = 10.5: 10.5 * 255 / 255 = 10.5 rounds up to 11) and one just below
    it; I_max = 510 (x = 21 -> 21 * 255 / 510 = 10.5 -> 11); 'norm8 > t8' is strict (x = 10 with
    t8 = 10 is out); LOW polarity is the complement."""
    x = np.array([0.0, 10.0, 200.0], np.float32)
    assert oracle_mod.binarize(x, 255.0, 10, 0).tolist() == [0, 0, 1]
    assert oracle_mod.binarize(x, 255.0, 255, 0).tolist() == [0, 0, 0]
    assert oracle_mod.binarize(x, 255.0, 10, 1).tolist() == [1, 1, 0]          # LOW: the complement
    below = np.nextafter(np.float32(10.5), np.float32(0))
    e = np.array([10.5, below, 11.0, 9.75], np.float32)
    assert oracle_mod.binarize(e, 255.0, 10, 0).tolist() == [1, 0, 1, 0]
    e2 = np.array([21.0, np.nextafter(np.float32(21.0), np.float32(0)), 20.0, 22.0], np.float32)
    assert oracle_mod.binarize(e2, 510.0, 10, 0).tolist() == [1, 0, 0, 1]
