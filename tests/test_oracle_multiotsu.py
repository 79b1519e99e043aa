"""Pins of the NEXT-3 multi-Otsu oracle (oracle.multi_otsu; "multi-Otsu adaptive
thresholding", AC4 S:565).

Anchors: the SPEC examples, closed forms for separated spikes, k = 2 against otsu2 (itself
pinned by OpenCV's THRESH_OTSU in test_oracle_threshold.py), Otsu's equivalence sigma_T^2 = sigma_W^2 +
sigma_B^2 (the maximiser of the between-class variance is the minimiser of the within-class
variance, computed here from the pixel values themselves), and reflection / scale invariance.
"""
from fractions import Fraction

import numpy as np
import pytest

import oracle


def _h(pairs):
    h = [0] * 256
    for v, c in pairs:
        h[v] += c
    return h


def test_spec_examples():
    assert oracle.multi_otsu(_h([(10, 50), (200, 50)]), 2) == (10,)            # S:173 smallest maximiser
    assert oracle.multi_otsu(_h([(0, 7), (128, 7), (255, 7)]), 3) == (0, 128)  # S:174 spikes separated
    with pytest.raises(oracle.Degenerate):
        oracle.multi_otsu(_h([(77, 100)]), 2)
    with pytest.raises(oracle.Degenerate):
        oracle.multi_otsu(_h([(3, 5), (90, 5)]), 3)


def test_three_spikes_closed_form():
    """Three populated bins a < b < c: the only tuples with non-empty classes put t1 in [a, b) and t2 in
    [b, c); all give the same variance, so the answer is (a, b) whatever the counts."""
    rng = np.random.default_rng(4)
    for _ in range(20):
        a, b, c = sorted(rng.choice(256, 3, replace=False))
        h = _h([(a, int(rng.integers(1, 10 ** 6))), (b, int(rng.integers(1, 10 ** 6))), (c, int(rng.integers(1, 10 ** 6)))])
        assert oracle.multi_otsu(h, 3) == (a, b)


def test_k2_equals_otsu2():
    rng = np.random.default_rng(8)
    for _ in range(20):
        h = list(rng.integers(0, 1000, 256) * (rng.random(256) < 0.5))
        if sum(1 for v in h if v) < 2:
            continue
        assert oracle.multi_otsu(h, 2) == (oracle.otsu2(h),)


def _within_class_argmin(values, classes):
    """Brute force from the pixels: the lexicographically smallest ascending tuple minimising
    sum_k sum_{p in class k} (p - mean_k)^2 over tuples with non-empty classes."""
    vals = np.sort(np.asarray(values, np.int64))
    best, best_t = None, None
    cand = range(255)
    tuples = [(t,) for t in cand] if classes == 2 else [(a, b) for a in cand for b in cand if a < b]
    for ts in tuples:
        edges = [-1] + list(ts) + [255]
        w = Fraction(0)
        ok = True
        for lo, hi in zip(edges[:-1], edges[1:]):
            cls = vals[(vals > lo) & (vals <= hi)]
            if cls.size == 0:
                ok = False
                break
            m = Fraction(int(cls.sum()), int(cls.size))
            w += sum(Fraction(int(c)) * (Fraction(int(p)) - m) ** 2 for p, c in zip(*np.unique(cls, return_counts=True)))
        if ok and (best is None or w < best):
            best, best_t = w, ts
    return best_t


@pytest.mark.parametrize("seed", range(3))
def test_within_class_equivalence(seed):
    rng = np.random.default_rng(100 + seed)
    nb = int(rng.integers(4, 9))                       # few distinct values keep the brute force small
    levels = np.sort(rng.choice(256, nb, replace=False))
    values = np.repeat(levels, rng.integers(1, 40, nb))
    h = np.bincount(values, minlength=256)
    assert oracle.multi_otsu(h, 3) == _within_class_argmin(values, 3)
    assert oracle.multi_otsu(h, 2) == _within_class_argmin(values, 2)


def test_reflection_and_scale():
    rng = np.random.default_rng(12)
    done = 0
    while done < 4:
        h = list(rng.integers(1, 500, 256))   # every bin populated: no two tuples give the same classes
        t1, t2 = oracle.multi_otsu(h, 3)
        r1, r2 = oracle.multi_otsu(h[::-1], 3)
        # bins i -> 255 - i: classes [0..t1], (t1..t2], (t2..255] become thresholds 254 - t2, 254 - t1
        # (a unique maximiser maps to a unique maximiser; random dense histograms have one)
        assert (r1, r2) == (254 - t2, 254 - t1)
        assert oracle.multi_otsu([3 * v for v in h], 3) == (t1, t2)
        done += 1
