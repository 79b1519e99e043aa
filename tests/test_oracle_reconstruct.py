"""Pins of the NEXT-4 oracle (oracle/reconstruct.py): decode / reconstruction (SPEC
S:359-367), confusion counts and the overlap metrics of Eqs. 7-14.

Anchors other than the oracle itself: the SPEC worked examples and golden values (S:429-431,
S:438-440; acceptance criterion 6), scikit-learn's independent implementations of
F1 (= DSC), Jaccard (= IoU), recall, accuracy, Cohen's kappa and ROC AUC of a binary score, exact
rational arithmetic (Fraction) for every rounding the decode does, and brute force.
"""
from fractions import Fraction

import numpy as np
import pytest
from sklearn import metrics as skm

import oracle

NAN_OK = dict(equal_nan=True, rtol=0, atol=1e-12)


# ------------------------------------------------------------------------ confusion, metrics
def test_confusion_spec_examples():
    n = 100
    k = np.zeros(n, bool)
    k[[3, 17, 42]] = True
    assert oracle.confusion(k, k) == (3, 0, 0, n - 3)
    assert oracle.confusion(np.ones(n, bool), np.zeros(n, bool)) == (0, n, 0, 0)
    pred = np.zeros((10, 10), bool)
    truth = np.zeros((10, 10), bool)
    pred.flat[0:10] = True                                                   # overlap 5, pred-only 5
    truth.flat[5:15] = True                                                  # truth-only 5
    assert oracle.confusion(pred, truth) == (5, 5, 5, 85)


def test_metrics_golden_values():
    m = oracle.overlap_metrics(tp=40, fp=10, fn=10, tn=40)                   # S:438, AC6
    assert abs(m["accuracy"] - 0.8) <= 1e-12
    assert abs(m["kappa"] - 0.6) <= 1e-12
    assert abs(m["auc"] - 0.8) <= 1e-12
    m = oracle.overlap_metrics(tp=7, fp=0, fn=0, tn=93)                      # S:439 perfect prediction
    assert all(v == 1.0 for v in m.values())
    m = oracle.overlap_metrics(tp=5, fp=5, fn=5, tn=85)
    assert m["dsc"] == 0.5 and abs(m["iou"] - 1 / 3) <= 1e-15


def test_metrics_undefined_are_nan():
    m = oracle.overlap_metrics(0, 0, 0, 50)          # empty prediction and truth
    for k in ("dsc", "iou", "sensitivity", "kappa", "auc"):
        assert np.isnan(m[k]), k
    assert m["specificity"] == 1.0 and m["accuracy"] == 1.0
    m = oracle.overlap_metrics(0, 0, 0, 0)
    assert all(np.isnan(v) for v in m.values())


@pytest.mark.parametrize("seed", range(4))
def test_metrics_vs_sklearn(seed):
    """Eqs. 7-14 against scikit-learn's own definitions on random masks of varied balance."""
    rng = np.random.default_rng(seed)
    for _ in range(25):
        n = int(rng.integers(2, 400))
        truth = rng.random(n) < rng.uniform(0.05, 0.95)
        pred = np.where(rng.random(n) < rng.uniform(0.0, 0.6), ~truth, truth)
        if truth.all() or (~truth).all():
            continue
        m = oracle.overlap_metrics(*oracle.confusion(pred, truth))
        ref = {"dsc": skm.f1_score(truth, pred),
               "iou": skm.jaccard_score(truth, pred),
               "sensitivity": skm.recall_score(truth, pred),
               "specificity": skm.recall_score(truth, pred, pos_label=False),
               "accuracy": skm.accuracy_score(truth, pred),
               "kappa": skm.cohen_kappa_score(truth, pred),
               "auc": skm.roc_auc_score(truth, pred.astype(np.float64))}
        for k, v in ref.items():
            np.testing.assert_allclose(m[k], v, **NAN_OK, err_msg=k)


def test_dsc_iou_identity():
    """AC6: dsc = 2 iou / (1 + iou) on 1000 random masks, to 1e-12."""
    rng = np.random.default_rng(7)
    for _ in range(1000):
        n = int(rng.integers(1, 200))
        pred, truth = rng.random(n) < rng.random(), rng.random(n) < rng.random()
        m = oracle.overlap_metrics(*oracle.confusion(pred, truth))
        if np.isnan(m["iou"]):
            assert np.isnan(m["dsc"])
            continue
        assert abs(m["dsc"] - 2 * m["iou"] / (1 + m["iou"])) <= 1e-12


def test_spatial_reduction_examples():
    assert oracle.spatial_reduction(100 * 100, 100 * 100) == 1.0             # S:465 full frame
    assert oracle.spatial_reduction(100 * 100, 2500) == 4.0
    assert np.isnan(oracle.spatial_reduction(100, 0))


# ------------------------------------------------------------------------ decode value
def _nearest_int_half_even(fr):
    return round(fr)   # Fraction.__round__: nearest integer, ties to even


@pytest.mark.parametrize("eb", [0.5, 1.0, 2.0, 3.0, 4.0, 1000.0])
def test_decode_u16_integer_step_exhaustive(eb):
    """Every uint16 value, quantised and decoded: x^ is the multiple of s nearest to x (ties: the even
    multiple), clamped to 65535, so |x - x^| <= eb; s = 1 (eb = 1/2) is lossless (AC3)."""
    x = np.arange(65536, dtype=np.uint16)
    s = oracle.step(eb)
    xh = oracle.decode_value(oracle.quantize(x, eb), s, np.uint16).astype(np.int64)
    xi = x.astype(np.int64)
    k = xi // int(s)
    lo, hi = k * int(s), (k + 1) * int(s)
    dlo, dhi = xi - lo, hi - xi
    want = np.where(dlo < dhi, lo, np.where(dhi < dlo, hi, np.where(k % 2 == 0, lo, hi)))
    np.testing.assert_array_equal(xh, np.minimum(want, 65535))
    assert np.all(np.abs(xi - xh) <= eb)
    if eb == 0.5:
        np.testing.assert_array_equal(xh, xi)


@pytest.mark.parametrize("eb", [0.3, 0.75, 1.25, 2.6])
def test_decode_u16_fractional_step(eb):
    """Non-integer s: x^ = nearest integer to the exact rational code * s, ties to even (G-37); the
    bound becomes eb + 1/2."""
    s = oracle.step(eb)
    codes = np.arange(0, 65536, 97, dtype=np.uint16)
    xh = oracle.decode_value(codes, s, np.uint16)
    for c, v in zip(codes, xh):
        assert int(v) == min(65535, _nearest_int_half_even(Fraction(int(c)) * Fraction(s)))
    x = np.arange(0, min(65536, int(65535 * s)), 13, dtype=np.uint16)   # codes must fit in 16 bits (G-4)
    back = oracle.decode_value(oracle.quantize(x, eb), s, np.uint16).astype(np.float64)
    assert np.all(np.abs(back - x) <= eb + 0.5)


def _nearest_f32(fr):
    """The float32 nearest to the rational fr, ties to an even significand (brute force over the
    neighbours of a candidate)."""
    c = np.float32(float(fr))
    cands = [np.nextafter(c, np.float32(-np.inf)), c, np.nextafter(c, np.float32(np.inf))]
    best = min(cands, key=lambda f: (abs(Fraction(float(f)) - fr),
                                     int(np.array(f, np.float32).view(np.uint32)) & 1))
    return best


def test_decode_f32_correct_rounding():
    rng = np.random.default_rng(3)
    for s in (oracle.step(1e-3), oracle.step(0.37), oracle.step(3.0e-7), oracle.step(12.5)):
        codes = np.concatenate([rng.integers(-(1 << 23), 1 << 23, 400), [0, 1, -1, (1 << 23), -(1 << 23)]])
        codes = codes.astype(np.int32)
        xh = oracle.decode_value(codes, s, np.float32)
        for c, v in zip(codes, xh):
            assert v == _nearest_f32(Fraction(int(c)) * Fraction(s)), (c, s)


def test_decode_f32_round_trip_bound():
    rng = np.random.default_rng(5)
    x = (rng.standard_normal(20000) * 3).astype(np.float32)
    eb = 1e-2
    s = oracle.step(eb)
    back = oracle.decode_value(oracle.quantize(x, eb), s, np.float32).astype(np.float64)
    # |x - code s| <= s / 2 exactly; the fp32 product adds at most half an ulp of x^
    ulp = np.spacing(np.abs(back).astype(np.float32)).astype(np.float64)
    assert np.all(np.abs(back - x) <= s / 2 + ulp / 2)


# ------------------------------------------------------------------------ mask / span forms
def _decode_mask_brute(K, codes, s, dtype):
    out = np.zeros(K.size, dtype)
    j = 0
    for i, k in enumerate(K.reshape(-1)):
        if k:
            out[i] = oracle.decode_value(np.array([codes[j]]), s, dtype)[0]
            j += 1
    return out.reshape(K.shape)


@pytest.mark.parametrize("dtype", [np.uint16, np.float32])
def test_decode_mask_brute_and_round_trip(dtype):
    rng = np.random.default_rng(11)
    shape = (3, 7, 45)
    x = (rng.integers(0, 4000, shape).astype(np.uint16) if dtype == np.uint16
         else rng.standard_normal(shape).astype(np.float32))
    K = (rng.random(shape) < 0.4).astype(np.uint8)
    eb = 2.0 if dtype == np.uint16 else 1e-3
    codes = oracle.extract(x, K, eb)
    s = oracle.step(eb)
    xh = oracle.decode_mask(K, codes, s, dtype)
    np.testing.assert_array_equal(xh, _decode_mask_brute(K, codes, s, dtype))
    assert np.all(xh[K == 0] == 0)
    d = np.abs(xh.astype(np.float64) - x.astype(np.float64))[K == 1]
    if dtype == np.uint16:
        assert np.all(d <= eb)
    else:
        assert np.all(d <= s / 2 + np.spacing(np.abs(xh[K == 1])).astype(np.float64) / 2)


def test_decode_spans_examples():
    # S:364 empty bundle -> the (zero) background exactly
    out = oracle.decode_spans(np.zeros((0, 3), np.int64), np.zeros(0, np.uint16), (2, 3, 5), 1.0, np.uint16)
    assert out.shape == (2, 3, 5) and not out.any()
    # S:365 analogue: s = 1 (eb = 1/2), u16 -> the spans' columns come back bit-exactly, the rest 0
    rng = np.random.default_rng(2)
    x = rng.integers(1, 60000, (4, 6, 37)).astype(np.uint16)
    K = np.zeros(x.shape, np.uint8)
    K[1, 2, 5:9] = 1
    K[1, 2, 20] = 1
    K[3, 0, 0] = 1
    K[3, 5, 36] = 1
    spans, codes = oracle.row_spans(x, K, 0.5)
    xh = oracle.decode_spans(spans, codes, x.shape, oracle.step(0.5), np.uint16)
    cover = np.zeros(x.shape, bool).reshape(-1, x.shape[2])
    for i, xs, xe in spans:
        cover[i, xs:xe] = True
    cover = cover.reshape(x.shape)
    np.testing.assert_array_equal(xh[cover], x[cover])
    assert not xh[~cover].any()
    assert np.all(cover[K == 1])                     # spans re-rasterise to a superset of K
    assert cover[1, 2, 5:21].all() and cover.sum() == 16 + 1 + 1


def test_decode_spans_slab_rows():
    """Records carry global rows; a slab starting at plane z0 subtracts row0 = z0 * Y."""
    spans = np.array([[7, 1, 3], [9, 0, 2]], np.int64)     # Y = 3: rows 7, 9 = planes 2, 3
    codes = np.array([5, 6, 7, 8], np.uint16)
    out = oracle.decode_spans(spans, codes, (2, 3, 4), 2.0, np.uint16, row0=6)
    want = np.zeros((6, 4), np.uint16)
    want[1, 1:3] = [10, 12]
    want[3, 0:2] = [14, 16]
    np.testing.assert_array_equal(out.reshape(6, 4), want)
