"""NEXT-4 oracle: reconstruction (decode / scatter) and ROI quality metrics -- TEST INFRASTRUCTURE ONLY.

Plain numpy / exact-rational statements, one voxel or one record at a time in the order the paper
and SPEC describe them.  Shares nothing with the product.

* decode_value   x^ = code * s, s = fl32(2 eb) (the inverse of a1, G-3), brought to the input dtype:
                 uint16 -> round half to even of the exact product, clamped to [0, 65535];
                 fp32   -> fl32(code) * s rounded once to fp32 (reading G-37)
* decode_mask    the ★ representation (a8: packed K + dense code stream in increasing i) scattered
                 back onto a zero canvas
* decode_spans   the paper's reconstruction: start from a zero raster, for
                 every geometry record overwrite columns [x_start, x_end) of row i with the decoded
                 section; rows without a record stay zero
* confusion      S:423-431: per-voxel tally of pred/truth (tp, fp, fn, tn)
* overlap_metrics Eqs. 7-14 in exact rational arithmetic, rounded once to
                 float; a zero denominator gives NaN
* spatial_reduction Fig. 4 caption: full area / ROI area
"""
from fractions import Fraction

import numpy as np


def step(eb):
    """G-3: s = fl32(2 eb)."""
    return float(np.float32(2.0 * float(np.float32(eb))))


def decode_value(codes, s, dtype):
    """x^ for an array of codes (uint16 codes for uint16 input, int32 codes for fp32 input).

    uint16: code * s is exact in binary64 (16-bit code, 24-bit s); np.rint rounds it half to even,
    then the clamp.  fp32: the code is taken to fp32 first (exact for |code| <= 2^24, which covers
    every code the quantiser makes, |code| <= 2^23), the product of two fp32 values is exact in
    binary64, and the float64 -> float32 conversion rounds it once (to nearest even)."""
    c = np.asarray(codes)
    if dtype == np.uint16:
        return np.clip(np.rint(c.astype(np.float64) * float(s)), 0.0, 65535.0).astype(np.uint16)
    if dtype == np.float32:
        return (c.astype(np.float32).astype(np.float64) * float(s)).astype(np.float32)
    raise TypeError(dtype)


def decode_mask(K, codes, s, dtype):
    """Scatter: voxel i (K[i] = 1) takes the decoded code of its rank among the kept voxels (the
    dense code stream is in increasing i, a8); every other voxel is 0."""
    K = np.asarray(K).astype(bool)
    flat = K.reshape(-1)
    out = np.zeros(flat.size, dtype)
    idx = np.flatnonzero(flat)
    assert len(codes) >= idx.size
    out[idx] = decode_value(np.asarray(codes)[: idx.size], s, dtype)
    return out.reshape(K.shape)


def decode_spans(spans, codes, shape, s, dtype, row0=0):
    """zero raster; record (i, x_start, x_end) overwrites row i - row0, columns
    [x_start, x_end), with the next x_end - x_start codes of the pixel section, decoded."""
    Z, Y, X = shape
    out = np.zeros((Z * Y, X), dtype)
    p = 0
    for i, xs, xe in np.asarray(spans, np.int64).reshape(-1, 3):
        n = int(xe - xs)
        out[int(i) - row0, int(xs):int(xe)] = decode_value(np.asarray(codes)[p:p + n], s, dtype)
        p += n
    return out.reshape(shape)


def confusion(pred, truth):
    """tp = #(pred and truth), fp = #(pred and not truth), fn = #(not pred and truth),
    tn = #(neither)."""
    pred = np.asarray(pred).astype(bool).reshape(-1)
    truth = np.asarray(truth).astype(bool).reshape(-1)
    assert pred.shape == truth.shape
    tp = int(np.count_nonzero(pred & truth))
    fp = int(np.count_nonzero(pred & ~truth))
    fn = int(np.count_nonzero(~pred & truth))
    tn = int(pred.size) - tp - fp - fn
    return tp, fp, fn, tn


def _q(num, den):
    return float(Fraction(num) / Fraction(den)) if den != 0 else float("nan")


def overlap_metrics(tp, fp, fn, tn):
    """Eqs. 7-14 as SPEC S:432-436 writes them out:
       dsc = 2tp / (2tp + fp + fn)                 (Eq. 7)
       iou = tp / (tp + fp + fn)                   (Eq. 8)
       sensitivity = tp / (tp + fn)                (Eq. 9)
       specificity = tn / (tn + fp)                (Eq. 10)
       accuracy = (tp + tn) / N                    (Eq. 11)
       f_c = ((tn + fn)(tn + fp) + (fp + tp)(fn + tp)) / N     (Eq. 13)
       kappa = ((tp + tn) - f_c) / (N - f_c)       (Eq. 12)
       auc = 1 - (fp / (fp + tn) + fn / (fn + tp)) / 2         (Eq. 14)
    with N = tp + tn + fp + fn; exact rationals, rounded once; NaN where a denominator is 0."""
    tp, fp, fn, tn = (int(v) for v in (tp, fp, fn, tn))
    N = tp + tn + fp + fn
    out = {"dsc": _q(2 * tp, 2 * tp + fp + fn),
           "iou": _q(tp, tp + fp + fn),
           "sensitivity": _q(tp, tp + fn),
           "specificity": _q(tn, tn + fp),
           "accuracy": _q(tp + tn, N)}
    if N == 0:
        out["kappa"] = float("nan")
    else:
        fc = Fraction((tn + fn) * (tn + fp) + (fp + tp) * (fn + tp), N)
        out["kappa"] = float((tp + tn - fc) / (N - fc)) if N - fc != 0 else float("nan")
    if fp + tn == 0 or fn + tp == 0:
        out["auc"] = float("nan")
    else:
        out["auc"] = float(1 - (Fraction(fp, fp + tn) + Fraction(fn, fn + tp)) / 2)
    return out


def spatial_reduction(area, roi_area):
    """Fig. 4 caption: (width x height) / sum(x_end - x_start); NaN for an empty ROI."""
    return _q(area, roi_area)
