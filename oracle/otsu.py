"""Otsu threshold on the 256-bin normalised-intensity histogram -- TEST INFRASTRUCTURE ONLY.

Plain definition, written out in exact rational arithmetic (``fractions.Fraction``):

* P:263-267 (paper §4.1 "Adaptive Thresholding"): multi-Otsu [Liao 2001] extending Otsu [1979];
  class count unstated.  Reading G-9: k = 2 classes ("Otsu-style", BASELINE.json north_star).
* the threshold maximises the between-class variance; ties are broken by the smallest
  threshold; fewer than k populated bins is an error.
* Otsu (1979): for a threshold t, class 0 = bins 0..t, class 1 = bins t+1..255,
  sigma_B^2(t) = w0 * w1 * (mu0 - mu1)^2  with  w_c = n_c / N,  mu_c = (sum over class of k*h[k]) / n_c.

Only thresholds t with both classes non-empty are candidates (the variance is undefined otherwise).
The binarised ROI is then norm8 > t (polarity HIGH) or norm8 <= t (polarity LOW, G-10).
"""
from fractions import Fraction


class Degenerate(ValueError):
    """Fewer than two populated bins: no threshold separates two classes."""


def between_class_variance(h8, t):
    """sigma_B^2(t) of Otsu (1979) as an exact Fraction, or None if a class is empty."""
    N = sum(h8)
    n0 = sum(h8[: t + 1])
    n1 = N - n0
    if n0 == 0 or n1 == 0:
        return None
    s0 = sum(k * h8[k] for k in range(t + 1))
    s1 = sum(k * h8[k] for k in range(t + 1, len(h8)))
    w0, w1 = Fraction(n0, N), Fraction(n1, N)
    mu0, mu1 = Fraction(s0, n0), Fraction(s1, n1)
    return w0 * w1 * (mu0 - mu1) ** 2


def otsu2(h8):
    """Smallest t in 0..254 maximising sigma_B^2(t) (S:170 tie-break).  Raises Degenerate."""
    h8 = [int(v) for v in h8]
    assert len(h8) == 256
    best, best_t = None, None
    for t in range(255):
        v = between_class_variance(h8, t)
        if v is None:
            continue
        if best is None or v > best:
            best, best_t = v, t
    if best_t is None:
        raise Degenerate("fewer than two populated histogram bins")
    return best_t


# ----------------------------------------------------------------------------- NEXT-3: multi-Otsu
def multi_otsu(h8, classes):
    """S:167-175 multi_otsu: the ascending tuple of classes - 1 thresholds in 0..254 maximising the
    between-class variance over every tuple whose classes are all non-empty; ties: the
    lexicographically smallest tuple.  Raises Degenerate with fewer than `classes` populated bins.

    Exhaustive over all tuples, as S:565 (AC4) states it; the class sums use prefix sums (a plain
    library step) so that k = 3 (32 385 tuples) runs in about a second."""
    h8 = [int(v) for v in h8]
    assert len(h8) == 256 and classes in (2, 3)
    if sum(1 for v in h8 if v) < classes:
        raise Degenerate("fewer populated bins than classes (S:171)")
    N = sum(h8)
    S = sum(k * h8[k] for k in range(256))
    cn = [0] * 257
    cs = [0] * 257
    for k in range(256):
        cn[k + 1] = cn[k] + h8[k]
        cs[k + 1] = cs[k] + k * h8[k]
    mu_T = Fraction(S, N)

    def var(ts):
        bounds = [-1] + list(ts) + [255]
        total = Fraction(0)
        for a, b in zip(bounds[:-1], bounds[1:]):
            n = cn[b + 1] - cn[a + 1]
            if n == 0:
                return None
            s = cs[b + 1] - cs[a + 1]
            total += Fraction(n, N) * (Fraction(s, n) - mu_T) ** 2
        return total

    tuples = ((t,) for t in range(255)) if classes == 2 else \
        ((t1, t2) for t1 in range(254) for t2 in range(t1 + 1, 255))
    best, best_t = None, None
    for ts in tuples:                       # ascending lexicographic order: strict > keeps the smallest
        v = var(ts)
        if v is not None and (best is None or v > best):
            best, best_t = v, ts
    if best_t is None:
        raise Degenerate("no tuple with all classes non-empty")
    return best_t
