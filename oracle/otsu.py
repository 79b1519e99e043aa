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
