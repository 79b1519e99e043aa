"""Pins of the NEXT-2 oracle: the paper's greedy absolute-error-bounded quantiser (§4.2.3
Steps 1-5).

oracle.greedy_quantize follows Steps 1-5 literally (interval intersection, floor midpoint, clip).  It
is checked against the SPEC worked examples, an independent feasibility-scan formulation (a group
[head, i] is feasible iff max - min <= 2E; value floor((max + min) / 2)) exhaustively on a
small alphabet and on random sequences, and the invariants S:293-298 (error bound, maximal groups,
E = 0 gives runs of equal values).
"""
import itertools

import numpy as np
import pytest

import oracle


def test_spec_examples():
    cases = [([5, 5, 7], 0, [5, 5, 7]),            # S:269 (G-34: two groups, not three)
             ([10, 12, 20], 2, [11, 11, 20]),
             ([], 1, []),
             ([255, 251], 3, [253, 253]),
             ([0, 255], 200, [127, 127])]
    for D, E, Q in cases:
        q, gs = oracle.greedy_quantize(np.array(D, np.uint16), E, 255)
        np.testing.assert_array_equal(q, Q)
    _, gs = oracle.greedy_quantize(np.array([10, 12, 20], np.uint16), 2, 255)
    np.testing.assert_array_equal(np.flatnonzero(gs), [0, 2])     # S:288 boundaries [0, 2]


def _feasibility(D, E):
    """extend greedily while max - min <= 2E; value floor((max + min) / 2)."""
    D = [int(v) for v in D]
    Q, starts, head = [0] * len(D), [], 0
    while head < len(D):
        lo = hi = D[head]
        i = head + 1
        while i < len(D) and max(hi, D[i]) - min(lo, D[i]) <= 2 * E:
            lo, hi = min(lo, D[i]), max(hi, D[i])
            i += 1
        for j in range(head, i):
            Q[j] = (lo + hi) // 2
        starts.append(head)
        head = i
    return np.array(Q, np.int64), starts


def test_fractional_bound_counterexample():
    """G-35: D = [0, 35], E = 17.5 is one feasible group (35 <= 2E) whose floor midpoint 17 is 18 from
    35 -- the paper's Steps 1-5 exceed E by 1/2 when frac(E) >= 1/2 (S:293 claims no violation)."""
    q, _ = oracle.greedy_quantize(np.array([0, 35], np.uint16), 17.5)
    np.testing.assert_array_equal(q, [17, 17])


def test_exhaustive_small_alphabet():
    # all sequences of length <= 6 over {0, 64, 128, 255}, E in {0, 2, 64, 100.5}
    for m in range(0, 7):
        for D in itertools.product([0, 64, 128, 255], repeat=m):
            for E in (0, 2, 64, 100.5):
                q, gs = oracle.greedy_quantize(np.array(D, np.uint16), E, 255)
                rq, rs = _feasibility(D, E)
                np.testing.assert_array_equal(q.astype(np.int64), rq)
                np.testing.assert_array_equal(np.flatnonzero(gs), rs)


@pytest.mark.parametrize("E", [0, 0.4, 1, 3, 17.5, 300])
def test_random_and_invariants(E):
    rng = np.random.default_rng(int(E * 10))
    for n in (1, 7, 100, 4096):
        walk = np.clip(np.cumsum(rng.integers(-6, 7, n)) + 30000, 0, 65535).astype(np.uint16)
        for D in (walk, rng.integers(0, 65536, n).astype(np.uint16), np.full(n, 9, np.uint16)):
            q, gs = oracle.greedy_quantize(D, E)
            rq, rs = _feasibility(D, E)
            np.testing.assert_array_equal(q.astype(np.int64), rq)
            np.testing.assert_array_equal(np.flatnonzero(gs), rs)
            # S:293 error bound.  With the floor midpoint the exact bound is ceil(floor(2E) / 2): E itself
            # for integer E and whenever frac(E) < 1/2, E + 1/2 otherwise (G-35)
            bound = -(-np.floor(2 * E) // 2)
            assert np.all(np.abs(q.astype(np.float64) - D) <= bound)
            if E == int(E) or E - int(E) < 0.5:
                assert np.all(np.abs(q.astype(np.float64) - D) <= E)
            starts = list(np.flatnonzero(gs)) + [n]
            for a, b in zip(starts[:-1], starts[1:]):                      # S:297 maximal groups
                seg = D[a:b].astype(np.int64)
                if b < n:
                    ext = np.append(seg, int(D[b]))
                    assert ext.max() - ext.min() > 2 * E
            if E == 0:                                                     # S:298 runs of equal values
                assert np.all((np.diff(D.astype(np.int64)) != 0) == gs[1:].astype(bool))
