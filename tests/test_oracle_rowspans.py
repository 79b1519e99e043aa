"""Pins of the NEXT-1 oracle (row spans: the paper's geometry + pixel sections).

oracle.row_spans is checked against the SPEC worked examples, a brute-force
numpy statement of the definition on random masks, and the invariants S:224-225 (re-rasterised
spans cover K, exactly for row-convex shapes; section lengths sum to the code count).
"""
import numpy as np
import pytest

import oracle


def test_spec_examples_geometry():
    # S:200 row bits 0,1,1,0,1 -> record (i, 1, 5)
    K = np.array([[[0, 1, 1, 0, 1]]], np.uint8)
    spans, _ = oracle.row_spans(np.zeros(K.shape, np.uint16), K, 0.5)
    np.testing.assert_array_equal(spans, [[0, 1, 5]])
    # S:201 all-zero mask -> empty table
    spans, codes = oracle.row_spans(np.zeros((2, 3, 7), np.uint16), np.zeros((2, 3, 7), np.uint8), 0.5)
    assert spans.shape == (0, 3) and codes.size == 0
    # S:202 full row of width W -> (i, 0, W)
    W = 13
    K = np.zeros((1, 3, W), np.uint8)
    K[0, 2] = 1
    spans, _ = oracle.row_spans(np.zeros(K.shape, np.uint16), K, 0.5)
    np.testing.assert_array_equal(spans, [[2, 0, W]])


def test_spec_examples_sections():
    # S:209 image row [9, 8, 7, 6], record (0, 1, 3) -> section [8, 7]  (eb = 0.5: step 1, codes = values)
    x = np.array([[[9, 8, 7, 6]]], np.uint16)
    K = np.array([[[0, 1, 1, 0]]], np.uint8)
    spans, codes = oracle.row_spans(x, K, 0.5)
    np.testing.assert_array_equal(spans, [[0, 1, 3]])
    np.testing.assert_array_equal(codes, [8, 7])
    # S:211 record (0, 0, 4) -> full row copy
    spans, codes = oracle.row_spans(x, np.ones(x.shape, np.uint8), 0.5)
    np.testing.assert_array_equal(spans, [[0, 0, 4]])
    np.testing.assert_array_equal(codes, [9, 8, 7, 6])


def _brute(x, K, eb):
    Z, Y, X = x.shape
    spans, secs = [], []
    q = oracle.quantize(x, eb)
    for i in range(Z * Y):
        nz = np.flatnonzero(K.reshape(Z * Y, X)[i])
        if nz.size:
            spans.append((i, nz.min(), nz.max() + 1))
            secs.append(q.reshape(Z * Y, X)[i, nz.min():nz.max() + 1])
    sp = np.array(spans, np.int64).reshape(-1, 3)
    return sp, (np.concatenate(secs) if secs else np.zeros(0, q.dtype))


@pytest.mark.parametrize("shape", [(1, 1, 1), (2, 5, 7), (3, 9, 40), (4, 16, 64)])
@pytest.mark.parametrize("dt", ["u16", "f32"])
def test_random_vs_brute_force(shape, dt):
    rng = np.random.default_rng(abs(hash((shape, dt))) % 2 ** 32)
    for p in (0.0, 0.05, 0.5, 1.0):
        K = (rng.random(shape) < p).astype(np.uint8)
        if dt == "u16":
            x, eb = rng.integers(0, 65536, shape).astype(np.uint16), 2.0
        else:
            x, eb = rng.normal(0, 3, shape).astype(np.float32), 0.01
        spans, codes = oracle.row_spans(x, K, eb)
        bs, bc = _brute(x, K, eb)
        np.testing.assert_array_equal(spans, bs)
        np.testing.assert_array_equal(codes, bc)


def test_invariants_cover_and_lengths():
    rng = np.random.default_rng(7)
    # a ball (row-convex): spans re-rasterise to exactly K; random masks: a superset
    z, y, xx = np.indices((9, 21, 33))
    ball = ((z - 4) ** 2 / 16 + (y - 10) ** 2 / 64 + (xx - 16) ** 2 / 144 <= 1).astype(np.uint8)
    noisy = (rng.random(ball.shape) < 0.2).astype(np.uint8)
    x = rng.integers(0, 4096, ball.shape).astype(np.uint16)
    for K, convex in ((ball, True), (noisy, False)):
        spans, codes = oracle.row_spans(x, K, 1.0)
        R = np.zeros(K.size, np.uint8).reshape(-1, K.shape[2])
        for i, a, b in spans:
            R[i, a:b] = 1
        R = R.reshape(K.shape)
        assert np.all(R >= K)                           # S:224 superset
        if convex:
            np.testing.assert_array_equal(R, K)         # equal for row-convex shapes
        assert codes.size == int((spans[:, 2] - spans[:, 1]).sum())   # S:225 sum of n_i
