"""Pins of the NEXT-3 background subtraction (oracle.background)."""
import numpy as np

import oracle


def test_spec_examples():
    I = np.array([[[10, 20]]], np.uint16)
    np.testing.assert_array_equal(oracle.background(I, np.array([[3, 3]], np.uint16), "sub"), [[[7, 17]]])
    np.testing.assert_array_equal(oracle.background(I, I[0], "sub"), np.zeros_like(I))
    np.testing.assert_array_equal(oracle.background(np.array([[[5]]], np.uint16), np.array([[9]], np.uint16),
                                                    "sub"), [[[0]]])


def test_brute_force_and_round_trips():
    rng = np.random.default_rng(0)
    I = rng.integers(0, 65536, (3, 4, 5)).astype(np.uint16)
    B = rng.integers(0, 65536, (4, 5)).astype(np.uint16)
    for op, f in (("sub", lambda a, b: max(0, a - b)), ("rev", lambda a, b: max(0, b - a)),
                  ("add", lambda a, b: min(65535, a + b))):
        got = oracle.background(I, B, op)
        for z in range(3):
            for y in range(4):
                for x in range(5):
                    assert got[z, y, x] == f(int(I[z, y, x]), int(B[y, x]))
    # restoring: add(sub(I, B), B) = max(I, B); rev(rev(I, B), B) = min(I, B) (exact where I <= B)
    np.testing.assert_array_equal(oracle.background(oracle.background(I, B, "sub"), B, "add"), np.maximum(I, B[None]))
    np.testing.assert_array_equal(oracle.background(oracle.background(I, B, "rev"), B, "rev"), np.minimum(I, B[None]))
