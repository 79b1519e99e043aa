"""Pins for the oracle's opening (a5), labelling (a6), filter (a7), extraction (a8) and bit-packing:
scipy.ndimage / OpenCV library routines, textbook special cases, invariants."""
import numpy as np
import pytest
import scipy.ndimage as ndi
import cv2

CROSS6 = ndi.generate_binary_structure(3, 1)
CROSS4 = np.zeros((3, 3, 3), bool)
CROSS4[1] = ndi.generate_binary_structure(2, 1)
STRUCT = {6: ndi.generate_binary_structure(3, 1), 18: ndi.generate_binary_structure(3, 2),
          26: ndi.generate_binary_structure(3, 3), 4: CROSS4, 8: np.zeros((3, 3, 3), bool)}
STRUCT[8][1] = True


def _rand_mask(rng, shape, p):
    return (rng.random(shape) < p).astype(np.uint8)


SHAPES = [(1, 1, 1), (1, 5, 7), (3, 4, 5), (6, 9, 11), (10, 10, 10), (2, 33, 40), (12, 7, 3)]


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("se", [6, 4])
def test_opening_vs_scipy(oracle_mod, shape, se):
    rng = np.random.default_rng(hash((shape, se)) % 2 ** 32)
    st = CROSS6 if se == 6 else CROSS4
    for p in [0.3, 0.6, 0.85]:
        m = _rand_mask(rng, shape, p)
        e = ndi.binary_erosion(m, structure=st, border_value=1)     # out-of-volume ignored (G-11)
        ref = ndi.binary_dilation(e, structure=st, border_value=0)
        o = oracle_mod.opening(m, se)
        np.testing.assert_array_equal(o, ref.astype(np.uint8))
        assert np.all(o <= m)                                      # opening is anti-extensive
        np.testing.assert_array_equal(oracle_mod.opening(o, se), o)  # and idempotent


def test_opening_vs_opencv_in_plane(oracle_mod):
    rng = np.random.default_rng(2)
    m = _rand_mask(rng, (4, 37, 53), 0.7)
    o = oracle_mod.opening(m, 4)
    k = cv2.getStructuringElement(cv2.MORPH_CROSS, (3, 3))
    for z in range(m.shape[0]):
        ref = cv2.morphologyEx(m[z], cv2.MORPH_OPEN, k)
        np.testing.assert_array_equal(o[z], ref)


def test_opening_special_cases(oracle_mod):
    m = np.zeros((5, 5, 5), np.uint8)
    m[1:4, 1:4, 1:4] = 1                      # a 3x3x3 cube opens to the 7-voxel cross
    o = oracle_mod.opening(m, 6)
    exp = np.zeros_like(m)
    exp[1:4, 1:4, 1:4] = CROSS6
    np.testing.assert_array_equal(o, exp)
    m = np.zeros((3, 3, 3), np.uint8)
    m[1, 1, 1] = 1                            # an isolated voxel is removed
    assert oracle_mod.opening(m, 6).sum() == 0
    full = np.ones((2, 3, 4), np.uint8)       # all-foreground survives (border ignored, not zero)
    np.testing.assert_array_equal(oracle_mod.opening(full, 6), full)


def _canonical_scipy(o, conn):
    lab, n = ndi.label(o, structure=STRUCT[conn])
    flat = lab.ravel()
    idx = np.arange(flat.size, dtype=np.uint64)
    mins = np.full(n + 1, np.iinfo(np.uint64).max, np.uint64)
    np.minimum.at(mins, flat, idx)
    sizes = np.bincount(flat, minlength=n + 1).astype(np.uint64)
    order = np.argsort(mins[1:]) + 1
    return lab, mins, sizes, order


@pytest.mark.parametrize("conn", [6, 18, 26, 4, 8])
@pytest.mark.parametrize("shape", SHAPES)
def test_label_vs_scipy(oracle_mod, conn, shape):
    rng = np.random.default_rng(hash((conn, shape)) % 2 ** 32)
    for p in [0.2, 0.45, 0.7]:
        o = _rand_mask(rng, shape, p)
        comp, cmin, csz = oracle_mod.label(o, conn)
        lab, mins, sizes, order = _canonical_scipy(o, conn)
        np.testing.assert_array_equal(cmin, mins[order])
        np.testing.assert_array_equal(csz, sizes[order])
        # per-voxel: same partition, named by min index
        rank = np.full(mins.size, np.iinfo(np.uint32).max, np.uint32)
        rank[order] = np.arange(order.size, dtype=np.uint32)
        np.testing.assert_array_equal(comp, rank[lab])


def test_label_checkerboard(oracle_mod):
    z, y, x = np.indices((4, 4, 4))
    o = ((z + y + x) % 2 == 0).astype(np.uint8)
    assert oracle_mod.label(o, 6)[1].size == 32      # no face neighbours: all singletons
    assert oracle_mod.label(o, 18)[1].size == 1      # edge neighbours connect everything
    assert oracle_mod.label(o, 26)[1].size == 1
    assert oracle_mod.label(o, 4)[1].size == 32
    assert oracle_mod.label(o, 8)[1].size == 4       # one component per plane in-plane


def test_label_2d_vs_opencv(oracle_mod):
    rng = np.random.default_rng(8)
    o = _rand_mask(rng, (3, 40, 61), 0.45)
    comp, cmin, csz = oracle_mod.label(o, 8)
    total = 0
    for z in range(o.shape[0]):
        n, lab = cv2.connectedComponents(o[z], connectivity=8)
        total += n - 1
        for c in range(1, n):
            ys, xs = np.nonzero(lab == c)
            ids = comp[z][ys, xs]
            assert np.all(ids == ids[0])
            assert csz[ids[0]] == ys.size
    assert total == cmin.size


def test_filter_and_extract(oracle_mod):
    rng = np.random.default_rng(6)
    x = rng.integers(0, 4096, (6, 20, 24)).astype(np.uint16)
    o = _rand_mask(rng, x.shape, 0.55)
    comp, cmin, csz = oracle_mod.label(o, 6)
    for min_size in [1, 2, 5, 40, 10 ** 9]:
        kept, K = oracle_mod.filter_components(comp, csz, min_size)
        keep_ids = np.nonzero(csz >= min_size)[0]
        np.testing.assert_array_equal(kept, (csz >= min_size).astype(np.uint8))
        np.testing.assert_array_equal(K, np.isin(comp, keep_ids).astype(np.uint8))
        assert K.sum() == csz[keep_ids].sum()
        stream = oracle_mod.extract(x, K, 2.0)
        np.testing.assert_array_equal(stream, oracle_mod.quantize(x, 2.0)[K.astype(bool)])
    # boundary sizes min-1 / min
    o = np.zeros((1, 1, 12), np.uint8)
    o[0, 0, 0:3] = 1
    o[0, 0, 5:9] = 1
    comp, cmin, csz = oracle_mod.label(o, 6)
    kept, K = oracle_mod.filter_components(comp, csz, 4)
    assert kept.tolist() == [0, 1] and K.ravel().tolist() == [0] * 5 + [1] * 4 + [0] * 3


def test_pack_bits_layout(oracle_mod):
    rng = np.random.default_rng(0)
    for n in [1, 31, 32, 33, 100, 1000]:
        m = (rng.random(n) < 0.5).astype(np.uint8)
        w = oracle_mod.pack_bits(m)
        assert w.size == (n + 31) // 32
        for i in range(n):
            assert (int(w[i // 32]) >> (i % 32)) & 1 == m[i]
        for i in range(n, 32 * w.size):
            assert (int(w[i // 32]) >> (i % 32)) & 1 == 0


# ------------------------------------------------------------------ NEXT-3 keep-largest
def test_keep_largest_spec_examples(oracle_mod):
    o = np.zeros((1, 8, 12), np.uint8)
    o[0, 1:2, 1:6] = 1                      # blob of area 5
    o[0, 4:7, 6:9] = 1                      # blob of area 9
    comp, cmin, csz = oracle_mod.label(o, 8)
    kept, K = oracle_mod.keep_largest(comp, csz)
    assert kept.tolist() == [0, 1]          # only the 9-blob survives
    assert K.sum() == 9 and K[0, 5, 7] == 1 and K[0, 1, 3] == 0
    z = np.zeros((1, 5, 5), np.uint8)        # all-zero -> all-zero
    comp, cmin, csz = oracle_mod.label(z, 8)
    kept, K = oracle_mod.keep_largest(comp, csz)
    assert kept.size == 0 and not K.any()
    f = np.ones((1, 5, 7), np.uint8)         # one full-frame component -> identity
    comp, cmin, csz = oracle_mod.label(f, 8)
    np.testing.assert_array_equal(oracle_mod.keep_largest(comp, csz)[1], f)


def test_keep_largest_ties_and_scipy(oracle_mod):
    """Equal areas: the component holding the smallest linear index wins; random volumes: the
    kept voxels are scipy.ndimage's largest component (sizes from np.bincount)."""
    o = np.zeros((2, 6, 10), np.uint8)
    o[1, 0, 0:4] = 1                          # area 4, first voxel at linear index 60
    o[0, 3, 5:9] = 1                          # area 4, first voxel at 35: wins the tie
    comp, cmin, csz = oracle_mod.label(o, 6)
    K = oracle_mod.keep_largest(comp, csz)[1]
    assert K[0, 3, 5:9].all() and K.sum() == 4
    rng = np.random.default_rng(5)
    for conn, st in ((6, ndi.generate_binary_structure(3, 1)), (26, ndi.generate_binary_structure(3, 3))):
        for _ in range(5):
            o = (rng.random((5, 9, 13)) < 0.3).astype(np.uint8)
            lab, n = ndi.label(o, structure=st)
            comp, cmin, csz = oracle_mod.label(o, conn)
            K = oracle_mod.keep_largest(comp, csz)[1]
            sizes = np.bincount(lab.reshape(-1))[1:]
            winners = np.flatnonzero(sizes == sizes.max()) + 1
            first = min(winners, key=lambda w: np.flatnonzero(lab.reshape(-1) == w)[0])
            np.testing.assert_array_equal(K, (lab == first).astype(np.uint8))
