"""Property-based pins (hypothesis) of the oracle on tiny inputs: the labelling against
scipy.ndimage on arbitrary masks and connectivities, the opening's algebraic laws, the quantiser's
error bound and the extraction / decode round trip."""
import numpy as np
import pytest
import scipy.ndimage as ndi
from hypothesis import given, settings, strategies as st
from hypothesis.extra.numpy import arrays

import oracle

STRUCT = {6: ndi.generate_binary_structure(3, 1), 18: ndi.generate_binary_structure(3, 2),
          26: ndi.generate_binary_structure(3, 3)}

masks = st.tuples(st.integers(1, 6), st.integers(1, 7), st.integers(1, 9)).flatmap(
    lambda s: arrays(np.uint8, s, elements=st.integers(0, 1)))


@settings(max_examples=120, deadline=None)
@given(m=masks, conn=st.sampled_from([6, 18, 26, 4, 8]))
def test_label_matches_scipy(m, conn):
    comp, cmin, csz = oracle.label(m, conn)
    if conn in STRUCT:
        lab, n = ndi.label(m, structure=STRUCT[conn])
    else:   # in-plane connectivity: each z-plane on its own
        st2 = ndi.generate_binary_structure(2, 1 if conn == 4 else 2)
        lab = np.zeros(m.shape, np.int64)
        n = 0
        for z in range(m.shape[0]):
            l2, k = ndi.label(m[z], structure=st2)
            lab[z] = np.where(l2 > 0, l2 + n, 0)
            n += k
    assert len(cmin) == n
    flat = lab.reshape(-1)
    for c, (mi, sz) in enumerate(zip(cmin, csz)):
        assert flat[int(mi)] > 0 and np.count_nonzero(flat == flat[int(mi)]) == int(sz)
        assert np.flatnonzero(flat == flat[int(mi)])[0] == int(mi)   # label = the component's min index
        assert np.array_equal(comp.reshape(-1) == c, flat == flat[int(mi)])


@settings(max_examples=80, deadline=None)
@given(m=masks, se=st.sampled_from([4, 6]))
def test_opening_laws(m, se):
    o = oracle.opening(m, se)
    assert np.all(o <= m)                                  # anti-extensive
    np.testing.assert_array_equal(oracle.opening(o, se), o)   # idempotent


@settings(max_examples=80, deadline=None)
@given(x=arrays(np.uint16, st.integers(1, 300), elements=st.integers(0, 65535)),
       eb=st.sampled_from([0.5, 1.0, 2.0, 3.0, 8.0]))
def test_quantise_decode_round_trip(x, eb):
    c = oracle.quantize(x, eb)
    xh = oracle.decode_value(c, oracle.step(eb), np.uint16).astype(np.int64)
    assert np.all(np.abs(xh - x.astype(np.int64)) <= eb)
    K = (np.arange(x.size) % 3 != 1).astype(np.uint8).reshape(1, 1, -1)
    codes = oracle.extract(x.reshape(1, 1, -1), K, eb)
    dm = oracle.decode_mask(K, codes, oracle.step(eb), np.uint16).reshape(-1)
    np.testing.assert_array_equal(dm[K.reshape(-1) == 1], xh[K.reshape(-1) == 1])
    assert not dm[K.reshape(-1) == 0].any()
