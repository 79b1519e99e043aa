"""The C-ABI library builds for sm_100a, loads without a GPU, and exports every symbol include/roix.h
declares; the ctypes struct mirrors match the C layout."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2602_15917_b200 import build

    build.build()
    from paper_2602_15917_b200 import _lib as L

    return L.load()


def _declared():
    src = open(os.path.join(ROOT, "include", "roix.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(roix_[a-z0-9_]+)\s*\(", src)))


def test_exports_every_declared_symbol(lib):
    names = _declared()
    assert len(names) >= 14
    for n in names:
        assert hasattr(lib, n), n
    from paper_2602_15917_b200 import _lib as L

    assert set(names) == set(L.EXPORTED)
    # every entry point has its Python binding of the same name (the helpers below are used raw)
    raw = {"roix_status_string", "roix_last_error", "roix_version", "roix_scalars_size"}
    missing = [n for n in names if n not in raw and not hasattr(L, n)]
    assert not missing, missing


def test_struct_layouts(lib):
    from paper_2602_15917_b200 import _lib as L

    assert lib.roix_scalars_size() == ctypes.sizeof(L.Scalars)
    assert lib.roix_version() == 1
    assert lib.roix_status_string(1) == b"invalid argument"


def test_host_validation_without_gpu(lib):
    """Host-detectable errors are reported before any launch (no GPU needed)."""
    from paper_2602_15917_b200 import _lib as L

    g = L.Geom(4, 4, 4, 0, 4)
    sz = ctypes.c_size_t()
    assert lib.roix_label_workspace(ctypes.byref(g), 0, ctypes.byref(sz)) == L.ROIX_E_INVALID
    assert lib.roix_label_workspace(ctypes.byref(g), 100, ctypes.byref(sz)) == L.ROIX_OK and sz.value > 0
    bad = L.Geom(4, 4, 4, 2, 4)    # slab beyond the volume
    assert lib.roix_label_workspace(ctypes.byref(bad), 100, ctypes.byref(sz)) == L.ROIX_E_INVALID
    assert lib.roix_histogram(None, 1, 10, None, None, 65536, None) == L.ROIX_E_INVALID
    assert lib.roix_histogram(ctypes.c_void_p(16), 1, 10, ctypes.c_void_p(16), ctypes.c_void_p(16), 256,
                              None) == L.ROIX_E_INVALID            # wrong nbins for u16
    assert lib.roix_morph(ctypes.c_void_p(16), 1, ctypes.byref(g), 5, None, None, ctypes.c_void_p(16),
                          ctypes.c_void_p(16), None, ctypes.c_void_p(16), 1 << 20, None) == L.ROIX_E_UNSUPPORTED
    assert b"se" in lib.roix_last_error()
    assert lib.roix_scalars_init(ctypes.c_void_p(16), ctypes.c_float(-1.0), None) == L.ROIX_E_INVALID
    assert lib.roix_resolve(ctypes.c_void_p(16), 1, ctypes.c_double(0.1), None) == L.ROIX_E_UNSUPPORTED


def test_sass_is_sm100a(lib):
    from paper_2602_15917_b200 import _lib as L

    out = subprocess.run(["cuobjdump", "--list-elf", L.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_overlap_metrics_host_vs_oracle(lib):
    """roix_overlap_metrics is host-only: Eqs. 7-14 against the oracle's exact rationals, the S:438-440
    golden values and 128-bit intermediates (N^2 > 2^64)."""
    import numpy as np

    import oracle
    from paper_2602_15917_b200 import _lib as L

    m = L.roix_overlap_metrics((40, 10, 10, 40))    # S:438 (tp, fp, fn, tn)
    assert abs(m["kappa"] - 0.6) <= 1e-12 and abs(m["auc"] - 0.8) <= 1e-12 and m["accuracy"] == 0.8
    m = L.roix_overlap_metrics((5, 5, 5, 85))
    assert m["dsc"] == 0.5 and abs(m["iou"] - 1 / 3) <= 1e-16
    rng = np.random.default_rng(1)
    cases = [(0, 0, 0, 0), (0, 0, 0, 9), (9, 0, 0, 0), (3 << 33, 5 << 30, 7 << 29, 11 << 33),
             (1 << 35, 1, 1, 1 << 35)] + [tuple(int(v) for v in rng.integers(0, 1 << int(rng.integers(1, 36)), 4))
                                           for _ in range(300)]
    for c in cases:
        want = oracle.overlap_metrics(*c)
        got = L.roix_overlap_metrics(c)
        for k in L.METRICS:
            np.testing.assert_allclose(got[k], want[k], rtol=2e-16, atol=0, equal_nan=True, err_msg="%s %s" % (k, c))
    assert lib.roix_overlap_metrics(None, None) == L.ROIX_E_INVALID


def test_host_validation_next_rows(lib):
    """NEXT-1..4 entry points reject bad arguments on the host, before any launch (no GPU needed)."""
    from paper_2602_15917_b200 import _lib as L

    P = ctypes.c_void_p(16)
    g = L.Geom(4, 4, 4, 0, 4)
    sz = ctypes.c_size_t()
    # multi-Otsu: class count 2 or 3 only
    assert lib.roix_threshold_multi(P, 256, L.F32, 0, 4, P, None) == L.ROIX_E_UNSUPPORTED
    assert lib.roix_threshold_multi(P, 255, L.F32, 0, 3, P, None) == L.ROIX_E_INVALID
    assert lib.roix_threshold_frames(P, 2, 0, 5, P, P, None) == L.ROIX_E_UNSUPPORTED
    # keep-largest on a sharded finish must go through roix_label_finish_keep
    out = L.LabelOut(16, None, None, None, 0, None)
    assert lib.roix_label_finish(P, ctypes.byref(g), L.KEEP_LARGEST, 8, P, 1 << 20, None, None, None, None,
                                 ctypes.byref(out), P, None) == L.ROIX_E_INVALID
    assert lib.roix_label_largest(P, ctypes.byref(g), 8, None, None, None, None, 2, P, P, None) == L.ROIX_E_INVALID
    # a merge map length pointer without the map arrays
    assert lib.roix_label_finish(P, ctypes.byref(g), 4, 8, P, 1 << 20, None, None, None, P,
                                 ctypes.byref(out), P, None) == L.ROIX_E_INVALID
    # device merge: workspace query and validation (no launch)
    assert lib.roix_merge_workspace(8, 1024, ctypes.byref(sz)) == L.ROIX_OK and sz.value >= 8 * 1024 * 12
    assert lib.roix_merge_workspace(0, 1024, ctypes.byref(sz)) == L.ROIX_E_INVALID
    assert lib.roix_merge_device(None, 2, 4, 4, P, P, P, P, P, 1 << 20, P, None) == L.ROIX_E_INVALID
    assert lib.roix_merge_device(P, 2, 4, 4, P, P, P, P, P, 0, P, None) == L.ROIX_E_INVALID   # ws too small
    # background: bad op, misaligned pointers
    assert lib.roix_background(P, P, ctypes.byref(g), 7, P, None) == L.ROIX_E_INVALID
    assert lib.roix_background(ctypes.c_void_p(18), P, ctypes.byref(g), L.BG_SUB, P, None) == L.ROIX_E_INVALID
    # decode: workspace size, alignment, dtype
    assert lib.roix_decode_workspace(1000, ctypes.byref(sz)) == L.ROIX_OK and sz.value > 0
    assert lib.roix_decode(P, P, 10, L.U16, 1000, P, P, P, 0, None) == L.ROIX_E_INVALID          # ws too small
    assert lib.roix_decode(P, P, 10, 9, 1000, P, P, P, 1 << 20, None) == L.ROIX_E_INVALID        # dtype
    assert lib.roix_decode(ctypes.c_void_p(20), P, 10, L.U16, 1000, P, P, P, 1 << 20, None) == L.ROIX_E_INVALID
    assert lib.roix_decode_spans_workspace(ctypes.byref(g), ctypes.byref(sz)) == L.ROIX_OK
    assert lib.roix_decode_spans(P, 4, P, 10, None, L.U16, ctypes.byref(g), P, P, P, sz.value, None) == \
        L.ROIX_E_INVALID                                                                           # counts NULL
    # confusion: counts required, masks aligned
    assert lib.roix_confusion(P, P, 10, None, None) == L.ROIX_E_INVALID
    assert lib.roix_confusion(ctypes.c_void_p(4), P, 10, P, None) == L.ROIX_E_INVALID
    # greedy: E must be finite and >= 0, qmax <= 65535
    assert lib.roix_greedy_quantize(P, 10, ctypes.c_double(-1.0), 255, P, P, P, P, 256, None) == L.ROIX_E_INVALID
    assert lib.roix_greedy_quantize(P, 10, ctypes.c_double(1.0), 70000, P, P, P, P, 256, None) == L.ROIX_E_INVALID
    assert b"qmax" in lib.roix_last_error()
