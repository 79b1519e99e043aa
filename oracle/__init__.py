"""ROIX oracle -- TEST INFRASTRUCTURE ONLY.

A plain, slow CPU statement of the ROIX-Comp hot path (BASELINE.json north_star; §4.1-4.2)
used to prove the CUDA path right.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import it.  It shares no code with
``paper_2602_15917_b200`` (the product) and never imports it.

Pieces:
* ``roix_oracle.c`` (single-threaded C, -O2 -ffp-contract=off): quantiser, range, histograms,
  norm8, binarisation, opening, BFS labelling, filter, extraction.
* ``otsu.py``: exact-rational 2-class Otsu.
* ``reconstruct.py``: NEXT-4 decode (mask and span forms), confusion counts and Eqs. 7-14.
* ``pipeline()`` below: the steps composed in the paper's order (Fig. 2):
  histogram -> normalise (Eq. 1) -> Otsu -> binarise (Eq. 2) -> opening -> CCL -> filter -> extract.

Parity status of each function: every function is pinned by tests/test_oracle_*.py
against closed forms, library routines (numpy / scipy.ndimage / OpenCV), SPEC worked examples or
brute force, except the *decisions* G-6, G-8..G-13 themselves, which are readings, not facts
("parity unpinned" for the choice of reading; the implementation of each reading is pinned).
"""
import ctypes
import os
import subprocess

import numpy as np

from .otsu import Degenerate, multi_otsu, otsu2  # noqa: F401
from .reconstruct import (confusion, decode_mask, decode_spans, decode_value, overlap_metrics,  # noqa: F401
                          spatial_reduction, step)

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "roix_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

OK, E_RANGE, E_NONFINITE, E_CAPACITY = 0, 1, 2, 3


def build(force=False):
    """Compile the C oracle (gcc, single-threaded, no fast-math, no FP contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + ".tmp%d" % os.getpid()
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math",
                               "-fPIC", "-shared", "-Wall", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is not None:
        return _lib
    lib = ctypes.CDLL(build())
    u64, i64, u32, f32, f64, vp, i32 = (ctypes.c_uint64, ctypes.c_int64, ctypes.c_uint32, ctypes.c_float,
                                        ctypes.c_double, ctypes.c_void_p, ctypes.c_int)
    sig = {
        "oracle_quantize_u16": (i32, [vp, u64, f32, vp]),
        "oracle_quantize_f32": (i32, [vp, u64, f32, vp]),
        "oracle_range_f32": (i32, [vp, u64, vp, vp]),
        "oracle_resolve_eb": (f32, [f32, f32, f64]),
        "oracle_hist_u16": (None, [vp, u64, vp]),
        "oracle_imax_u16": (u32, [vp]),
        "oracle_norm8_u16": (u32, [u32, u32]),
        "oracle_norm8_f32": (u32, [f32, f32]),
        "oracle_hist8_from_u16": (None, [vp, u32, vp]),
        "oracle_hist8_f32": (None, [vp, u64, f32, vp]),
        "oracle_binarize_u16": (None, [vp, u64, u32, u32, i32, vp]),
        "oracle_binarize_f32": (None, [vp, u64, f32, u32, i32, vp]),
        "oracle_open": (i32, [vp, i64, i64, i64, i32, vp]),
        "oracle_label": (i64, [vp, i64, i64, i64, i32, vp, vp, vp, u64]),
        "oracle_filter": (None, [vp, u64, vp, u64, u64, vp, vp]),
        "oracle_extract_u16": (i64, [vp, vp, u64, f32, vp]),
        "oracle_extract_f32": (i64, [vp, vp, u64, f32, vp]),
        "oracle_row_spans": (i64, [vp, vp, i32, i64, i64, i64, f32, vp, vp, vp]),
        "oracle_greedy_quantize": (i64, [vp, u64, f64, u32, vp, vp]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype, fn.argtypes = res, args
    _lib = lib
    return lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def _c(a, dtype):
    a = np.ascontiguousarray(a)
    assert a.dtype == dtype, (a.dtype, dtype)
    return a


class OracleError(RuntimeError):
    pass


# ---------------------------------------------------------------- step functions (numpy in/out)
def quantize(x, eb):
    """a1: codes = RNE(x / fl32(2 eb)) for every voxel (u16 -> u16 codes, f32 -> i32 codes)."""
    x = np.ascontiguousarray(x)
    lib = _load()
    if x.dtype == np.uint16:
        out = np.empty(x.shape, np.uint16)
        st = lib.oracle_quantize_u16(_p(x), x.size, float(eb), _p(out))
    elif x.dtype == np.float32:
        out = np.empty(x.shape, np.int32)
        st = lib.oracle_quantize_f32(_p(x), x.size, float(eb), _p(out))
    else:
        raise TypeError(x.dtype)
    if st != OK:
        raise OracleError("quantize status %d" % st)
    return out


def value_range(x):
    """a0: (min, max) of an fp32 volume; raises on a non-finite voxel (G-32)."""
    x = _c(x, np.float32)
    mn, mx = ctypes.c_float(), ctypes.c_float()
    st = _load().oracle_range_f32(_p(x), x.size, ctypes.byref(mn), ctypes.byref(mx))
    if st != OK:
        raise OracleError("range status %d" % st)
    return mn.value, mx.value


def resolve_eb(mn, mx, rel):
    """G-6: eb_abs = fl32(rel * (fl64(max) - fl64(min)))."""
    return float(_load().oracle_resolve_eb(mn, mx, rel))


def hist_u16(x, h=None):
    x = _c(x, np.uint16)
    h = np.zeros(65536, np.uint64) if h is None else h
    _load().oracle_hist_u16(_p(x), x.size, _p(h))
    return h


def imax_u16(h):
    return int(_load().oracle_imax_u16(_p(_c(h, np.uint64))))


def imax_f32(mx):
    """G-8: I_max = the global maximum, or 1 when it is <= 0."""
    return float(mx) if mx > 0 else 1.0


def norm8_u16(v, imax):
    return int(_load().oracle_norm8_u16(int(v), int(imax)))


def norm8_f32(x, imax):
    return int(_load().oracle_norm8_f32(float(x), float(imax)))


def hist8_from_u16(h, imax):
    h8 = np.zeros(256, np.uint64)
    _load().oracle_hist8_from_u16(_p(_c(h, np.uint64)), int(imax), _p(h8))
    return h8


def hist8_f32(x, imax):
    x = _c(x, np.float32)
    h8 = np.zeros(256, np.uint64)
    _load().oracle_hist8_f32(_p(x), x.size, float(imax), _p(h8))
    return h8


def binarize(x, imax, t8, polarity):
    """a4 (Eq. 2): m = norm8(x) > t8 (polarity 0 = HIGH) or <= t8 (1 = LOW), one byte per voxel."""
    x = np.ascontiguousarray(x)
    m = np.empty(x.shape, np.uint8)
    if x.dtype == np.uint16:
        _load().oracle_binarize_u16(_p(x), x.size, int(imax), int(t8), int(polarity), _p(m))
    else:
        x = _c(x, np.float32)
        _load().oracle_binarize_f32(_p(x), x.size, float(imax), int(t8), int(polarity), _p(m))
    return m


def opening(m, se):
    """a5 (G-11): dilate(erode(m)) with the radius-1 cross (se = 6: 3-D, se = 4: in-plane)."""
    m = _c(m, np.uint8)
    assert m.ndim == 3
    o = np.empty_like(m)
    st = _load().oracle_open(_p(m), *m.shape, int(se), _p(o))
    if st != OK:
        raise OracleError("open status %d" % st)
    return o


def label(o, conn):
    """a6: BFS components in raster order -> (comp ordinal per voxel, min_index[], size[])."""
    o = _c(o, np.uint8)
    assert o.ndim == 3
    comp = np.empty(o.shape, np.uint32)
    cap = int(o.sum()) + 1
    cmin = np.empty(cap, np.uint64)
    csz = np.empty(cap, np.uint64)
    nc = _load().oracle_label(_p(o), *o.shape, int(conn), _p(comp), _p(cmin), _p(csz), cap)
    if nc < 0:
        raise OracleError("label failed")
    return comp, cmin[:nc].copy(), csz[:nc].copy()


def filter_components(comp, csize, min_size):
    """a7: kept[c] = size >= min_size; K = voxels of kept components (bytes)."""
    comp = _c(comp, np.uint32)
    csize = _c(csize, np.uint64)
    kept = np.empty(max(csize.size, 1), np.uint8)
    K = np.empty(comp.shape, np.uint8)
    _load().oracle_filter(_p(comp), comp.size, _p(csize), csize.size, int(min_size), _p(kept), _p(K))
    return kept[: csize.size].copy(), K


def keep_largest(comp, csize):
    """NEXT-3 keep-largest mode ("select the largest by area"): only the
    component with the most voxels survives; ties go to the component containing the smallest linear
    index (S:187's raster-order anchor).  The table from `label` is in increasing minimum index, so
    the first maximum is the winner.  Returns (kept flags, K) like filter_components."""
    comp = _c(comp, np.uint32)
    csize = np.asarray(csize, np.uint64)
    kept = np.zeros(csize.size, np.uint8)
    if csize.size == 0:
        return kept, np.zeros(comp.shape, np.uint8)
    best = 0
    for c in range(1, csize.size):
        if csize[c] > csize[best]:
            best = c
    kept[best] = 1
    return kept, (comp == best).astype(np.uint8)


def extract(x, K, eb):
    """a8: codes of the voxels with K = 1, in increasing linear index."""
    x = np.ascontiguousarray(x)
    K = _c(K, np.uint8)
    lib = _load()
    if x.dtype == np.uint16:
        out = np.empty(int(K.sum()), np.uint16)
        n = lib.oracle_extract_u16(_p(x), _p(K), x.size, float(eb), _p(out))
    else:
        x = _c(x, np.float32)
        out = np.empty(int(K.sum()), np.int32)
        n = lib.oracle_extract_f32(_p(x), _p(K), x.size, float(eb), _p(out))
    if n < 0:
        raise OracleError("extract failed")
    return out[:n]


def row_spans(x, K, eb):
    """NEXT-1: the geometry records (i, x_start, x_end exclusive) of every
    row i = z*Y + y of K with a set bit, in increasing i, and the pixel sections -- the codes of
    x[i][x_start:x_end], interior gaps included -- concatenated.  Returns (spans (m, 3) int64,
    codes)."""
    x = np.ascontiguousarray(x)
    K = _c(K, np.uint8)
    assert x.ndim == 3 and K.shape == x.shape
    Z, Y, X = x.shape
    is_f32 = x.dtype == np.float32
    if not is_f32:
        x = _c(x, np.uint16)
    spans = np.empty((Z * Y + 1, 3), np.int64)
    codes = np.empty(x.size + 1, np.int32 if is_f32 else np.uint16)
    nc = ctypes.c_int64()
    m = _load().oracle_row_spans(_p(K), _p(x), int(is_f32), Z, Y, X, float(eb), _p(spans), _p(codes),
                                 ctypes.byref(nc))
    if m < 0:
        raise OracleError("row_spans failed")
    return spans[:m].copy(), codes[: nc.value].copy()


def greedy_quantize(D, E, qmax=65535):
    """NEXT-2: the paper's greedy absolute-error-bounded quantiser on a uint16
    sequence: (Q, group_start) with |Q - D| <= E, groups the greedy left-to-right maximal runs with a
    non-empty interval intersection, Q = floor((u + l) / 2) of the group, clipped to [0, qmax]."""
    D = _c(np.asarray(D).reshape(-1), np.uint16)
    Q = np.empty(max(D.size, 1), np.uint16)
    gs = np.empty(max(D.size, 1), np.uint8)
    _load().oracle_greedy_quantize(_p(D), D.size, float(E), int(qmax), _p(Q), _p(gs))
    return Q[: D.size].copy(), gs[: D.size].copy()


def pack_bits(mask):
    """G-16: bit (i mod 32) of uint32 word i // 32, LSB first, trailing pad bits zero."""
    b = np.packbits(np.ascontiguousarray(mask, dtype=np.uint8).reshape(-1).astype(bool), bitorder="little")
    pad = (-b.size) % 4
    if pad:
        b = np.concatenate([b, np.zeros(pad, np.uint8)])
    return b.view("<u4").copy()


# ---------------------------------------------------------------- the composed hot path
def background(x, B, op):
    """NEXT-3 background subtraction (M(x, y) = I(x, y) - B(x, y); SPEC S:61-69 clamps at 0)
    on a uint16 stack x[Z][Y][X] with one reference frame B[Y][X] applied to every frame:
      "sub": max(0, I - B)        the paper's M
      "rev": max(0, B - I)        transmission frames, where the sample darkens I (reading G-10)
      "add": min(65535, M + B)    the reconstruction's "combined with the precomputed background"
                                   for "sub"; "rev" is its own inverse on the ROI (B - (B - I))."""
    x = np.asarray(x).astype(np.int64)
    B = np.asarray(B).astype(np.int64)[None]
    if op == "sub":
        r = np.maximum(0, x - B)
    elif op == "rev":
        r = np.maximum(0, B - x)
    elif op == "add":
        r = np.minimum(65535, x + B)
    else:
        raise ValueError(op)
    return r.astype(np.uint16)


def frame_thresholds(x, classes=2, polarity=0):
    """NEXT-3 per-frame thresholds (uint16 frame stacks): every z-plane is its own image, as in the
    paper's 2-D setting -- its own I_max (Eq. 1), 256-bin normalised histogram and
    (multi-)Otsu thresholds.  Returns [(imax, thresholds, t8)] per frame; t8 is the ROI threshold
    (the lowest for HIGH, the highest for LOW, G-39).  Raises Degenerate for a frame with too few
    populated bins."""
    out = []
    for z in range(x.shape[0]):
        h = hist_u16(x[z])
        imax = imax_u16(h)
        h8 = hist8_from_u16(h, imax)
        ts = (otsu2(h8),) if classes == 2 else multi_otsu(h8, classes)
        out.append((imax, ts, ts[0] if polarity == 0 else ts[-1]))
    return out


def pipeline(x, *, eb=None, rel_eb=None, conn=6, se=6, min_size=64, polarity=0, classes=2, keep="size",
             frames=False, background_ref=None, bg="sub"):
    """The whole path on one volume x[Z][Y][X] (uint16 or float32).  Returns a dict of every
    intermediate the CUDA path exposes.  Raises Degenerate when Otsu has no valid threshold.
    classes = 3 (NEXT-3): multi-Otsu; the ROI is norm8 > the lowest threshold (HIGH) or
    norm8 <= the highest (LOW, reading G-39).  keep = "largest" (NEXT-3): only the largest component
    survives (min_size unused).  frames = True (NEXT-3, uint16): per-frame thresholds
    (frame_thresholds); the mask of frame z is Eq. 2 with frame z's I_max and threshold.
    background_ref (NEXT-3, uint16): the path runs on background(x, background_ref, bg)."""
    x = np.ascontiguousarray(x)
    assert x.ndim == 3
    out = {}
    if background_ref is not None:
        x = background(x, background_ref, bg)
        out["x"] = x
    if x.dtype == np.float32:
        mn, mx = value_range(x)
        out["min"], out["max"] = mn, mx
        if rel_eb is not None:
            eb = resolve_eb(mn, mx, rel_eb)
        imax = imax_f32(mx)
        h8 = hist8_f32(x, imax)
    else:
        h = hist_u16(x)
        out["hist"] = h
        imax = imax_u16(h)
        h8 = hist8_from_u16(h, imax)
    out["eb"], out["i_max"], out["h8"] = float(np.float32(eb)), imax, h8
    if frames:
        assert x.dtype == np.uint16
        ft = frame_thresholds(x, classes, polarity)
        out["frames"] = ft
        m = np.concatenate([binarize(x[z:z + 1], imax_z, t8_z, polarity) for z, (imax_z, _, t8_z) in enumerate(ft)])
        return _after_binarize(out, x, m, se, conn, min_size, keep)
    if classes == 2:
        t8 = otsu2(h8)
        out["thresholds"] = (t8,)
    else:
        ts = multi_otsu(h8, classes)
        out["thresholds"] = ts
        t8 = ts[0] if polarity == 0 else ts[-1]
    out["t8"] = t8
    m = binarize(x, imax, t8, polarity)
    return _after_binarize(out, x, m, se, conn, min_size, keep)


def _after_binarize(out, x, m, se, conn, min_size, keep):
    """a5..a8 on the binarised mask m."""
    o = opening(m, se)
    comp, cmin, csz = label(o, conn)
    kept, K = keep_largest(comp, csz) if keep == "largest" else filter_components(comp, csz, min_size)
    out.update(m=m, o=o, comp=comp, comp_min=cmin, comp_size=csz, kept=kept, K=K)
    out["stream"] = extract(x, K, out["eb"])
    out["count"] = int(out["stream"].size)
    return out
