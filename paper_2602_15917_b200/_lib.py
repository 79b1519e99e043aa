"""ctypes binding of libroix (include/roix.h): argument marshalling only -- every step of the path runs
in the library's CUDA kernels.  Functions keep the C names; pointer arguments take integers (e.g. a
torch tensor's ``data_ptr()``) and streams take ``torch.cuda.Stream.cuda_stream``.

There is no CPU fallback: importing this module on a box without the built library raises.
"""
import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libroix.so")

ROIX_OK, ROIX_E_INVALID, ROIX_E_UNSUPPORTED, ROIX_E_CUDA = 0, 1, 2, 3
ERR_NONFINITE, ERR_RANGE, ERR_CAPACITY, ERR_DEGENERATE, ERR_FORMAT = 1, 2, 4, 8, 16
U16, F32 = 1, 2
POL_HIGH, POL_LOW = 0, 1


class Frame(ctypes.Structure):
    """Mirror of roix_frame (NEXT-3 per-frame thresholds)."""
    _fields_ = [("thr_u16", ctypes.c_uint32), ("t8", ctypes.c_uint32), ("t8_all", ctypes.c_uint32),
                ("i_max", ctypes.c_uint32)]


class Scalars(ctypes.Structure):
    """Mirror of roix_scalars (device-resident; read back with ``Scalars.from_buffer_copy``)."""
    _fields_ = [("err", ctypes.c_uint32), ("min_ord", ctypes.c_uint32), ("max_ord", ctypes.c_uint32),
                ("polarity", ctypes.c_uint32), ("eb", ctypes.c_float), ("s", ctypes.c_float),
                ("s_inv", ctypes.c_float), ("s_int", ctypes.c_uint32), ("s_magic", ctypes.c_uint32),
                ("t8_all", ctypes.c_uint32), ("i_max", ctypes.c_float), ("t8", ctypes.c_uint32),
                ("thr_u16", ctypes.c_uint32), ("thr_f32", ctypes.c_float), ("count", ctypes.c_uint64),
                ("n_components", ctypes.c_uint64), ("n_kept", ctypes.c_uint64), ("n_runs", ctypes.c_uint64),
                ("spec_lo", ctypes.c_uint32), ("spec_hi", ctypes.c_uint32), ("spec_state", ctypes.c_uint32),
                ("run_slots", ctypes.c_uint32), ("n_uncertain", ctypes.c_uint64), ("edges", ctypes.c_float * 256)]


class Geom(ctypes.Structure):
    _fields_ = [("nz", ctypes.c_uint64), ("ny", ctypes.c_uint64), ("nx", ctypes.c_uint64),
                ("z0", ctypes.c_uint64), ("gz", ctypes.c_uint64)]


class LabelOut(ctypes.Structure):
    _fields_ = [("keep_bits", ctypes.c_void_p), ("comp_min", ctypes.c_void_p), ("comp_size", ctypes.c_void_p),
                ("comp_kept", ctypes.c_void_p), ("comp_cap", ctypes.c_uint64), ("labels", ctypes.c_void_p)]


class BRun(ctypes.Structure):
    _fields_ = [("y", ctypes.c_uint32), ("x0", ctypes.c_uint32), ("x1", ctypes.c_uint32), ("pad", ctypes.c_uint32),
                ("label", ctypes.c_uint64)]


class RoixError(RuntimeError):
    pass


_lib = None
_vp, _u64, _u32, _f32, _f64, _i32 = (ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_float,
                                     ctypes.c_double, ctypes.c_int)
_SIGS = {
    "roix_status_string": (ctypes.c_char_p, [_i32]),
    "roix_last_error": (ctypes.c_char_p, []),
    "roix_version": (_i32, []),
    "roix_scalars_size": (ctypes.c_size_t, []),
    "roix_scalars_init": (_i32, [_vp, _f32, _vp]),
    "roix_range": (_i32, [_vp, _u64, _vp, _vp]),
    "roix_resolve": (_i32, [_vp, _i32, _f64, _vp]),
    "roix_quantize": (_i32, [_vp, _i32, _u64, _vp, _vp, _vp]),
    "roix_histogram": (_i32, [_vp, _i32, _u64, _vp, _vp, _u32, _vp]),
    "roix_histogram_clear": (_i32, [_vp, _u64, _vp]),
    "roix_threshold": (_i32, [_vp, _u32, _i32, _i32, _vp, _vp]),
    "roix_morph_workspace": (_i32, [ctypes.POINTER(Geom), ctypes.POINTER(ctypes.c_size_t)]),
    "roix_morph": (_i32, [_vp, _i32, ctypes.POINTER(Geom), _u32, _vp, _vp, _vp, _vp, _vp, _vp, ctypes.c_size_t, _vp]),
    "roix_histogram_binarize_workspace": (_i32, [ctypes.POINTER(Geom), ctypes.POINTER(ctypes.c_size_t)]),
    "roix_histogram_binarize": (_i32, [_vp, _i32, ctypes.POINTER(Geom), _i32, _vp, _vp, _u32, _vp, ctypes.c_size_t,
                                       _vp]),
    "roix_morph_prebinarized": (_i32, [_vp, _i32, ctypes.POINTER(Geom), _u32, _vp, _vp, _vp, _vp, _vp, _vp,
                                       ctypes.c_size_t, _vp]),
    "roix_binarize_planes": (_i32, [_vp, _i32, ctypes.POINTER(Geom), _u64, _u64, _vp, _vp, _vp]),
    "roix_label_workspace": (_i32, [ctypes.POINTER(Geom), _u64, ctypes.POINTER(ctypes.c_size_t)]),
    "roix_label": (_i32, [_vp, _vp, ctypes.POINTER(Geom), _u32, _u64, _u64, _vp, ctypes.c_size_t,
                          ctypes.POINTER(LabelOut), _vp, _vp]),
    "roix_morph_slots": (_i32, [_vp, _i32, ctypes.POINTER(Geom), _u32, _vp, _vp, _vp, _vp, _vp, _vp, _u32, _vp,
                                ctypes.c_size_t, _vp]),
    "roix_label_slots": (_i32, [_vp, _vp, _vp, _u32, ctypes.POINTER(Geom), _u32, _u64, _u64, _vp, ctypes.c_size_t,
                                ctypes.POINTER(LabelOut), _vp, _vp]),
    "roix_label_local_slots": (_i32, [_vp, _vp, _vp, _u32, ctypes.POINTER(Geom), _u32, _u64, _vp, ctypes.c_size_t,
                                      _vp, _vp]),
    "roix_label_local": (_i32, [_vp, _vp, ctypes.POINTER(Geom), _u32, _u64, _vp, ctypes.c_size_t, _vp, _vp]),
    "roix_label_boundary": (_i32, [_vp, ctypes.POINTER(Geom), _u64, _i32, _vp, _u64, _vp, _vp, _vp]),
    "roix_label_link": (_i32, [_vp, ctypes.POINTER(Geom), _u64, _u32, _vp, _vp, _vp, _u64, _vp, _vp, _vp]),
    "roix_label_boundary_roots": (_i32, [_vp, ctypes.POINTER(Geom), _u64, _vp, _vp, _u64, _vp, _vp, _vp]),
    "roix_merge": (_i32, [_vp, _u64, _vp, _vp, _u64, _vp, _vp, _vp, _vp]),
    "roix_merge_workspace": (_i32, [_u32, _u64, ctypes.POINTER(ctypes.c_size_t)]),
    "roix_merge_device": (_i32, [_vp, _u32, _u64, _u64, _vp, _vp, _vp, _vp, _vp, ctypes.c_size_t, _vp, _vp]),
    "roix_label_finish": (_i32, [_vp, ctypes.POINTER(Geom), _u64, _u64, _vp, ctypes.c_size_t, _vp, _vp, _vp, _vp,
                                 ctypes.POINTER(LabelOut), _vp, _vp]),
    "roix_extract_workspace": (_i32, [_u64, ctypes.POINTER(ctypes.c_size_t)]),
    "roix_extract": (_i32, [_vp, _i32, _u64, _vp, _vp, _vp, _u64, _vp, _vp, ctypes.c_size_t, _vp]),
    "roix_row_spans_workspace": (_i32, [ctypes.POINTER(Geom), ctypes.POINTER(ctypes.c_size_t)]),
    "roix_row_spans": (_i32, [_vp, _vp, _i32, ctypes.POINTER(Geom), _vp, _vp, _u64, _vp, _u64, _vp, _vp,
                              ctypes.c_size_t, _vp]),
    "roix_greedy_workspace": (_i32, [_u64, ctypes.POINTER(ctypes.c_size_t)]),
    "roix_greedy_quantize": (_i32, [_vp, _u64, _f64, _u32, _vp, _vp, _vp, _vp, ctypes.c_size_t, _vp]),
    "roix_extract_runs": (_i32, [_vp, _i32, ctypes.POINTER(Geom), _u64, _vp, ctypes.c_size_t, _vp, _vp, _u64, _vp,
                                 _vp]),
    "roix_label_largest": (_i32, [_vp, ctypes.POINTER(Geom), _u64, _vp, _vp, _vp, _vp, _u32, _vp, _vp, _vp]),
    "roix_label_finish_keep": (_i32, [_vp, ctypes.POINTER(Geom), _u64, _vp, ctypes.c_size_t, _vp, _vp, _vp, _vp, _vp,
                                      ctypes.POINTER(LabelOut), _vp, _vp]),
    "roix_background": (_i32, [_vp, _vp, ctypes.POINTER(Geom), _i32, _vp, _vp]),
    "roix_histogram_frames": (_i32, [_vp, ctypes.POINTER(Geom), _vp, _vp, _vp]),
    "roix_threshold_frames": (_i32, [_vp, _u64, _i32, _u32, _vp, _vp, _vp]),
    "roix_morph_frames": (_i32, [_vp, ctypes.POINTER(Geom), _u32, _vp, _vp, _vp, _vp, _vp, _vp, _vp, ctypes.c_size_t,
                                 _vp]),
    "roix_threshold_multi": (_i32, [_vp, _u32, _i32, _i32, _u32, _vp, _vp]),
    "roix_decode_workspace": (_i32, [_u64, ctypes.POINTER(ctypes.c_size_t)]),
    "roix_decode": (_i32, [_vp, _vp, _u64, _i32, _u64, _vp, _vp, _vp, ctypes.c_size_t, _vp]),
    "roix_decode_spans_workspace": (_i32, [ctypes.POINTER(Geom), ctypes.POINTER(ctypes.c_size_t)]),
    "roix_decode_spans": (_i32, [_vp, _u64, _vp, _u64, _vp, _i32, ctypes.POINTER(Geom), _vp, _vp, _vp,
                                 ctypes.c_size_t, _vp]),
    "roix_confusion": (_i32, [_vp, _vp, _u64, _vp, _vp]),
    "roix_overlap_metrics": (_i32, [ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(ctypes.c_double)]),
}


def load():
    """Load the in-tree libroix.so (built by paper_2602_15917_b200.build / __graft_entry__.build)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RoixError("libroix.so is not built (run __graft_entry__.build()); there is no CPU fallback")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype, fn.argtypes = res, args
    assert lib.roix_scalars_size() == ctypes.sizeof(Scalars), "roix_scalars layout mismatch"
    _lib = lib
    return lib


def _check(status, name):
    if status != ROIX_OK:
        lib = load()
        raise RoixError("%s: %s (%s)" % (name, lib.roix_status_string(status).decode(),
                                         lib.roix_last_error().decode()))


def _wrap(name):
    def f(*args):
        _check(getattr(load(), name)(*args), name)
    f.__name__ = name
    return f


roix_scalars_init = _wrap("roix_scalars_init")
roix_range = _wrap("roix_range")
roix_resolve = _wrap("roix_resolve")
roix_quantize = _wrap("roix_quantize")
roix_histogram = _wrap("roix_histogram")
roix_histogram_clear = _wrap("roix_histogram_clear")
roix_threshold = _wrap("roix_threshold")
roix_morph = _wrap("roix_morph")
roix_binarize_planes = _wrap("roix_binarize_planes")
roix_histogram_binarize = _wrap("roix_histogram_binarize")
roix_morph_prebinarized = _wrap("roix_morph_prebinarized")
roix_label = _wrap("roix_label")
roix_extract = _wrap("roix_extract")
roix_extract_runs = _wrap("roix_extract_runs")
roix_row_spans = _wrap("roix_row_spans")
roix_greedy_quantize = _wrap("roix_greedy_quantize")
roix_threshold_multi = _wrap("roix_threshold_multi")
roix_histogram_frames = _wrap("roix_histogram_frames")
roix_background = _wrap("roix_background")
BG_SUB, BG_REV, BG_ADD = 0, 1, 2
roix_threshold_frames = _wrap("roix_threshold_frames")
roix_morph_frames = _wrap("roix_morph_frames")
roix_label_largest = _wrap("roix_label_largest")
roix_label_finish_keep = _wrap("roix_label_finish_keep")
KEEP_LARGEST = (1 << 64) - 1
roix_decode = _wrap("roix_decode")
roix_decode_spans = _wrap("roix_decode_spans")
roix_confusion = _wrap("roix_confusion")
roix_label_local = _wrap("roix_label_local")
roix_morph_slots = _wrap("roix_morph_slots")
roix_label_slots = _wrap("roix_label_slots")
roix_label_local_slots = _wrap("roix_label_local_slots")
roix_label_boundary = _wrap("roix_label_boundary")
roix_label_link = _wrap("roix_label_link")
roix_label_boundary_roots = _wrap("roix_label_boundary_roots")
roix_label_finish = _wrap("roix_label_finish")
roix_merge_device = _wrap("roix_merge_device")


def roix_merge_workspace(G, root_cap):
    out = ctypes.c_size_t()
    _check(load().roix_merge_workspace(G, root_cap, ctypes.byref(out)), "roix_merge_workspace")
    return out.value


def roix_merge(pairs, labels, sizes):
    """Host merge (numpy uint64 arrays): pairs (k, 2), labels (m,), sizes (m,) ->
    (labels, final_labels, totals) for the distinct labels in increasing order."""
    import numpy as np

    pairs = np.ascontiguousarray(pairs, dtype=np.uint64).reshape(-1)
    labels = np.ascontiguousarray(labels, dtype=np.uint64)
    sizes = np.ascontiguousarray(sizes, dtype=np.uint64)
    m = labels.size
    ol, of, ot = (np.empty(max(m, 1), np.uint64) for _ in range(3))
    nout = ctypes.c_uint64()
    p = lambda a: a.ctypes.data_as(ctypes.c_void_p)
    _check(load().roix_merge(p(pairs), pairs.size // 2, p(labels), p(sizes), m, p(ol), p(of), p(ot),
                             ctypes.byref(nout)), "roix_merge")
    k = nout.value
    return ol[:k].copy(), of[:k].copy(), ot[:k].copy()


def roix_label_workspace(geom, run_capacity):
    out = ctypes.c_size_t()
    _check(load().roix_label_workspace(ctypes.byref(geom), run_capacity, ctypes.byref(out)), "roix_label_workspace")
    return out.value


def roix_histogram_binarize_workspace(geom):
    out = ctypes.c_size_t()
    _check(load().roix_histogram_binarize_workspace(ctypes.byref(geom), ctypes.byref(out)),
           "roix_histogram_binarize_workspace")
    return out.value


def roix_morph_workspace(geom):
    out = ctypes.c_size_t()
    _check(load().roix_morph_workspace(ctypes.byref(geom), ctypes.byref(out)), "roix_morph_workspace")
    return out.value


def roix_extract_workspace(n):
    out = ctypes.c_size_t()
    _check(load().roix_extract_workspace(n, ctypes.byref(out)), "roix_extract_workspace")
    return out.value


def roix_row_spans_workspace(geom):
    out = ctypes.c_size_t()
    _check(load().roix_row_spans_workspace(ctypes.byref(geom), ctypes.byref(out)), "roix_row_spans_workspace")
    return out.value


def roix_greedy_workspace(n):
    out = ctypes.c_size_t()
    _check(load().roix_greedy_workspace(n, ctypes.byref(out)), "roix_greedy_workspace")
    return out.value


def roix_decode_workspace(n):
    out = ctypes.c_size_t()
    _check(load().roix_decode_workspace(n, ctypes.byref(out)), "roix_decode_workspace")
    return out.value


def roix_decode_spans_workspace(geom):
    out = ctypes.c_size_t()
    _check(load().roix_decode_spans_workspace(ctypes.byref(geom), ctypes.byref(out)), "roix_decode_spans_workspace")
    return out.value


METRICS = ("dsc", "iou", "sensitivity", "specificity", "accuracy", "kappa", "auc")


def roix_overlap_metrics(counts):
    """Eqs. 7-14 from host confusion counts (tp, fp, fn, tn) -> dict of METRICS (NaN: undefined)."""
    c = (ctypes.c_uint64 * 4)(*[int(v) for v in counts])
    out = (ctypes.c_double * 7)()
    _check(load().roix_overlap_metrics(c, out), "roix_overlap_metrics")
    return dict(zip(METRICS, list(out)))


def scalars_size():
    return load().roix_scalars_size()


EXPORTED = sorted(_SIGS)
