"""Streaming oracle for the full-size uint16 configs -- TEST INFRASTRUCTURE ONLY.

SURVEY.md §8(c2): the full-size C3 / C4 / C5 volumes (17-34 G voxels) do not fit the in-memory
oracle, so the same definitions run plane by plane (``roix_oracle.c`` STREAMING MODE):

  pass A  histogram of every plane -> I_max (Eq. 1), h8, Otsu t8
  pass B  binarise (Eq. 2), opening (G-11), raster-scan union-find labelling (G-14)
  pass C  K = voxels of kept components (G-13) and the code stream (a1 + a8, G-17)

The input comes from ``feed(z0, nz)`` (the generated phantom, plane range [z0, z0+nz) as a uint16
numpy array), called once per pass.  Outputs too large to keep (o, K, the stream) are returned as
chunk digests (``digest.ChunkDigest``); the histogram, threshold, counts and the component table
are returned whole.  Only ``tests/`` and ``scripts/make_fullsize_golden.py`` use this module."""
import ctypes
import time

import numpy as np

from . import _load, _p, hist8_from_u16, imax_u16, otsu2
from .digest import ChunkDigest, table_digest

_SIGS = {
    "os_create": (ctypes.c_void_p, [ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                                    ctypes.c_int, ctypes.c_uint32, ctypes.c_uint32]),
    "os_free": (None, [ctypes.c_void_p]),
    "os_feed": (ctypes.c_int64, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
    "os_resolve": (ctypes.c_int64, [ctypes.c_void_p, ctypes.c_uint64]),
    "os_table": (ctypes.c_int64, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                  ctypes.c_uint64]),
    "os_extract": (ctypes.c_int64, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_float,
                                    ctypes.c_void_p, ctypes.c_void_p]),
    "os_nruns": (ctypes.c_uint64, [ctypes.c_void_p]),
    "os_nlabels": (ctypes.c_uint64, [ctypes.c_void_p]),
    "oracle_hist_u16": (None, [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p]),
}


def _lib():
    lib = _load()
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype, fn.argtypes = res, args
    return lib


def _planes(Z, plane_bytes, budget=1 << 30):
    step = max(1, min(Z, budget // max(plane_bytes, 1)))
    for z0 in range(0, Z, step):
        yield z0, min(step, Z - z0)


def fullsize_u16(feed, shape, *, eb, conn, se, min_size, polarity, want_o=True, log=None):
    """The whole path on a streamed uint16 volume; returns a dict of artefacts (digests for o, K,
    the stream).  Planes must be whole bytes of mask bits (Y*X % 8 == 0) so the packed planes
    concatenate into the volume's bit array (G-16)."""
    lib = _lib()
    Z, Y, X = (int(v) for v in shape)
    A = Y * X
    assert A % 8 == 0, "plane bits must be whole bytes"
    t = {}
    # pass A: histogram -> I_max -> h8 -> Otsu
    t0 = time.time()
    h = np.zeros(65536, np.uint64)
    for z0, nz in _planes(Z, 2 * A):
        x = np.ascontiguousarray(feed(z0, nz), dtype=np.uint16)
        lib.oracle_hist_u16(_p(x), x.size, _p(h))
    imax = imax_u16(h)
    h8 = hist8_from_u16(h, imax)
    t8 = otsu2(h8)
    t["A"] = time.time() - t0
    if log:
        log("pass A: I_max %d t8 %d (%.0f s)" % (imax, t8, t["A"]))
    # pass B: binarise, open, label
    t0 = time.time()
    st = lib.os_create(Z, Y, X, conn, se, polarity, imax, t8)
    if not st:
        raise RuntimeError("os_create failed")
    try:
        o_dig = ChunkDigest()
        obuf = np.empty((3, A), np.uint8)

        def take(k):
            if k < 0:
                raise RuntimeError("os_feed failed")
            for j in range(k):
                if want_o:
                    o_dig.feed(np.packbits(obuf[j], bitorder="little"))

        for z0, nz in _planes(Z, 2 * A):
            x = np.ascontiguousarray(feed(z0, nz), dtype=np.uint16)
            for q in range(nz):
                take(lib.os_feed(st, _p(x[q]), _p(obuf)))
        take(lib.os_feed(st, None, _p(obuf)))
        ncomp = lib.os_resolve(st, int(min_size))
        if ncomp < 0:
            raise RuntimeError("os_resolve failed")
        cmin = np.empty(max(ncomp, 1), np.uint64)
        csz = np.empty(max(ncomp, 1), np.uint64)
        kept = np.empty(max(ncomp, 1), np.uint8)
        if lib.os_table(st, _p(cmin), _p(csz), _p(kept), max(ncomp, 1)) != ncomp:
            raise RuntimeError("os_table failed")
        cmin, csz, kept = cmin[:ncomp], csz[:ncomp], kept[:ncomp]
        t["B"] = time.time() - t0
        if log:
            log("pass B: %d components, %d runs (%.0f s)" % (ncomp, lib.os_nruns(st), t["B"]))
        # pass C: K and the stream
        t0 = time.time()
        k_dig, s_dig = ChunkDigest(), ChunkDigest()
        K = np.empty(A, np.uint8)
        codes = np.empty(A, np.uint16)
        count = 0
        for z0, nz in _planes(Z, 2 * A):
            x = np.ascontiguousarray(feed(z0, nz), dtype=np.uint16)
            for q in range(nz):
                c = lib.os_extract(st, z0 + q, _p(x[q]), float(np.float32(eb)), _p(K), _p(codes))
                if c < 0:
                    raise RuntimeError("os_extract failed (quantiser range)")
                k_dig.feed(np.packbits(K, bitorder="little"))
                s_dig.feed(codes[:c])
                count += c
        t["C"] = time.time() - t0
        if log:
            log("pass C: %d kept voxels (%.0f s)" % (count, t["C"]))
        return {"shape": [Z, Y, X], "i_max": int(imax), "t8": int(t8),
                "hist_nonzero": int((h > 0).sum()), "hist_sum": int(h.sum()),
                "hist_digest": table_digest(h, np.zeros(0, np.uint64), np.zeros(0, np.uint8)),
                "n_components": int(ncomp), "n_kept": int(kept.sum()), "count": int(count),
                "n_runs": int(lib.os_nruns(st)), "table_digest": table_digest(cmin, csz, kept),
                "table": {"min_index": cmin.tolist(), "size": csz.tolist(), "kept": kept.tolist()}
                if ncomp <= 50000 else None,
                "o": o_dig.result() if want_o else None, "K": k_dig.result(), "stream": s_dig.result(),
                "oracle_seconds": t}
    finally:
        lib.os_free(st)
