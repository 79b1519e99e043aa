"""-m gpu: BASELINE.json's full-size configs (C3 128x9700x13900 frames, C4 2048^3, C5 4096x4096x2048) in
the launch configuration bench.py times, checked against the oracle where it can compute the answer
(the full histogram streamed through oracle.hist_u16, the exact Otsu threshold from it, sampled
planes of the opening recomputed from 5 binarised planes, the code stream of sampled planes) and
by properties that hold at any size for the rest (component table, kept mask)."""
import ctypes
import gc

import numpy as np
import pytest
import torch

import oracle
import synth
from gpu_util import ptr, st
from paper_2602_15917_b200 import Pipeline
from paper_2602_15917_b200 import _lib as L

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

CHUNK = 1 << 28   # voxels per host chunk


@pytest.fixture(scope="module", autouse=True)
def _build():
    from paper_2602_15917_b200 import build

    build.build()
    synth.build()
    oracle.build()


def _u16(t):
    return t.cpu().numpy().view(np.uint16)


def _plane_bits(words, bit0, nbits):
    """bits [bit0, bit0 + nbits) of a device word array -> uint8 host mask"""
    w0, w1 = bit0 // 32, (bit0 + nbits + 31) // 32 + 1
    w = words[w0:min(w1, words.numel())].cpu().numpy().astype(np.int32).view(np.uint8)
    bits = np.unpackbits(w, bitorder="little")
    off = bit0 - 32 * w0
    return bits[off:off + nbits]


@pytest.mark.parametrize("name", ["C3", "C4", "C5"])
def test_fullsize(name):
    cfg = synth.CONFIGS[name]
    gc.collect()
    torch.cuda.empty_cache()
    free, _ = torch.cuda.mem_get_info()
    if cfg.nbytes * 2.3 > free:
        pytest.skip("not enough device memory on this GPU")
    x = synth.generate(cfg)
    p = Pipeline(cfg.shape, cfg.dtype, eb=cfg.eb, conn=cfg.conn, se=cfg.se, min_size=cfg.min_size,
                 polarity=cfg.polarity)
    r = p.run(x)
    Z, Y, X = cfg.shape
    n = cfg.n
    # --- histogram, I_max, Otsu threshold: the oracle over the whole volume, streamed in chunks
    flat = x.view(-1)
    h = np.zeros(65536, np.uint64)
    for a in range(0, n, CHUNK):
        oracle.hist_u16(_u16(flat[a:a + CHUNK]), h)
    np.testing.assert_array_equal(p.hist.cpu().numpy(), h.astype(np.int64))
    imax = oracle.imax_u16(h)
    t8 = oracle.otsu2(oracle.hist8_from_u16(h, imax))
    assert r.i_max == imax and r.t8 == t8
    # --- opening on sampled planes: o(z) from the oracle's binarisation of planes z-2 .. z+2
    o = torch.full_like(p.o, -1)
    L.roix_morph(ptr(x), p.cdtype, ctypes.byref(p.geom), p.se, None, None, ptr(p.sc), ptr(o), None,
                 ptr(p.morph_ws), p.morph_ws.numel(), st())
    torch.cuda.synchronize()
    rng = np.random.default_rng(0)
    planes = sorted({0, 1, Z - 1, Z // 2} | set(rng.integers(2, Z - 2, 3).tolist()))
    for z in planes:
        lo, hi = (max(0, z - 2), min(Z, z + 3)) if cfg.se == 6 else (z, z + 1)
        sub = _u16(x[lo:hi])
        m = oracle.binarize(sub, imax, t8, cfg.polarity)
        ref = oracle.opening(m, cfg.se)[z - lo]
        got = _plane_bits(o, z * Y * X, Y * X).reshape(Y, X)
        np.testing.assert_array_equal(got, ref, err_msg="plane %d" % z)
    # --- component table and kept mask: properties at any size
    nc = r.n_components
    assert nc == r.comp_min.numel() and nc > 0
    cmin = r.comp_min.cpu().numpy()
    csz = r.comp_size.cpu().numpy()
    kept = r.comp_kept.cpu().numpy()
    assert np.all(np.diff(cmin) > 0)                                   # sorted by min index (G-14)
    np.testing.assert_array_equal(kept, (csz >= cfg.min_size).astype(np.uint8))
    ow = o[: p.nwords].cpu().numpy().view(np.uint32)
    kw = r.keep_bits.cpu().numpy().view(np.uint32)
    pop_o = int(np.bitwise_count(ow).sum())
    pop_k = int(np.bitwise_count(kw).sum())
    assert int(csz.sum()) == pop_o                                     # every o voxel in one component
    assert pop_k == int(csz[kept.astype(bool)].sum()) == r.count       # K = voxels of kept components
    assert not np.any(kw & ~ow)                                        # K is a subset of o
    # each component's min-index voxel is set in o (and in K iff kept)
    pick = rng.choice(nc, min(nc, 2000), replace=False)
    for c in pick:
        i = int(cmin[c])
        assert (ow[i // 32] >> (i % 32)) & 1
        assert ((kw[i // 32] >> (i % 32)) & 1) == kept[c]
    # --- code stream on sampled planes: the kept voxels of plane z, quantised by the oracle
    for z in planes[:4]:
        b0 = z * Y * X
        before = int(np.bitwise_count(kw[: b0 // 32]).sum()) + int(
            np.bitwise_count(kw[b0 // 32] & np.uint32((1 << (b0 % 32)) - 1)))
        kz = _plane_bits(r.keep_bits, b0, Y * X)
        xz = _u16(x[z]).reshape(-1)
        ref = oracle.quantize(xz[kz.astype(bool)], cfg.eb)
        got = r.codes[before:before + ref.size].cpu().numpy().view(np.uint16)
        np.testing.assert_array_equal(got, ref, err_msg="plane %d" % z)
        # K on the plane is a union of whole x-runs of o (a run is kept or dropped entirely)
        oz = _plane_bits(o, b0, Y * X).reshape(Y, X).astype(np.int8)
        kz2 = kz.reshape(Y, X).astype(np.int8)
        starts = np.diff(np.concatenate([np.zeros((Y, 1), np.int8), oz], axis=1), axis=1) == 1
        run_id = np.cumsum(starts, axis=1) * oz
        for yy in rng.integers(0, Y, 50):
            for rid in np.unique(run_id[yy][run_id[yy] > 0]):
                vals = kz2[yy][run_id[yy] == rid]
                assert vals.min() == vals.max()
    del x, p, o, r, flat
    gc.collect()
    torch.cuda.empty_cache()
