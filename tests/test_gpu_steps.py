"""-m gpu: each C-ABI call against the oracle, element by element, on seeded inputs that span several
tiles and ragged tails.  Bit-exact everywhere (integer, mask and index outputs; the fp32 quantiser is
exact by construction, G-4)."""
import ctypes

import numpy as np
import pytest
import torch

import oracle
from gpu_util import (dev, dtype_code, ord2f, gpu_threshold, host_u16, mask_to_words, new_sc, ptr, read_sc, st,
                      words_to_mask, write_sc)
from paper_2602_15917_b200 import _lib as L

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _build():
    from paper_2602_15917_b200 import build

    build.build()
    oracle.build()


def _quantize_gpu(x_np, eb):
    x = dev(x_np)
    sc = new_sc(eb)
    L.roix_resolve(ptr(sc), dtype_code(x_np), 0.0, st())
    out = torch.empty(x_np.size + 8, dtype=torch.int16 if x_np.dtype == np.uint16 else torch.int32, device="cuda")
    L.roix_quantize(ptr(x), dtype_code(x_np), x_np.size, ptr(sc), ptr(out), st())
    s = read_sc(sc)
    o = out[: x_np.size].cpu().numpy()
    return (o.view(np.uint16) if x_np.dtype == np.uint16 else o), s


# ------------------------------------------------------------------------------------- a1 quantise
@pytest.mark.parametrize("eb", [0.5, 1.0, 1.5, 2.0, 2.5, 3.0, 4.0, 0.75, 1.25, 100.0, 2047.5, 6.3])
def test_quantize_u16_exhaustive(eb):
    x = np.concatenate([np.arange(65536), np.arange(5)]).astype(np.uint16)   # ragged tail (n % 8 = 5)
    got, s = _quantize_gpu(x, eb)
    assert s.err == 0
    np.testing.assert_array_equal(got, oracle.quantize(x, eb))


def test_quantize_u16_range_error():
    x = np.arange(65536, dtype=np.uint16)
    _, s = _quantize_gpu(x, 0.25)            # s = 0.5: codes above 65535 -> ERR_RANGE (oracle raises too)
    assert s.err & L.ERR_RANGE
    with pytest.raises(oracle.OracleError):
        oracle.quantize(x, 0.25)


@pytest.mark.parametrize("eb", [1.3e-3, 0.01, 0.37, 5.0])
def test_quantize_f32_random_ties_near_ties(eb):
    rng = np.random.default_rng(17)
    s = np.float32(2 * np.float32(eb))
    k = rng.integers(-3000, 3000, 20000)
    ties = ((k + 0.5) * np.float64(s)).astype(np.float32)
    x = np.concatenate([rng.normal(0.5, 0.4, 100003), rng.uniform(-1000, 1000, 50001) * s, ties,
                        np.nextafter(ties, np.float32(np.inf)), np.nextafter(ties, np.float32(-np.inf)),
                        [0.0, -0.0, np.float32(1e-30), -np.float32(1e-30)]]).astype(np.float32)
    got, sc = _quantize_gpu(x, eb)
    assert sc.err == 0
    np.testing.assert_array_equal(got, oracle.quantize(x, eb))


def test_quantize_f32_nonfinite_and_range():
    x = np.array([1.0, np.nan, 2.0], np.float32)
    _, s = _quantize_gpu(x, 1.0)
    assert s.err & L.ERR_NONFINITE
    x = np.array([1.0, 2.0 ** 24], np.float32)
    _, s = _quantize_gpu(x, 0.5)
    assert s.err & L.ERR_RANGE


# ------------------------------------------------------------------------ a0 range, eb, norm8 edges
def test_range_resolve_edges():
    rng = np.random.default_rng(3)
    x_np = np.concatenate([rng.normal(0.02, 0.005, 300001), rng.uniform(0.3, 1.2, 7777)]).astype(np.float32)
    x, sc, h = gpu_threshold(x_np, rel_eb=1e-3)
    s = read_sc(sc)
    mn, mx = oracle.value_range(x_np)
    assert ord2f(s.min_ord) == mn and ord2f(s.max_ord) == mx
    assert s.eb == oracle.resolve_eb(mn, mx, 1e-3)
    assert s.i_max == oracle.imax_f32(mx)
    # edges[k] = smallest float with norm8 >= k (checked with the oracle's norm8)
    for k in range(1, 256):
        e = np.float32(s.edges[k])
        assert oracle.norm8_f32(e, s.i_max) >= k
        assert oracle.norm8_f32(np.nextafter(e, np.float32(-np.inf)), s.i_max) < k
    np.testing.assert_array_equal(h.cpu().numpy(), oracle.hist8_f32(x_np, s.i_max).astype(np.int64))


def test_range_nonfinite():
    x_np = np.ones(1000, np.float32)
    x_np[999] = np.inf
    x = dev(x_np)
    sc = new_sc(0.0)
    L.roix_range(ptr(x), x_np.size, ptr(sc), st())
    assert read_sc(sc).err & L.ERR_NONFINITE


# ---------------------------------------------------------------------------- a2 histogram, a3 Otsu
def test_histogram_u16_full_range_and_accumulate():
    rng = np.random.default_rng(5)
    x_np = np.concatenate([rng.normal(400, 60, 500000).clip(0, 4095), rng.integers(0, 65536, 300000),
                           [65535, 16383, 16384, 0]]).astype(np.uint16)
    x = dev(x_np)
    sc = new_sc(1.0)
    h = torch.zeros(65536, dtype=torch.int64, device="cuda")
    for _ in range(2):
        L.roix_histogram(ptr(x), L.U16, x_np.size, ptr(sc), ptr(h), 65536, st())
    ref = oracle.hist_u16(x_np).astype(np.int64)
    np.testing.assert_array_equal(h.cpu().numpy(), 2 * ref)


@pytest.mark.parametrize("case", ["mode0", "mode350", "mode16300", "bimodal", "spread", "tiny"])
def test_histogram_u16_replicated_window(case):
    """k_hist_u16_rw counts values near each CTA's mode in a lane-banked copy of the bins: modes at
    the bottom of the value range, mid-range, at the top of the 16 K shared window (the replicated
    window reaching past it), two modes, a flat spread, and fewer groups than threads."""
    rng = np.random.default_rng(11)
    n = 3 if case == "tiny" else 24_000_017        # > 2 CTAs per SM x 1024 threads x 8 voxels x 2 steps
    if case == "mode0":
        x_np = np.abs(rng.normal(0, 40, n))
    elif case == "mode350":
        x_np = rng.normal(350, 70, n)
    elif case == "mode16300":
        x_np = rng.normal(16300, 90, n)
    elif case == "bimodal":
        x_np = np.where(rng.random(n) < 0.4, rng.normal(200, 40, n), rng.normal(2500, 100, n))
    elif case == "spread":
        x_np = rng.integers(0, 65536, n)
    else:
        x_np = np.array([7, 7, 65535])
    x_np = np.clip(x_np, 0, 65535).astype(np.uint16)
    x = dev(x_np)
    sc = new_sc(1.0)
    h = torch.zeros(65536, dtype=torch.int64, device="cuda")
    L.roix_histogram(ptr(x), L.U16, x_np.size, ptr(sc), ptr(h), 65536, st())
    assert read_sc(sc).err == 0
    np.testing.assert_array_equal(h.cpu().numpy(), oracle.hist_u16(x_np).astype(np.int64))


@pytest.mark.parametrize("seed", range(6))
def test_threshold_u16_vs_oracle(seed):
    rng = np.random.default_rng(seed)
    bg = rng.normal(rng.uniform(200, 800), rng.uniform(20, 80), 200000)
    fg = rng.normal(rng.uniform(1500, 3500), rng.uniform(40, 120), int(rng.integers(5000, 100000)))
    x_np = np.concatenate([bg, fg]).clip(0, 65535 if seed % 2 else 4095).astype(np.uint16)
    for pol in (0, 1):
        x, sc, h = gpu_threshold(x_np, eb=2.0, polarity=pol)
        s = read_sc(sc)
        hist = oracle.hist_u16(x_np)
        imax = oracle.imax_u16(hist)
        t8 = oracle.otsu2(oracle.hist8_from_u16(hist, imax))
        assert s.err == 0 and s.i_max == imax and s.t8 == t8 and s.polarity == pol
        # raw threshold: the first value whose norm8 exceeds t8
        assert oracle.norm8_u16(s.thr_u16, imax) > t8 >= oracle.norm8_u16(s.thr_u16 - 1, imax)


def test_threshold_degenerate():
    for v in (0, 7):
        x_np = np.full(1000, v, np.uint16)
        _, sc, _ = gpu_threshold(x_np)
        assert read_sc(sc).err & L.ERR_DEGENERATE
        with pytest.raises(oracle.Degenerate):
            h = oracle.hist_u16(x_np)
            oracle.otsu2(oracle.hist8_from_u16(h, oracle.imax_u16(h)))


def test_threshold_f32_vs_oracle():
    rng = np.random.default_rng(9)
    x_np = np.concatenate([rng.normal(0.02, 0.005, 400000), rng.uniform(0.3, 1.2, 90000)]).astype(np.float32)
    x, sc, h = gpu_threshold(x_np, rel_eb=1e-3)
    s = read_sc(sc)
    h8 = oracle.hist8_f32(x_np, oracle.imax_f32(x_np.max()))
    t8 = oracle.otsu2(h8)
    assert s.t8 == t8
    assert oracle.norm8_f32(s.thr_f32, s.i_max) > t8
    assert oracle.norm8_f32(np.nextafter(np.float32(s.thr_f32), np.float32(-np.inf)), s.i_max) <= t8


def _h8_cases(rng):
    cases = [np.bincount([0] * 7 + [128] * 7 + [255] * 7, minlength=256),          # S:174 spikes
             np.bincount([10] * 50 + [200] * 50, minlength=256),                    # S:173 (k = 3: 2 bins)
             np.bincount([5, 9, 9, 250], minlength=256)]
    for _ in range(12):                                                               # dense / sparse / modal
        cases.append(rng.integers(0, 1000, 256) * (rng.random(256) < rng.uniform(0.05, 1.0)))
    for _ in range(6):                                                                # three or four modes
        v = np.concatenate([rng.normal(rng.uniform(10, 245), rng.uniform(2, 20), int(rng.integers(1000, 200000)))
                            for _ in range(int(rng.integers(3, 5)))])
        cases.append(np.bincount(np.clip(np.rint(v), 0, 255).astype(np.int64), minlength=256))
    big = np.zeros(256, np.int64)
    big[[3, 60, 61, 200]] = [1 << 34, 1 << 33, 12345, (1 << 34) + 7]                 # N near 2^35 (C5)
    cases.append(big)
    cases.append(np.full(256, 1 << 26, np.int64))                                     # uniform (symmetric)
    return cases


@pytest.mark.parametrize("classes", [2, 3])
def test_threshold_multi_vs_oracle(classes):
    """NEXT-3: roix_threshold_multi on 256-bin norm8 histograms (the fp32 form)
    against the exact exhaustive oracle -- spikes, ties, sparse and multi-modal histograms, counts near
    2^35 -- for both polarities; fewer populated bins than classes -> DEGENERATE."""
    rng = np.random.default_rng(31 + classes)
    x_np = np.concatenate([rng.normal(0.02, 0.005, 4000), rng.uniform(0.3, 1.2, 900)]).astype(np.float32)
    for h8 in _h8_cases(rng):
        try:
            want = oracle.multi_otsu(list(h8), classes)
        except oracle.Degenerate:
            want = None
        for pol in (0, 1):
            _, sc, _ = gpu_threshold(x_np, rel_eb=1e-3)
            h = torch.from_numpy(np.asarray(h8, np.int64)).cuda()
            L.roix_threshold_multi(ptr(h), 256, L.F32, pol, classes, ptr(sc), st())
            s = read_sc(sc)
            if want is None:
                assert s.err & L.ERR_DEGENERATE
                continue
            assert s.err == 0
            got = tuple((s.t8_all >> (8 * k)) & 255 for k in range(classes - 1))
            assert got == want, (got, want)
            assert s.t8 == (want[0] if pol == 0 else want[-1])
            assert s.thr_f32 == s.edges[s.t8 + 1]


def test_threshold_multi_u16_raw_hist():
    """classes = 3 from a raw 65536-bin histogram (the u16 form: I_max and the norm8 fold on the GPU)."""
    rng = np.random.default_rng(77)
    x_np = np.concatenate([rng.normal(400, 60, 300000), rng.normal(1800, 90, 60000),
                           rng.normal(3100, 120, 40000)]).clip(0, 4095).astype(np.uint16)
    for pol in (0, 1):
        x = dev(x_np)
        sc = new_sc(2.0)
        L.roix_resolve(ptr(sc), L.U16, 0.0, st())
        h = torch.zeros(65536, dtype=torch.int64, device="cuda")
        L.roix_histogram(ptr(x), L.U16, x_np.size, ptr(sc), ptr(h), 65536, st())
        L.roix_threshold_multi(ptr(h), 65536, L.U16, pol, 3, ptr(sc), st())
        s = read_sc(sc)
        hist = oracle.hist_u16(x_np)
        imax = oracle.imax_u16(hist)
        t1, t2 = oracle.multi_otsu(oracle.hist8_from_u16(hist, imax), 3)
        assert s.err == 0 and s.i_max == imax and (s.t8_all & 255, s.t8_all >> 8) == (t1, t2)
        t8 = t1 if pol == 0 else t2
        assert s.t8 == t8 and oracle.norm8_u16(s.thr_u16, imax) > t8 >= oracle.norm8_u16(s.thr_u16 - 1, imax)


# ------------------------------------------------ NEXT-3 per-frame thresholds (uint16 frame stacks)
FRAME_SHAPES = [(1, 1, 1), (3, 5, 7), (4, 9, 13), (6, 33, 31), (5, 32, 32), (3, 40, 1390), (7, 17, 100), (2, 64, 512),
                (130, 3, 5)]


def _frame_stack(rng, shape):
    Z, Y, X = shape
    base = rng.uniform(300, 3000, Z)[:, None, None]
    x = rng.normal(base, 40, shape)
    yy, xx = np.indices((Y, X))
    blob = ((yy - Y / 2) ** 2 / max(Y / 3, 1) ** 2 + (xx - X / 2) ** 2 / max(X / 4, 1) ** 2) < 1
    x[:, blob] += rng.uniform(1500, 20000, Z)[:, None]
    x[:, 0, 0] = 0                                      # every frame has >= 2 populated bins
    return np.clip(x, 0, 65535).astype(np.uint16)


def _frames_gpu(x_np, pol, classes, se=4):
    Z, Y, X = x_np.shape
    x = dev(x_np)
    g = L.Geom(Z, Y, X, 0, Z)
    sc = new_sc(1.0)
    L.roix_resolve(ptr(sc), L.U16, 0.0, st())
    h = torch.zeros(Z * 65536, dtype=torch.int64, device="cuda")
    L.roix_histogram_frames(ptr(x), ctypes.byref(g), ptr(sc), ptr(h), st())
    fr = torch.full((4 * Z,), -1, dtype=torch.int32, device="cuda")
    L.roix_threshold_frames(ptr(h), Z, pol, classes, ptr(sc), ptr(fr), st())
    o = torch.full(((x_np.size + 31) // 32 + 4,), -1, dtype=torch.int32, device="cuda")
    runs = torch.full((Z * Y,), -1, dtype=torch.int32, device="cuda")
    ws = torch.empty(L.roix_morph_workspace(g), dtype=torch.uint8, device="cuda")
    L.roix_morph_frames(ptr(x), ctypes.byref(g), se, None, None, ptr(fr), ptr(sc), ptr(o), ptr(runs), ptr(ws),
                        ws.numel(), st())
    s = read_sc(sc)
    return s, h.cpu().numpy().reshape(Z, 65536), fr.cpu().numpy().view(np.uint32).reshape(Z, 4), o, ws


@pytest.mark.parametrize("shape", FRAME_SHAPES)
@pytest.mark.parametrize("classes", [2, 3])
@pytest.mark.parametrize("se", [4, 6])
def test_frames_vs_oracle(shape, classes, se):
    """roix_histogram_frames / roix_threshold_frames / roix_morph_frames against the oracle's per-frame
    statement: frame sizes that are not multiples of 8 voxels (unaligned frame starts), frames smaller
    than a 1024-voxel warp iteration, 16-byte groups straddling frames, both polarities."""
    rng = np.random.default_rng(abs(hash((shape, classes, "frames"))) % 2 ** 32)
    x_np = _frame_stack(rng, shape)
    Z = shape[0]
    for pol in (0, 1):
        try:
            ft = oracle.frame_thresholds(x_np, classes, pol)
        except oracle.Degenerate:
            s, *_ = _frames_gpu(x_np, pol, classes)
            assert s.err & L.ERR_DEGENERATE
            continue
        s, h, fr, o, ws = _frames_gpu(x_np, pol, classes, se)
        assert s.err == 0
        for z in range(Z):
            np.testing.assert_array_equal(h[z], oracle.hist_u16(x_np[z]).astype(np.int64))
            imax, ts, t8 = ft[z]
            thr, g8, g8all, gimax = fr[z]
            assert gimax == imax and g8 == t8
            assert tuple((g8all >> (8 * k)) & 255 for k in range(classes - 1)) == ts
            assert oracle.norm8_u16(thr, imax) > t8 >= oracle.norm8_u16(thr - 1, imax)
        m = np.concatenate([oracle.binarize(x_np[z:z + 1], ft[z][0], ft[z][2], pol) for z in range(Z)])
        if se == 6:   # the 3-D opening reads the mask k_binarize wrote (the 2-D one binarises its rows itself)
            np.testing.assert_array_equal(words_to_mask(ws[: ((x_np.size + 31) // 32) * 4].view(torch.int32),
                                                        x_np.size).reshape(shape), m)
        np.testing.assert_array_equal(words_to_mask(o, x_np.size).reshape(shape), oracle.opening(m, se))


@pytest.mark.parametrize("shape", [(1, 1, 1), (3, 5, 7), (2, 4, 8), (5, 33, 31), (4, 40, 1390), (130, 3, 5)])
def test_background_vs_oracle(shape):
    """NEXT-3 roix_background: SUB / REV / ADD against the oracle, frames that are
    and are not whole 16-byte units, out-of-place and in place."""
    rng = np.random.default_rng(abs(hash((shape, "bg"))) % 2 ** 32)
    x_np = rng.integers(0, 65536, shape).astype(np.uint16)
    B_np = rng.integers(0, 65536, shape[1:]).astype(np.uint16)
    Z, Y, X = shape
    g = L.Geom(Z, Y, X, 0, Z)
    B = dev(B_np)
    for op, name in ((L.BG_SUB, "sub"), (L.BG_REV, "rev"), (L.BG_ADD, "add")):
        want = oracle.background(x_np, B_np, name)
        x = dev(x_np)
        out = torch.full((x_np.size + 8,), -1, dtype=torch.int16, device="cuda")
        L.roix_background(ptr(x), ptr(B), ctypes.byref(g), op, ptr(out), st())
        torch.cuda.synchronize()
        np.testing.assert_array_equal(host_u16(out)[: x_np.size].reshape(shape), want)
        assert np.all(out.cpu().numpy()[x_np.size:] == -1)
        L.roix_background(ptr(x), ptr(B), ctypes.byref(g), op, ptr(x), st())   # in place
        torch.cuda.synchronize()
        np.testing.assert_array_equal(host_u16(x).reshape(shape), want)


def test_frames_degenerate():
    x_np = np.stack([np.arange(64, dtype=np.uint16).reshape(8, 8) * 50, np.full((8, 8), 7, np.uint16)])
    s, *_ = _frames_gpu(x_np, 0, 2)
    assert s.err & L.ERR_DEGENERATE


# ------------------------------------------------------------------------- a4 + a5 binarise + open
MORPH_SHAPES = [(1, 1, 1), (1, 1, 40), (2, 3, 5), (3, 5, 7), (5, 33, 65), (7, 64, 64), (9, 17, 100),
                (4, 70, 139), (3, 20, 1390), (11, 9, 256), (6, 40, 96), (33, 8, 32),
                (5, 17, 768), (9, 40, 512), (3, 3, 1024), (130, 5, 256),
                # whole-row 3-D kernel (X % 32 == 0, W = X/32 a power of two <= 128): every segment width,
                # ragged row tiles, several z-chunks
                (17, 13, 128), (19, 7, 2048), (3, 5, 4096), (20, 37, 512), (18, 11, 64), (40, 3, 32),
                # in-plane register-row kernel (32 <= X, W + 1 <= 512 words): C3's row width, the widest
                # row it takes, the first it leaves to the shared-memory kernel, rows of one word + 1 bit
                (2, 9, 13900), (2, 3, 16352), (2, 3, 16353), (4, 7, 33), (3, 4, 31),
                # several plane chunks (binarised on one stream, opened on another): chunk starts on word
                # boundaries after 4, 8 and 1 planes
                (16, 20, 1390), (24, 7, 100), (13, 5, 64),
                # register-row opening corner cases: one-row and two-row planes, a 128-word row
                (5, 1, 100), (4, 2, 64), (3, 3, 4096), (6, 1, 33)]


def _morph_gpu(x_np, thr, pol, se):
    Z, Y, X = x_np.shape
    x = dev(x_np)
    sc = new_sc(1.0)
    s = read_sc(sc)
    s.polarity = pol
    if x_np.dtype == np.uint16:
        s.thr_u16 = thr
    else:
        s.thr_f32 = thr
    write_sc(sc, s)
    n = x_np.size
    o = torch.full(((n + 31) // 32 + 4,), -1, dtype=torch.int32, device="cuda")   # garbage-initialised
    runs = torch.full((Z * Y,), -1, dtype=torch.int32, device="cuda")
    g = L.Geom(Z, Y, X, 0, Z)
    ws = torch.empty(L.roix_morph_workspace(g), dtype=torch.uint8, device="cuda")
    L.roix_morph(ptr(x), dtype_code(x_np), ctypes.byref(g), se, None, None, ptr(sc), ptr(o), ptr(runs), ptr(ws),
                 ws.numel(), st())
    assert read_sc(sc).err == 0
    return o, runs


def _runs_per_row(mask3):
    Z, Y, X = mask3.shape
    m = mask3.reshape(Z * Y, X).astype(np.int8)
    d = np.diff(np.concatenate([np.zeros((Z * Y, 1), np.int8), m], axis=1), axis=1)
    return (d == 1).sum(axis=1)


@pytest.mark.parametrize("shape", MORPH_SHAPES)
@pytest.mark.parametrize("se", [6, 4])
@pytest.mark.parametrize("dt", ["u16", "f32"])
def test_morph_random_masks(shape, se, dt):
    rng = np.random.default_rng(abs(hash((shape, se, dt))) % 2 ** 32)
    for p, pol in [(0.75, 0), (0.6, 1), (0.9, 0)]:
        m = rng.random(shape) < p
        if dt == "u16":
            x_np = np.where(m, rng.integers(1000, 4000, shape), rng.integers(0, 999, shape)).astype(np.uint16)
            thr = 1000
        else:
            x_np = np.where(m, rng.uniform(0.5, 1.0, shape), rng.uniform(-1.0, 0.4999, shape)).astype(np.float32)
            thr = np.float32(0.5)
        mm = m if pol == 0 else ~m
        ref = oracle.opening(mm.astype(np.uint8), se)
        o, runs = _morph_gpu(x_np, thr, pol, se)
        n = x_np.size
        got = words_to_mask(o, n).reshape(shape)
        np.testing.assert_array_equal(got, ref)
        w = o.cpu().numpy().view(np.uint32)
        if n % 32:
            assert w[n // 32] >> (n % 32) == 0           # pad bits zero (G-16)
        np.testing.assert_array_equal(runs.cpu().numpy(), _runs_per_row(ref))


def _crosses(rng, shape, per_row, columns=False):
    """Planes of isolated 3x3 crosses (each survives the in-plane opening whole; `columns`: the same
    crosses in every plane, which survive the 3-D opening) -- rows with a few short runs, several of
    them inside one 32-bit word -- over a dense random band (rows with many runs)."""
    Z, Y, X = shape
    m = np.zeros(shape, bool)
    for z in range(Z):
        if columns and z:
            m[z] = m[0]
        else:
            for _ in range(max(1, int(per_row * Y / 3))):
                y, x = rng.integers(1, Y - 1), rng.integers(1, X - 1)
                m[z, y - 1:y + 2, x] = True
                m[z, y, x - 1:x + 2] = True
    for z in range(Z):
        m[z, : Y // 4] |= rng.random((Y // 4, X)) < 0.8
    return m


@pytest.mark.parametrize("shape,se", [((2, 12, 13900), 4), ((3, 20, 1390), 4), ((4, 12, 33), 4), ((2, 8, 16352), 4),
                                      ((16, 12, 1390), 4), ((11, 9, 96), 4),
                                      ((3, 11, 64), 4), ((2, 10, 100), 4), ((2, 9, 16400), 4), ((3, 8, 20), 4),
                                      ((3, 12, 1024), 6), ((4, 10, 2048), 6), ((3, 8, 4096), 6), ((3, 9, 96), 6)])
def test_morph_run_slots_vs_oracle(shape, se):
    """roix_morph_slots: row_runs of every row and, for rows with 1..32 runs, the run records (x0, x1
    exclusive) against the runs of the oracle's opening -- se = 4: register-row kernel (X >= 32,
    W + 1 <= 512), shared-memory kernel (W >= 512), rows shorter than a word; se = 6: the 3-D openings,
    which write row_runs and no records."""
    rng = np.random.default_rng(sum(shape))
    Z, Y, X = shape
    rs = 32
    for per_row in (0.5, 4.0, 12.0):
        m = _crosses(rng, shape, per_row, columns=se == 6)
        x_np = np.where(m, 3000, 100).astype(np.uint16)
        ref = oracle.opening(m.astype(np.uint8), se).astype(bool)
        x = dev(x_np)
        sc = new_sc(1.0)
        s = read_sc(sc)
        s.thr_u16 = 1000
        write_sc(sc, s)
        n = x_np.size
        o = torch.full(((n + 31) // 32 + 4,), -1, dtype=torch.int32, device="cuda")
        runs = torch.full((Z * Y,), -1, dtype=torch.int32, device="cuda")
        slots = torch.full((Z * Y * rs * 2,), -1, dtype=torch.int32, device="cuda")
        g = L.Geom(Z, Y, X, 0, Z)
        ws = torch.empty(L.roix_morph_workspace(g), dtype=torch.uint8, device="cuda")
        L.roix_morph_slots(ptr(x), L.U16, ctypes.byref(g), se, None, None, ptr(sc), ptr(o), ptr(runs), ptr(slots),
                           rs, ptr(ws), ws.numel(), st())
        sv = read_sc(sc)
        assert sv.err == 0
        np.testing.assert_array_equal(words_to_mask(o, n).reshape(shape), ref)
        got_runs = runs.cpu().numpy()
        np.testing.assert_array_equal(got_runs, _runs_per_row(ref))
        if sv.run_slots == 0:                     # the kernel wrote no records (X < 32 path)
            continue
        assert sv.run_slots == rs
        sl = slots.cpu().numpy().view(np.uint32).reshape(Z * Y, rs, 2)
        rows = ref.reshape(Z * Y, X).astype(np.int8)
        checked = 0
        for r in range(Z * Y):
            k = got_runs[r]
            if not 0 < k <= rs:
                continue
            d = np.diff(np.concatenate([[0], rows[r], [0]]))
            x0, x1 = np.nonzero(d == 1)[0], np.nonzero(d == -1)[0]
            np.testing.assert_array_equal(sl[r, :k, 0], x0)
            np.testing.assert_array_equal(sl[r, :k, 1], x1)
            checked += 1
        assert checked > 0


@pytest.mark.parametrize("thr", [0, 1, 1000, 0x7fff, 0x8000, 0x8001, 0xfffe, 0xffff, 0x10000])
@pytest.mark.parametrize("pol", [0, 1])
def test_binarize_every_u16_value(thr, pol):
    """The uint16 compare (two voxels per 32-bit word, SWAR) against a plain compare, exhaustively: every
    uint16 value, thresholds on both sides of 2^15 and past the range, both polarities."""
    vals = np.arange(65536, dtype=np.uint32)
    x_np = np.stack([vals.astype(np.uint16), vals[::-1].astype(np.uint16)]).reshape(2, 256, 256)
    x = dev(x_np)
    sc = new_sc(1.0)
    s = read_sc(sc)
    s.thr_u16 = thr
    s.polarity = pol
    write_sc(sc, s)
    g = L.Geom(2, 256, 256, 0, 2)
    pw = 256 * 256 // 32
    out = torch.full((2 * pw,), -1, dtype=torch.int32, device="cuda")
    L.roix_binarize_planes(ptr(x), L.U16, ctypes.byref(g), 0, 2, ptr(sc), ptr(out), st())
    torch.cuda.synchronize()
    ref = x_np.astype(np.uint32) >= thr
    if pol:
        ref = ~ref
    np.testing.assert_array_equal(out.cpu().numpy().view(np.uint32), oracle.pack_bits(ref.reshape(-1).astype(np.uint8)))


def test_binarize_planes_halo_layout():
    rng = np.random.default_rng(2)
    shape = (6, 13, 37)
    x_np = rng.integers(0, 2000, shape).astype(np.uint16)
    x = dev(x_np)
    sc = new_sc(1.0)
    s = read_sc(sc)
    s.thr_u16 = 1000
    write_sc(sc, s)
    g = L.Geom(*shape, 0, shape[0])
    pw = (13 * 37 + 31) // 32
    out = torch.full((3 * pw,), -1, dtype=torch.int32, device="cuda")
    L.roix_binarize_planes(ptr(x), L.U16, ctypes.byref(g), 2, 3, ptr(sc), ptr(out), st())
    torch.cuda.synchronize()
    for p in range(3):
        ref = oracle.pack_bits((x_np[2 + p] >= 1000).astype(np.uint8))
        np.testing.assert_array_equal(out[p * pw:(p + 1) * pw].cpu().numpy().view(np.uint32), ref)


# --------------------------------------------------------------------------------- a6 + a7 label
LABEL_SHAPES = [(1, 1, 1), (1, 1, 70), (2, 3, 5), (4, 9, 33), (6, 17, 64), (10, 10, 10), (3, 31, 97), (5, 40, 130),
                # rows longer than the register path (W > 128 words): the batched long-row run extraction
                (2, 5, 4500), (1, 3, 13900)]


def _label_gpu(mask, conn, min_size, with_runs, inplace=True, labels=True, cap=None):
    Z, Y, X = mask.shape
    n = mask.size
    o = mask_to_words(mask.astype(np.uint8))
    g = L.Geom(Z, Y, X, 0, Z)
    if cap is None:
        cap = max(1, Z * Y * ((X + 1) // 2))
    wsb = L.roix_label_workspace(g, cap)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    cmin = torch.full((cap,), -7, dtype=torch.int64, device="cuda")
    csz = torch.full((cap,), -7, dtype=torch.int64, device="cuda")
    ckp = torch.full((cap,), 9, dtype=torch.uint8, device="cuda")
    lab = torch.empty(n, dtype=torch.int64, device="cuda") if labels else None
    K = o if inplace else torch.full_like(o, -1)
    runs = None
    if with_runs:
        m3 = mask.reshape(Z * Y, X).astype(np.int8)
        d = np.diff(np.concatenate([np.zeros((Z * Y, 1), np.int8), m3], axis=1), axis=1)
        runs = torch.from_numpy((d == 1).sum(axis=1).astype(np.int32)).cuda()
    out = L.LabelOut(K.data_ptr(), cmin.data_ptr(), csz.data_ptr(), ckp.data_ptr(), cap,
                     lab.data_ptr() if labels else None)
    sc = new_sc(1.0)
    L.roix_label(ptr(o), ptr(runs), ctypes.byref(g), conn, min_size, cap, ptr(ws), wsb, ctypes.byref(out), ptr(sc),
                 st())
    s = read_sc(sc)
    nc = int(s.n_components)
    return s, K, cmin[:nc].cpu().numpy(), csz[:nc].cpu().numpy(), ckp[:nc].cpu().numpy(), lab


@pytest.mark.parametrize("conn", [6, 18, 26, 4, 8])
@pytest.mark.parametrize("shape", LABEL_SHAPES)
def test_label_random_vs_oracle(conn, shape):
    rng = np.random.default_rng(abs(hash((conn, shape))) % 2 ** 32)
    for p, min_size, with_runs in [(0.3, 1, False), (0.5, 3, True), (0.7, 10, True)]:
        mask = (rng.random(shape) < p).astype(np.uint8)
        s, K, cmin, csz, ckp, lab = _label_gpu(mask, conn, min_size, with_runs)
        assert s.err == 0
        comp, rmin, rsz = oracle.label(mask, conn)
        kept, rK = oracle.filter_components(comp, rsz, min_size)
        np.testing.assert_array_equal(cmin, rmin.astype(np.int64))
        np.testing.assert_array_equal(csz, rsz.astype(np.int64))
        np.testing.assert_array_equal(ckp, kept)
        np.testing.assert_array_equal(words_to_mask(K, mask.size).reshape(shape), rK)
        exp = np.full(mask.size, -1, np.int64)
        fg = comp.ravel() != np.iinfo(np.uint32).max
        exp[fg] = rmin[comp.ravel()[fg]].astype(np.int64)
        np.testing.assert_array_equal(lab.cpu().numpy(), exp)
        assert s.n_kept == int(kept.sum())


@pytest.mark.parametrize("conn", [6, 26, 8])
@pytest.mark.parametrize("shape", [(1, 1, 1), (2, 3, 5), (5, 17, 65), (9, 40, 512), (33, 8, 32), (4, 70, 139)])
def test_label_keep_largest_vs_oracle(conn, shape):
    """NEXT-3 keep-largest: only the largest component survives, ties to the
    smallest min index; the table still lists every component (comp_kept one-hot)."""
    rng = np.random.default_rng(abs(hash((conn, shape, "largest"))) % 2 ** 32)
    masks = [(rng.random(shape) < p).astype(np.uint8) for p in (0.2, 0.45)] + [np.zeros(shape, np.uint8)]
    tie = np.zeros(shape, np.uint8)                  # two single-voxel components: the first one wins
    tie.reshape(-1)[[0, tie.size - 1]] = 1
    masks.append(tie)
    for mask in masks:
        s, K, cmin, csz, ckp, _ = _label_gpu(mask, conn, L.KEEP_LARGEST, True)
        assert s.err == 0
        comp, rmin, rsz = oracle.label(mask, conn)
        kept, rK = oracle.keep_largest(comp, rsz)
        np.testing.assert_array_equal(cmin, rmin.astype(np.int64))
        np.testing.assert_array_equal(ckp, kept)
        np.testing.assert_array_equal(words_to_mask(K, mask.size).reshape(shape), rK)
        assert s.n_kept == int(kept.sum())


@pytest.mark.parametrize("conn", [6, 18, 26, 4, 8])
@pytest.mark.parametrize("cap", [1 << 20, 1 << 23], ids=["ub4K", "ub16K"])
def test_label_union_blocks_vs_oracle(conn, cap):
    """Both union-block sizes of k_union_local (4 K runs below run_capacity 2^23, 16 K runs from 2^23:
    the configuration the full-size C3/C4/C5 steps run in) against the oracle's BFS, on masks with
    ~10^5-10^6 runs, so that many blocks and cross-block pairs occur (k_label.cu)."""
    rng = np.random.default_rng(1000 + conn + (cap >> 20))
    shape = (24, 160, 256)
    for p in (0.3, 0.55):
        mask = (rng.random(shape) < p).astype(np.uint8)
        s, K, cmin, csz, ckp, lab = _label_gpu(mask, conn, 3, True, cap=cap)
        assert s.err == 0 and s.n_runs > 4 * (16384 if cap >= 1 << 23 else 4096)
        comp, rmin, rsz = oracle.label(mask, conn)
        kept, rK = oracle.filter_components(comp, rsz, 3)
        np.testing.assert_array_equal(cmin, rmin.astype(np.int64))
        np.testing.assert_array_equal(csz, rsz.astype(np.int64))
        np.testing.assert_array_equal(ckp, kept)
        np.testing.assert_array_equal(words_to_mask(K, mask.size).reshape(shape), rK)
        exp = np.full(mask.size, -1, np.int64)
        fg = comp.ravel() != np.iinfo(np.uint32).max
        exp[fg] = rmin[comp.ravel()[fg]].astype(np.int64)
        np.testing.assert_array_equal(lab.cpu().numpy(), exp)


def test_label_not_inplace_and_checkerboard():
    z, y, x = np.indices((6, 8, 40))
    cb = ((z + y + x) % 2 == 0).astype(np.uint8)
    for conn, ncomp in [(6, cb.sum()), (18, 1), (26, 1), (4, cb.sum()), (8, 6)]:
        s, K, cmin, csz, ckp, _ = _label_gpu(cb, conn, 2, False, inplace=False, labels=False)
        assert s.n_components == ncomp
        exp = oracle.filter_components(*[oracle.label(cb, conn)[i] for i in (0, 2)], 2)[1]
        np.testing.assert_array_equal(words_to_mask(K, cb.size).reshape(cb.shape), exp)


def test_label_capacity_error():
    mask = np.ones((2, 4, 64), np.uint8)
    mask[:, :, ::2] = 0                                  # 256 runs
    o = mask_to_words(mask)
    g = L.Geom(2, 4, 64, 0, 2)
    wsb = L.roix_label_workspace(g, 100)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    out = L.LabelOut(o.data_ptr(), None, None, None, 0, None)
    sc = new_sc(1.0)
    L.roix_label(ptr(o), None, ctypes.byref(g), 6, 1, 100, ptr(ws), wsb, ctypes.byref(out), ptr(sc), st())
    s = read_sc(sc)
    assert s.err & L.ERR_CAPACITY and s.n_runs == 256


# ---------------------------------------------------------------------------------- a8 extract
@pytest.mark.parametrize("n", [1, 31, 1000, 8192, 8193, 100003, 1 << 20])
@pytest.mark.parametrize("dt", ["u16", "f32"])
def test_extract_vs_oracle(n, dt):
    rng = np.random.default_rng(n)
    K = (rng.random(n) < rng.uniform(0.05, 0.9)).astype(np.uint8)
    K[: min(n, 40)] = 1
    if dt == "u16":
        x_np, eb = rng.integers(0, 65536, n).astype(np.uint16), 2.0
    else:
        x_np, eb = rng.normal(0, 3, n).astype(np.float32), 0.01
    x = dev(x_np)
    sc = new_sc(eb)
    L.roix_resolve(ptr(sc), dtype_code(x_np), 0.0, st())
    kw = mask_to_words(K)
    ref = oracle.extract(x_np, K, eb)
    out = torch.full((n + 8,), -1, dtype=torch.int16 if dt == "u16" else torch.int32, device="cuda")
    wsb = L.roix_extract_workspace(n)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    L.roix_extract(ptr(x), dtype_code(x_np), n, ptr(kw), ptr(sc), ptr(out), n, None, ptr(ws), wsb, st())
    s = read_sc(sc)
    assert s.err == 0 and s.count == ref.size
    got = out[: ref.size].cpu().numpy()
    np.testing.assert_array_equal(got.view(np.uint16) if dt == "u16" else got, ref)
    # capacity: writes stop at capacity and the error bit is set
    cap = ref.size // 2
    out2 = torch.full((n + 8,), -1, dtype=out.dtype, device="cuda")
    sc2 = new_sc(eb)
    L.roix_resolve(ptr(sc2), dtype_code(x_np), 0.0, st())
    L.roix_extract(ptr(x), dtype_code(x_np), n, ptr(kw), ptr(sc2), ptr(out2), cap, None, ptr(ws), wsb, st())
    s2 = read_sc(sc2)
    if ref.size > cap:
        assert s2.err & L.ERR_CAPACITY
    got2 = out2.cpu().numpy()
    got2 = got2.view(np.uint16) if dt == "u16" else got2
    np.testing.assert_array_equal(got2[:cap], ref[:cap])
    assert np.all(out2.cpu().numpy()[cap:] == -1)


def _runs_mask(rng, n, mean_run, p_on):
    """1-D masks made of x-runs: alternating off / on stretches of geometric lengths (mean_run), so
    16-byte groups are mostly fully kept or empty, with run ends at every phase."""
    out = np.zeros(n, np.uint8)
    i, on = 0, rng.random() < p_on
    while i < n:
        L = int(rng.geometric(1.0 / mean_run))
        if on:
            out[i:i + L] = 1
        i += L
        on = not on if rng.random() < 0.9 else on
    return out


@pytest.mark.parametrize("dt", ["u16", "f32"])
@pytest.mark.parametrize("n", [1, 37, 1024, 1031, 32768, 32768 + 1000, 100_003, 1 << 20, 3_000_017])
def test_extract_runs_masks_vs_oracle(n, dt):
    """roix_extract on run-structured masks (the shape of every phantom's K: long x-runs), at every
    16-byte phase of the output (offset 0..7 / 0..3), for every quantiser mode (s = 1, 2^k, other
    integers, non-integer), with capacity overflow: the vector stores (aligned groups, pairs of fully
    kept groups) and the element path (run ends, chunk ends) against oracle.extract."""
    rng = np.random.default_rng(n + (7 if dt == "f32" else 0))
    ebs = [0.5, 2.0, 4.0, 1.5, 0.75] if dt == "u16" else [0.01]   # s = 1, 4, 8, 3, 1.5
    for mean_run, p_on, holes in [(300, 0.5, 0), (40, 0.5, 0), (5, 0.5, 0), (2000, 0.8, 0), (2000, 0.8, 0.003)]:
        K = _runs_mask(rng, n, mean_run, p_on)
        if holes:   # isolated one-voxel gaps inside long runs (C3's noise holes): rows mixing both store forms
            K[rng.random(n) < holes] = 0
        if dt == "u16":
            x_np = rng.integers(0, 65536, n).astype(np.uint16)
        else:
            x_np = rng.normal(0, 3, n).astype(np.float32)
        x = dev(x_np)
        kw = mask_to_words(K)
        wsb = L.roix_extract_workspace(n)
        ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
        for eb in ebs:
            ref = oracle.extract(x_np, K, eb)
            for off in ([0, 1, 3, 5, 7] if dt == "u16" else [0, 1, 2, 3]):
                for capacity in (off + ref.size, off + ref.size // 2 + 1):
                    sc = new_sc(eb)
                    L.roix_resolve(ptr(sc), dtype_code(x_np), 0.0, st())
                    offd = torch.tensor([off], dtype=torch.int64, device="cuda")
                    buf = torch.full((n + off + 16,), -1, dtype=torch.int16 if dt == "u16" else torch.int32,
                                     device="cuda")
                    L.roix_extract(ptr(x), dtype_code(x_np), n, ptr(kw), ptr(sc), ptr(buf), capacity, ptr(offd),
                                   ptr(ws), wsb, st())
                    s = read_sc(sc)
                    got = buf.cpu().numpy()
                    got = got.view(np.uint16) if dt == "u16" else got
                    lim = min(ref.size, capacity - off)
                    np.testing.assert_array_equal(got[off:off + lim], ref[:lim],
                                                  err_msg="run %d eb %g off %d cap %d" % (mean_run, eb, off, capacity))
                    assert np.all(buf.cpu().numpy()[:off] == -1) and np.all(buf.cpu().numpy()[capacity:] == -1)
                    if off + ref.size > capacity:
                        assert s.err & L.ERR_CAPACITY
                    else:
                        assert s.err == 0 and s.count == ref.size


# ---------------------------------------------------------- a8 extract from the labelling's runs
def _blobby(rng, shape, p, run):
    """Masks whose x-runs are mostly long (runs of `run` voxels merged at random phases)."""
    Z, Y, X = shape
    base = rng.random((Z, Y, X // run + 2)) < p
    m = np.repeat(base, run, axis=2)
    sh = rng.integers(0, run, (Z, Y))
    out = np.empty(shape, np.uint8)
    for z in range(Z):
        for y in range(Y):
            out[z, y] = m[z, y, sh[z, y]: sh[z, y] + X]
    return out


@pytest.mark.parametrize("shape", [(1, 1, 1), (3, 7, 33), (6, 17, 64), (9, 40, 512), (4, 24, 2048), (5, 13, 1000),
                                   (2, 3, 9000)])
@pytest.mark.parametrize("dt", ["u16", "f32"])
def test_extract_runs_vs_oracle(shape, dt):
    """roix_extract_runs (the pipeline's a8) writes exactly oracle.extract(x, K) for the K that the
    labelling kept, at any stream offset (all 16-byte phases) and with capacity overflow."""
    rng = np.random.default_rng(abs(hash((shape, dt))) % 2 ** 32)
    n = int(np.prod(shape))
    for mask, min_size, conn in [(_blobby(rng, shape, 0.6, 37), 5, 6), ((rng.random(shape) < 0.5).astype(np.uint8), 2, 26),
                                 (np.ones(shape, np.uint8), 1, 6), (np.zeros(shape, np.uint8), 1, 6)]:
        Z, Y, X = shape
        g = L.Geom(Z, Y, X, 0, Z)
        cap = max(1, Z * Y * ((X + 1) // 2))
        wsb = L.roix_label_workspace(g, cap)
        ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
        o = mask_to_words(mask)
        out = L.LabelOut(o.data_ptr(), None, None, None, 0, None)
        sc = new_sc(1.0)
        L.roix_label(ptr(o), None, ctypes.byref(g), conn, min_size, cap, ptr(ws), wsb, ctypes.byref(out), ptr(sc), st())
        comp, rmin, rsz = oracle.label(mask, conn)
        _, rK = oracle.filter_components(comp, rsz, min_size)
        if dt == "u16":
            x_np, eb = rng.integers(0, 65536, shape).astype(np.uint16), 2.0
        else:
            x_np, eb = rng.normal(0, 3, shape).astype(np.float32), 0.01
        ref = oracle.extract(x_np.ravel(), rK.ravel(), eb)
        x = dev(x_np)
        for off, capacity in [(0, n), (3, n + 3), (5, n + 5), (7, n + 7), (1, ref.size // 2 + 1)]:
            sc2 = new_sc(eb)
            L.roix_resolve(ptr(sc2), dtype_code(x_np), 0.0, st())
            offd = torch.tensor([off], dtype=torch.int64, device="cuda")
            buf = torch.full((n + 16,), -1, dtype=torch.int16 if dt == "u16" else torch.int32, device="cuda")
            L.roix_extract_runs(ptr(x), dtype_code(x_np), ctypes.byref(g), cap, ptr(ws), wsb, ptr(sc2), ptr(buf),
                                capacity, ptr(offd), st())
            s2 = read_sc(sc2)
            got = buf.cpu().numpy()
            got = got.view(np.uint16) if dt == "u16" else got
            if off + ref.size > capacity:
                assert s2.err & L.ERR_CAPACITY
                lim = capacity - off
                np.testing.assert_array_equal(got[off:capacity], ref[:lim])
            else:
                assert s2.err == 0 and s2.count == ref.size
                np.testing.assert_array_equal(got[off:off + ref.size], ref)
            raw = buf.cpu().numpy()
            assert np.all(raw[:off] == -1) and np.all(raw[min(capacity, off + ref.size):] == -1)


# ------------------------------------------------------------------- NEXT-1 row spans
def _spans_gpu(x_np, K, eb, z0=0, gz=None, span_cap=None, code_cap=None):
    Z, Y, X = x_np.shape
    g = L.Geom(Z, Y, X, z0, gz if gz is not None else Z)
    wsb = L.roix_row_spans_workspace(g)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    rows = Z * Y
    scap = rows if span_cap is None else span_cap
    ccap = x_np.size if code_cap is None else code_cap
    spans = torch.full((max(scap, 1) * 2 + 2,), -1, dtype=torch.int64, device="cuda")   # 16-byte records
    codes = torch.full((max(ccap, 1) + 8,), -1, dtype=torch.int16 if x_np.dtype == np.uint16 else torch.int32,
                       device="cuda")
    counts = torch.zeros(2, dtype=torch.int64, device="cuda")
    sc = new_sc(eb)
    L.roix_resolve(ptr(sc), dtype_code(x_np), 0.0, st())
    kw = mask_to_words(K)
    x = dev(x_np)
    L.roix_row_spans(ptr(kw), ptr(x), dtype_code(x_np), ctypes.byref(g), ptr(sc), ptr(spans), scap, ptr(codes), ccap,
                     ptr(counts), ptr(ws), wsb, st())
    s = read_sc(sc)
    ns, nc = (int(v) for v in counts.cpu().numpy())
    sp = spans.cpu().numpy()
    rec = np.stack([sp[0:2 * ns:2], sp[1:2 * ns:2] & 0xffffffff, sp[1:2 * ns:2] >> 32], axis=1) if ns else \
        np.zeros((0, 3), np.int64)
    cd = codes.cpu().numpy()
    return s, rec, (cd.view(np.uint16) if x_np.dtype == np.uint16 else cd), ns, nc, sp


@pytest.mark.parametrize("shape", [(1, 1, 1), (2, 3, 5), (3, 7, 33), (4, 9, 64), (2, 5, 1000), (3, 40, 512),
                                   (2, 3, 2100)])
@pytest.mark.parametrize("dt", ["u16", "f32"])
def test_row_spans_vs_oracle(shape, dt):
    rng = np.random.default_rng(abs(hash((shape, dt, "spans"))) % 2 ** 32)
    for K in (_blobby(rng, shape, 0.3, 29), (rng.random(shape) < 0.05).astype(np.uint8), np.zeros(shape, np.uint8),
              np.ones(shape, np.uint8)):
        if dt == "u16":
            x_np, eb = rng.integers(0, 65536, shape).astype(np.uint16), 2.0
        else:
            x_np, eb = rng.normal(0, 3, shape).astype(np.float32), 0.01
        rs, rc = oracle.row_spans(x_np, K, eb)
        s, rec, cd, ns, nc, _ = _spans_gpu(x_np, K, eb)
        assert s.err == 0
        assert ns == len(rs) and nc == rc.size
        np.testing.assert_array_equal(rec, rs)
        np.testing.assert_array_equal(cd[:nc], rc)


def test_row_spans_global_rows_and_capacity():
    rng = np.random.default_rng(11)
    shape = (3, 6, 40)
    K = (rng.random(shape) < 0.3).astype(np.uint8)
    x_np = rng.integers(0, 4096, shape).astype(np.uint16)
    rs, rc = oracle.row_spans(x_np, K, 1.0)
    # a slab starting at global plane 5: row indices are global (z0 * Y + local row)
    s, rec, cd, ns, nc, _ = _spans_gpu(x_np, K, 1.0, z0=5, gz=12)
    assert s.err == 0
    np.testing.assert_array_equal(rec[:, 0], rs[:, 0] + 5 * shape[1])
    np.testing.assert_array_equal(cd[:nc], rc)
    # capacities: error bit, nothing written past either capacity
    s, rec, cd, ns, nc, sp = _spans_gpu(x_np, K, 1.0, span_cap=3, code_cap=10)
    assert s.err & L.ERR_CAPACITY and ns == len(rs) and nc == rc.size
    np.testing.assert_array_equal(sp[0:6:2], rs[:3, 0])
    assert np.all(sp[6:] == -1)
    np.testing.assert_array_equal(cd[:10], rc[:10])
    assert np.all(cd.view(np.int16)[10:] == -1)


# ------------------------------------------------------ NEXT-2 greedy quantiser (Steps 1-5)
def _greedy_gpu(D, E, qmax=65535):
    n = D.size
    wsb = L.roix_greedy_workspace(n)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    d = dev(D) if n else torch.empty(8, dtype=torch.int16, device="cuda")
    q = torch.full((max(n, 1) + 8,), -1, dtype=torch.int16, device="cuda")
    gb = torch.full(((n + 31) // 32 + 2,), -1, dtype=torch.int32, device="cuda")
    ng = torch.zeros(1, dtype=torch.int64, device="cuda")
    L.roix_greedy_quantize(ptr(d), n, float(E), qmax, ptr(q), ptr(gb), ptr(ng), ptr(ws), wsb, st())
    torch.cuda.synchronize()
    return q.cpu().numpy().view(np.uint16)[:n], words_to_mask(gb, n), int(ng.item())


@pytest.mark.parametrize("E", [0, 0.4, 1, 2, 17.5, 300, 70000])
def test_greedy_vs_oracle(E):
    rng = np.random.default_rng(int(E * 7) % 2 ** 31)
    seqs = [np.zeros(0, np.uint16), np.array([5, 5, 7], np.uint16), np.full(1000, 77, np.uint16),
            rng.integers(0, 65536, 5000).astype(np.uint16),
            np.clip(np.cumsum(rng.integers(-3, 4, 100003)) + 30000, 0, 65535).astype(np.uint16),
            np.clip(rng.normal(2500, 100, 70001), 0, 65535).astype(np.uint16),
            np.repeat(rng.integers(0, 4000, 300), rng.integers(1, 200, 300)).astype(np.uint16)]
    for D in seqs:
        rq, rg = oracle.greedy_quantize(D, E)
        q, g, ng = _greedy_gpu(D, E)
        np.testing.assert_array_equal(q, rq)
        np.testing.assert_array_equal(g, rg)
        assert ng == int(rg.sum())


def test_greedy_8bit_spec_examples():
    for D, E, Q in [([10, 12, 20], 2, [11, 11, 20]), ([255, 251], 3, [253, 253]), ([0, 255], 200, [127, 127])]:
        q, g, ng = _greedy_gpu(np.array(D, np.uint16), E, 255)
        np.testing.assert_array_equal(q, Q)


# ------------------------------------- NEXT-4 decode and confusion
def _untouched(a, dt):
    """the -1 fill of the output buffers (int16 -1 for u16, -1.0 for f32) is still there"""
    return bool(np.all(a.view(np.int16) == -1)) if dt == "u16" else bool(np.all(a == -1.0))


def _decode_gpu(K, codes_np, dt, eb, n=None, ncodes=None):
    n = K.size if n is None else n
    npdt = np.uint16 if dt == "u16" else np.float32
    sc = new_sc(eb)
    L.roix_resolve(ptr(sc), L.U16 if dt == "u16" else L.F32, 0.0, st())
    kw = mask_to_words(K)
    codes = dev(np.concatenate([codes_np, np.zeros(8, codes_np.dtype)]))
    ncodes = codes_np.size if ncodes is None else ncodes
    xh = torch.full((n + 16,), -1, dtype=torch.int16 if dt == "u16" else torch.float32, device="cuda")
    wsb = L.roix_decode_workspace(n)
    ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device="cuda")
    L.roix_decode(ptr(kw), ptr(codes), ncodes, L.U16 if dt == "u16" else L.F32, n, ptr(sc), ptr(xh), ptr(ws), wsb,
                  st())
    s = read_sc(sc)
    out = xh.cpu().numpy()
    return s, (out.view(np.uint16) if dt == "u16" else out), npdt


@pytest.mark.parametrize("n", [1, 33, 8192, 8193, 100003, 1 << 20])
@pytest.mark.parametrize("dt", ["u16", "f32"])
def test_decode_mask_vs_oracle(n, dt):
    rng = np.random.default_rng(n * 3 + (dt == "f32"))
    shape = (1, 1, n)
    for K in (_blobby(rng, shape, 0.3, 40) if n > 64 else (rng.random(shape) < 0.5).astype(np.uint8),
              (rng.random(shape) < 0.03).astype(np.uint8), np.zeros(shape, np.uint8), np.ones(shape, np.uint8)):
        if dt == "u16":
            x_np, eb = rng.integers(0, 65536, shape).astype(np.uint16), 2.0
        else:
            x_np, eb = rng.normal(0, 3, shape).astype(np.float32), 0.01
        codes = oracle.extract(x_np, K, eb)
        want = oracle.decode_mask(K, codes, oracle.step(eb), x_np.dtype).reshape(-1)
        s, got, _ = _decode_gpu(K, codes, dt, eb)
        assert s.err == 0
        np.testing.assert_array_equal(got[:n], want)
        assert _untouched(got[n:], dt)   # nothing past n


@pytest.mark.parametrize("eb", [0.5, 0.75, 1.25, 3.0, 1000.0])
def test_decode_u16_steps(eb):
    """Integer and fractional steps (G-37) on every code value, through the mask form."""
    codes = np.arange(65536, dtype=np.uint16)
    K = np.ones((1, 1, 65536), np.uint8)
    s, got, _ = _decode_gpu(K, codes, "u16", eb)
    assert s.err == 0
    np.testing.assert_array_equal(got[:65536], oracle.decode_value(codes, oracle.step(eb), np.uint16))


def test_decode_f32_codes_extremes():
    rng = np.random.default_rng(9)
    codes = np.concatenate([rng.integers(-(1 << 23), 1 << 23, 50000), [0, 1, -1, 1 << 23, -(1 << 23)]]).astype(np.int32)
    K = np.ones((1, 1, codes.size), np.uint8)
    for eb in (1e-3, 0.37, 3e-7, 12.5):
        s, got, _ = _decode_gpu(K, codes, "f32", eb)
        assert s.err == 0
        np.testing.assert_array_equal(got[:codes.size], oracle.decode_value(codes, oracle.step(eb), np.float32))


def test_decode_capacity_error():
    K = np.ones((1, 1, 1000), np.uint8)
    codes = np.arange(1000, dtype=np.uint16)
    s, got, _ = _decode_gpu(K, codes, "u16", 1.0, ncodes=999)
    assert s.err & L.ERR_CAPACITY
    assert np.all(got.view(np.int16) == -1)


def _decode_spans_gpu(rec, codes_np, shape, dt, eb, z0=0, counts=None, span_cap=None, code_cap=None):
    Z, Y, X = shape
    g = L.Geom(Z, Y, X, z0, z0 + Z)
    sc = new_sc(eb)
    L.roix_resolve(ptr(sc), L.U16 if dt == "u16" else L.F32, 0.0, st())
    m = len(rec)
    sp = np.zeros((max(m, 1), 2), np.int64)
    if m:
        sp[:m, 0] = rec[:, 0]
        sp[:m, 1] = rec[:, 1] | (rec[:, 2] << 32)
    spans = torch.from_numpy(sp.reshape(-1).copy()).cuda()
    codes = dev(np.concatenate([codes_np, np.zeros(8, codes_np.dtype)]))
    cnt = torch.tensor(counts if counts is not None else [m, codes_np.size], dtype=torch.int64, device="cuda")
    xh = torch.full((Z * Y * X + 16,), -1, dtype=torch.int16 if dt == "u16" else torch.float32, device="cuda")
    wsb = L.roix_decode_spans_workspace(g)
    ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device="cuda")
    L.roix_decode_spans(ptr(spans), m if span_cap is None else span_cap, ptr(codes),
                        codes_np.size if code_cap is None else code_cap, ptr(cnt), L.U16 if dt == "u16" else L.F32,
                        ctypes.byref(g), ptr(sc), ptr(xh), ptr(ws), wsb, st())
    s = read_sc(sc)
    out = xh.cpu().numpy()
    return s, (out.view(np.uint16) if dt == "u16" else out)


@pytest.mark.parametrize("shape", [(1, 1, 1), (2, 3, 5), (3, 7, 33), (4, 9, 64), (2, 5, 1000), (3, 40, 512),
                                   (2, 3, 2100)])
@pytest.mark.parametrize("dt", ["u16", "f32"])
def test_decode_spans_vs_oracle(shape, dt):
    """roix_row_spans -> roix_decode_spans on the GPU against the oracle's row_spans -> decode_spans."""
    rng = np.random.default_rng(abs(hash((shape, dt, "dspans"))) % 2 ** 32)
    n = int(np.prod(shape))
    for K in (_blobby(rng, shape, 0.3, 29), (rng.random(shape) < 0.05).astype(np.uint8), np.zeros(shape, np.uint8),
              np.ones(shape, np.uint8)):
        if dt == "u16":
            x_np, eb = rng.integers(0, 65536, shape).astype(np.uint16), 2.0
        else:
            x_np, eb = rng.normal(0, 3, shape).astype(np.float32), 0.01
        rs, rc = oracle.row_spans(x_np, K, eb)
        want = oracle.decode_spans(rs, rc, shape, oracle.step(eb), x_np.dtype).reshape(-1)
        s0, rec, cd, ns, nc, _ = _spans_gpu(x_np, K, eb)
        assert s0.err == 0
        s, got = _decode_spans_gpu(rec, cd[:nc], shape, dt, eb)
        assert s.err == 0
        np.testing.assert_array_equal(got[:n], want)
        assert _untouched(got[n:], dt)


def test_decode_spans_lossless_slab_and_format_errors():
    rng = np.random.default_rng(21)
    shape = (3, 6, 40)
    x_np = rng.integers(0, 60000, shape).astype(np.uint16)
    K = (rng.random(shape) < 0.2).astype(np.uint8)
    rs, rc = oracle.row_spans(x_np, K, 0.5)   # s = 1: lossless on the span columns (AC3 analogue)
    rec = rs.copy()
    rec[:, 0] += 4 * shape[1]                  # a slab at global plane 4: records carry global rows
    s, got = _decode_spans_gpu(rec, rc, shape, "u16", 0.5, z0=4)
    assert s.err == 0
    got = got[:x_np.size].reshape(-1, shape[2])
    for i, xs, xe in rs:
        np.testing.assert_array_equal(got[i, xs:xe], x_np.reshape(-1, shape[2])[i, xs:xe])
    # format errors: nothing decoded
    bad = [rec[::-1].copy(), rec.copy(), rec.copy(), rec.copy()]
    bad[1][0, 2] = shape[2] + 1                # x_end past the row
    bad[2][0, 1] = bad[2][0, 2]                # empty record
    bad[3][0, 0] = 0                           # row outside the slab
    for b in bad:
        s, got = _decode_spans_gpu(b, rc, shape, "u16", 0.5, z0=4)
        assert s.err & L.ERR_FORMAT
        assert np.all(got.view(np.int16) == -1)
    s, got = _decode_spans_gpu(rec, rc, shape, "u16", 0.5, z0=4, counts=[len(rec), rc.size + 1])
    assert s.err & L.ERR_FORMAT                # section lengths disagree with counts[1]
    s, got = _decode_spans_gpu(rec, rc, shape, "u16", 0.5, z0=4, code_cap=rc.size - 1)
    assert s.err & L.ERR_CAPACITY
    s, got = _decode_spans_gpu(rec, rc, shape, "u16", 0.5, z0=4, span_cap=len(rec) - 1)
    assert s.err & L.ERR_CAPACITY


def _confusion_gpu(pred, truth):
    n = pred.size
    c = torch.full((4,), -1, dtype=torch.int64, device="cuda")
    pw, tw = mask_to_words(pred), mask_to_words(truth)    # keep both alive across the call
    L.roix_confusion(ptr(pw), ptr(tw), n, ptr(c), st())
    torch.cuda.synchronize()
    return tuple(int(v) for v in c.cpu().numpy())


@pytest.mark.parametrize("n", [0, 1, 31, 32, 127, 128, 129, 100003, 1 << 22])
def test_confusion_vs_oracle(n):
    rng = np.random.default_rng(n)
    for p, t in ((0.5, 0.5), (0.02, 0.9), (1.0, 0.0)):
        pred = (rng.random(n) < p).astype(np.uint8)
        truth = (rng.random(n) < t).astype(np.uint8)
        got = _confusion_gpu(pred, truth)
        assert got == oracle.confusion(pred, truth)
        m = L.roix_overlap_metrics(got)
        want = oracle.overlap_metrics(*got)
        for k in L.METRICS:
            np.testing.assert_allclose(m[k], want[k], rtol=1e-15, atol=0, equal_nan=True, err_msg=k)


def test_confusion_ignores_pad_bits():
    n = 70
    w = torch.full((8,), -1, dtype=torch.int32, device="cuda")   # every bit set, pad bits too
    z = torch.zeros(8, dtype=torch.int32, device="cuda")
    c = torch.zeros(4, dtype=torch.int64, device="cuda")
    L.roix_confusion(ptr(w), ptr(z), n, ptr(c), st())
    torch.cuda.synchronize()
    assert tuple(c.cpu().numpy()) == (0, n, 0, 0)

