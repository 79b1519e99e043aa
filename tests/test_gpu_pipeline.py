"""-m gpu: the whole path (paper_2602_15917_b200.Pipeline, every step through the C ABI) against the
composed oracle on the seeded synthetic phantoms of BASELINE.json's configs: C1 and C2 at full size,
C3 / C4 / C5 scaled down (same recipe, every length scaled) so the oracle finishes in seconds.
Full-size C3-C5 are covered by tests/test_gpu_fullsize.py (sampled / property checks)."""
import ctypes

import numpy as np
import pytest
import torch

import oracle
import synth
from gpu_util import dev, ptr, st, words_to_mask
from paper_2602_15917_b200 import Pipeline
from paper_2602_15917_b200 import _lib as L

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _build():
    from paper_2602_15917_b200 import build

    build.build()
    oracle.build()
    synth.build()


CASES = [synth.CONFIGS["C1"], synth.CONFIGS["C2"], synth.scaled("C3", 0.25, frames=4),
         synth.scaled("C4", 0.125), synth.scaled("C5", 0.125), synth.scaled("C4", 0.0625), synth.scaled("C1", 0.37)]


def _check(cfg, p, x, res, classes=2, keep="size"):
    x_np = synth.to_numpy(x, cfg)
    ref = oracle.pipeline(x_np, eb=cfg.eb or None, rel_eb=cfg.rel_eb or None, conn=cfg.conn, se=cfg.se,
                          min_size=cfg.min_size, polarity=cfg.polarity, classes=classes, keep=keep)
    s = res.scalars
    assert s.err == 0
    assert res.t8 == ref["t8"] and res.i_max == ref["i_max"] and res.eb == ref["eb"]
    if cfg.dtype == "u16":
        np.testing.assert_array_equal(p.hist.cpu().numpy(), ref["hist"].astype(np.int64))
    # o: re-run the fused binarise+open with the pipeline's threshold
    o = torch.full_like(p.o, -1)
    L.roix_morph(ptr(x), p.cdtype, ctypes.byref(p.geom), p.se, None, None, ptr(p.sc), ptr(o), None, ptr(p.morph_ws),
                 p.morph_ws.numel(), st())
    np.testing.assert_array_equal(words_to_mask(o, p.n).reshape(cfg.shape), ref["o"])
    np.testing.assert_array_equal(words_to_mask(res.keep_bits, p.n).reshape(cfg.shape), ref["K"])
    np.testing.assert_array_equal(res.comp_min.cpu().numpy(), ref["comp_min"].astype(np.int64))
    np.testing.assert_array_equal(res.comp_size.cpu().numpy(), ref["comp_size"].astype(np.int64))
    np.testing.assert_array_equal(res.comp_kept.cpu().numpy(), ref["kept"])
    assert res.count == ref["count"]
    got = res.codes.cpu().numpy()
    np.testing.assert_array_equal(got.view(np.uint16) if cfg.dtype == "u16" else got, ref["stream"])
    return ref


@pytest.mark.parametrize("extract", ["mask", "runs"])
@pytest.mark.parametrize("cfg", CASES, ids=lambda c: c.name)
def test_pipeline_vs_oracle(cfg, extract):
    x = synth.generate(cfg)
    p = Pipeline(cfg.shape, cfg.dtype, eb=cfg.eb, rel_eb=cfg.rel_eb, conn=cfg.conn, se=cfg.se,
                 min_size=cfg.min_size, polarity=cfg.polarity, extract=extract)
    res = p.run(x)
    ref = _check(cfg, p, x, res)
    # the step reduces the data (paper: spatial reduction 1.5x-8.5x)
    assert 0 < ref["count"] < p.n


@pytest.mark.parametrize("cfg", [synth.CONFIGS["C2"], synth.scaled("C4", 0.25), synth.scaled("C5", 0.25)],
                         ids=lambda c: c.name)
def test_pipeline_union_block_16k_vs_oracle(cfg):
    """run_capacity >= 2^23 selects k_union_local's 16 K-run union blocks -- the configuration of the
    full-size C3/C4/C5 steps the bench times (Pipeline sizes run_capacity = max(2^22, n/256)) -- here
    on volumes the oracle finishes in seconds, every artefact element by element."""
    x = synth.generate(cfg)
    p = Pipeline(cfg.shape, cfg.dtype, eb=cfg.eb, rel_eb=cfg.rel_eb, conn=cfg.conn, se=cfg.se,
                 min_size=cfg.min_size, polarity=cfg.polarity, run_capacity=1 << 23)
    res = p.run(x)
    assert p.run_capacity >= 1 << 23
    assert res.n_runs > 2 * 16384          # several union blocks, so cross-block pairs occur
    _check(cfg, p, x, res)


@pytest.mark.parametrize("shape,conn,se", [((6, 40, 64), 6, 6), ((5, 33, 256), 26, 6), ((4, 50, 100), 8, 4),
                                           ((3, 64, 2048), 18, 6), ((2, 30, 1000), 4, 4), ((4, 37, 1024), 6, 6),
                                           ((3, 21, 4096), 26, 6), ((5, 19, 2048), 6, 6)])
def test_pipeline_run_slots_vs_oracle(shape, conn, se):
    """The opening's run records (roix_morph_slots, 32 per row: the in-plane openings) feed a6 for
    rows with <= 32 runs; rows with more, and slabs whose opening writes none (3-D), are re-read
    from o.  Two-level volumes with random masks of several densities
    give rows of every run count on both sides of 32, in one volume; every artefact against the
    oracle."""
    from paper_2602_15917_b200.pipeline import Pipeline as P, run_slots_for

    rng = np.random.default_rng(sum(shape) + conn)
    for p in (0.55, 0.7, 0.85):
        m = rng.random(shape) < p
        m[:, : shape[1] // 3] &= rng.random((shape[0], shape[1] // 3, shape[2])) < 0.97   # blobby rows too
        xv = np.where(m, 3000, 100).astype(np.uint16)
        xv[0, 0, 0], xv[-1, -1, -1] = 3000, 100
        x = torch.from_numpy(xv.view(np.int16)).cuda()
        cfg = synth.Config("rand", shape, "u16", eb=2.0, conn=conn, se=se, min_size=3)
        pl = P(shape, "u16", eb=2.0, conn=conn, se=se, min_size=3)
        assert pl.rs == run_slots_for(shape, se)
        res = pl.run(x)
        assert res.scalars.run_slots == pl.rs   # the opening wrote run records of that width
        _check(cfg, pl, x, res)


def test_slab_generation_is_g_invariant():
    cfg = synth.scaled("C5", 0.0625)
    full = synth.generate(cfg)
    Z = cfg.shape[0]
    for G in (2, 4, 8):
        parts = [synth.generate(cfg, z0=g * Z // G, nz=(g + 1) * Z // G - g * Z // G) for g in range(G)]
        assert torch.equal(torch.cat(parts), full)


def test_determinism_repeated_runs():
    cfg = synth.scaled("C4", 0.0625)
    x = synth.generate(cfg)
    p = Pipeline(cfg.shape, cfg.dtype, eb=cfg.eb, conn=cfg.conn, se=cfg.se, min_size=cfg.min_size)
    first = p.run(x)
    codes0, k0 = first.codes.clone(), first.keep_bits.clone()
    t0 = (first.comp_min.clone(), first.comp_size.clone())
    for _ in range(5):
        r = p.run(x)
        assert torch.equal(r.codes, codes0) and torch.equal(r.keep_bits, k0)
        assert torch.equal(r.comp_min, t0[0]) and torch.equal(r.comp_size, t0[1])


def test_edge_cases():
    # degenerate: constant volume -> DEGENERATE error, raised
    x = dev(np.full((4, 8, 40), 9, np.uint16))
    p = Pipeline((4, 8, 40), "u16", eb=1.0)
    with pytest.raises(L.RoixError):
        p.run(x)
    # empty ROI after cleanup: a checkerboard of two levels opens to nothing -> count 0, valid
    z, y, xx = np.indices((4, 8, 40))
    cb = np.where((z + y + xx) % 2 == 0, 1000, 10).astype(np.uint16)
    r = Pipeline((4, 8, 40), "u16", eb=1.0).run(dev(cb))
    assert r.count == 0 and r.n_components == 0
    assert not words_to_mask(r.keep_bits, cb.size).any()
    # a single bright cube: kept iff its (opened) size reaches min_size -- boundary sizes min-1 / min
    v = np.full((6, 9, 41), 100, np.uint16)
    v[1:5, 2:6, 3:7] = 3000
    size = int(oracle.pipeline(v, eb=2.0, min_size=1)["comp_size"][0])    # 4^3 cube opens to 32 voxels
    assert size == 32
    for ms, kept in [(size, True), (size + 1, False)]:
        r = Pipeline(v.shape, "u16", eb=2.0, min_size=ms).run(dev(v))
        ref = oracle.pipeline(v, eb=2.0, min_size=ms)
        assert r.count == ref["count"] == (size if kept else 0)
    # all foreground except one voxel; ragged n (not a multiple of 8 or 32)
    v = np.full((3, 7, 13), 2000, np.uint16)
    v[1, 3, 6] = 5
    r = Pipeline(v.shape, "u16", eb=0.5, min_size=1).run(dev(v))
    ref = oracle.pipeline(v, eb=0.5, min_size=1)
    assert r.count == ref["count"]
    np.testing.assert_array_equal(r.codes.cpu().numpy().view(np.uint16), ref["stream"])


@pytest.mark.parametrize("cfg", [synth.CONFIGS["C1"], synth.CONFIGS["C2"], synth.scaled("C3", 0.25, frames=4),
                                 synth.scaled("C5", 0.125)], ids=lambda c: c.name)
def test_fused_histogram_binarize_equals_two_pass(cfg):
    """roix_histogram_binarize + roix_morph_prebinarized give exactly the two-pass result."""
    x = synth.generate(cfg)
    kw = dict(eb=cfg.eb, rel_eb=cfg.rel_eb, conn=cfg.conn, se=cfg.se, min_size=cfg.min_size, polarity=cfg.polarity)
    a = Pipeline(cfg.shape, cfg.dtype, fused=True, **kw)
    ra = a.run(x)
    b = Pipeline(cfg.shape, cfg.dtype, fused=False, **kw)
    rb = b.run(x)
    assert ra.scalars.spec_state in (2, 3)     # resolved, or fell back to the plain binarisation
    assert torch.equal(a.hist, b.hist) and ra.t8 == rb.t8
    assert torch.equal(ra.keep_bits, rb.keep_bits) and torch.equal(ra.codes, rb.codes)
    assert torch.equal(ra.comp_min, rb.comp_min) and torch.equal(ra.comp_size, rb.comp_size)


def test_fused_speculation_miss_falls_back():
    """A volume whose sampled rows are unrepresentative (objects only in the odd rows; the sample
    takes every 2nd row here): the window misses the exact threshold or the queue overflows, and the
    plain binarisation runs -- same result as the two-pass path and the oracle."""
    rng = np.random.default_rng(3)
    Z, Y, X = 64, 128, 256
    v = rng.normal(300, 30, (Z, Y, X))
    odd = v[:, 1::2, :]
    obj = rng.random(odd.shape) < 0.3
    odd[obj] = rng.normal(3000, 50, obj.sum())
    v[:, 1::2, :] = odd
    v = v.clip(0, 65535).astype(np.uint16)
    x = dev(v)
    for pol in (0, 1):
        kw = dict(eb=2.0, conn=6, se=6, min_size=4, polarity=pol)
        ra = Pipeline(v.shape, "u16", fused=True, **kw).run(x)
        rb = Pipeline(v.shape, "u16", fused=False, **kw).run(x)
        assert ra.scalars.spec_state == 3
        assert torch.equal(ra.keep_bits, rb.keep_bits) and torch.equal(ra.codes, rb.codes)
        ref = oracle.pipeline(v, eb=2.0, conn=6, se=6, min_size=4, polarity=pol)
        assert ra.count == ref["count"]


@pytest.mark.parametrize("cfg", [synth.CONFIGS["C1"], synth.scaled("C4", 0.0625), synth.scaled("C2", 0.25)],
                         ids=lambda c: c.name)
def test_pipeline_row_spans_vs_oracle(cfg):
    """NEXT-1 inside the pipeline: the row spans of K (the paper's geometry + pixel sections)."""
    x = synth.generate(cfg)
    p = Pipeline(cfg.shape, cfg.dtype, eb=cfg.eb, rel_eb=cfg.rel_eb, conn=cfg.conn, se=cfg.se,
                 min_size=cfg.min_size, polarity=cfg.polarity, spans=True)
    res = p.run(x)
    K = words_to_mask(res.keep_bits, p.n).reshape(cfg.shape)
    rs, rc = oracle.row_spans(synth.to_numpy(x, cfg), K, res.eb)
    rec, codes = p.row_spans()
    np.testing.assert_array_equal(rec.numpy(), rs)
    got = codes.cpu().numpy()
    np.testing.assert_array_equal(got.view(np.uint16) if cfg.dtype == "u16" else got, rc)
    # the spans cover K: at least as many codes as the kept voxels
    assert rc.size >= res.count


# ------------------------------------------------------------------ NEXT-4 reconstruction and quality
QCASES = [synth.CONFIGS["C1"], synth.CONFIGS["C2"], synth.scaled("C3", 0.25, frames=4), synth.scaled("C4", 0.0625),
          synth.scaled("C5", 0.0625)]


@pytest.mark.parametrize("cfg", QCASES, ids=lambda c: c.name)
def test_pipeline_decode_vs_oracle(cfg):
    """P:410-412 / S:359-367: both reconstructions of the pipeline's output (mask + code stream, and the
    paper's row spans) against the oracle's decode of the oracle's own K / stream / spans."""
    x = synth.generate(cfg)
    p = Pipeline(cfg.shape, cfg.dtype, eb=cfg.eb, rel_eb=cfg.rel_eb, conn=cfg.conn, se=cfg.se,
                 min_size=cfg.min_size, polarity=cfg.polarity, spans=True)
    res = p.run(x)
    x_np = synth.to_numpy(x, cfg)
    ref = oracle.pipeline(x_np, eb=cfg.eb or None, rel_eb=cfg.rel_eb or None, conn=cfg.conn, se=cfg.se,
                          min_size=cfg.min_size, polarity=cfg.polarity)
    npdt = np.uint16 if cfg.dtype == "u16" else np.float32
    s = oracle.step(ref["eb"])
    want = oracle.decode_mask(ref["K"], ref["stream"], s, npdt)
    got = p.decode()
    torch.cuda.synchronize()
    assert p.scalars().err == 0
    g = got.cpu().numpy()
    g = g.view(np.uint16) if cfg.dtype == "u16" else g
    np.testing.assert_array_equal(g, want)
    # the error bound on the ROI (G-37): integer steps for u16: eb exactly; fp32: |x - code s| <= s/2
    # exactly, plus half an ulp of x^ from the fp32 product
    K = ref["K"].astype(bool)
    d = np.abs(g.astype(np.float64) - x_np.astype(np.float64))[K]
    if cfg.dtype == "u16":
        assert d.size == 0 or d.max() <= ref["eb"]
    else:
        assert np.all(d <= s / 2 + np.spacing(np.abs(g[K])).astype(np.float64) / 2)
    rs, rc = oracle.row_spans(x_np, ref["K"], ref["eb"])
    want_sp = oracle.decode_spans(rs, rc, cfg.shape, s, npdt)
    got_sp = p.decode(from_spans=True)
    torch.cuda.synchronize()
    assert p.scalars().err == 0
    gs = got_sp.cpu().numpy()
    np.testing.assert_array_equal(gs.view(np.uint16) if cfg.dtype == "u16" else gs, want_sp)
    np.testing.assert_array_equal((gs.view(np.uint16) if cfg.dtype == "u16" else gs)[K], g[K])


@pytest.mark.parametrize("cfg", QCASES, ids=lambda c: c.name)
def test_quality_vs_ground_truth(cfg):
    """the confusion of K against the generator's ground truth (roix_confusion) equals the
    oracle's tally of the same masks; the segmentation is good on these phantoms (sanity, not a pin)."""
    tw = torch.empty(synth.truth_words(cfg) + 4, dtype=torch.int32, device="cuda")
    x = synth.generate(cfg, truth=tw)
    p = Pipeline(cfg.shape, cfg.dtype, eb=cfg.eb, rel_eb=cfg.rel_eb, conn=cfg.conn, se=cfg.se,
                 min_size=cfg.min_size, polarity=cfg.polarity, spans=True)
    res = p.run(x)
    q = p.quality(tw)
    K = words_to_mask(res.keep_bits, p.n)
    T = words_to_mask(tw, p.n)
    c = oracle.confusion(K, T)
    assert tuple(q["counts"].values()) == c
    want = oracle.overlap_metrics(*c)
    for k in L.METRICS:
        np.testing.assert_allclose(q[k], want[k], rtol=2e-16, equal_nan=True, err_msg=k)
    assert q["dsc"] > 0.9, q
    assert q["spatial_reduction_voxels"] == p.n / res.count
    assert 1.0 <= q["spatial_reduction"] <= q["spatial_reduction_voxels"]


def test_truth_slab_invariance():
    cfg = synth.scaled("C4", 0.0625)
    Z, Y, X = cfg.shape
    tw = torch.empty(synth.truth_words(cfg), dtype=torch.int32, device="cuda")
    synth.generate(cfg, truth=tw)
    full = words_to_mask(tw, cfg.n).reshape(cfg.shape)
    assert 0 < full.sum() < full.size
    for z0, nz in ((0, 3), (5, 7), (Z - 2, 2)):
        t = torch.empty(synth.truth_words(cfg, nz), dtype=torch.int32, device="cuda")
        synth.generate(cfg, z0=z0, nz=nz, truth=t)
        np.testing.assert_array_equal(words_to_mask(t, nz * Y * X).reshape(nz, Y, X), full[z0:z0 + nz])


# ------------------------------------------------------------------ NEXT-3 multi-Otsu in the pipeline
@pytest.mark.parametrize("cfg", [synth.CONFIGS["C1"], synth.CONFIGS["C2"], synth.scaled("C3", 0.25, frames=4),
                                 synth.scaled("C5", 0.0625)], ids=lambda c: c.name)
def test_pipeline_multi_otsu_vs_oracle(cfg):
    """classes = 3 end to end: every intermediate equals the oracle's (thresholds (t1, t2), K, table,
    stream); C2 is the multi-modal phantom the 2-class split under-segments (DESIGN.md NEXT-4)."""
    x = synth.generate(cfg)
    p = Pipeline(cfg.shape, cfg.dtype, eb=cfg.eb, rel_eb=cfg.rel_eb, conn=cfg.conn, se=cfg.se,
                 min_size=cfg.min_size, polarity=cfg.polarity, classes=3)
    res = p.run(x)
    ref = _check(cfg, p, x, res, classes=3)
    s = res.scalars
    assert (s.t8_all & 255, s.t8_all >> 8) == ref["thresholds"]


def test_sharded_multi_otsu_g_invariant():
    from paper_2602_15917_b200.sharded import run_simulated

    cfg = synth.scaled("C5", 0.0625)
    x = synth.generate(cfg)
    kw = dict(eb=cfg.eb, conn=cfg.conn, se=cfg.se, min_size=cfg.min_size, classes=3)
    one = Pipeline(cfg.shape, cfg.dtype, **kw).run(x)
    for G in (2, 4):
        states = run_simulated(x, G, **kw)
        for S in states:
            assert S.scalars().err == 0 and S.scalars().t8_all == one.scalars.t8_all
        codes = torch.cat([S.collect().codes for S in states])
        keep = np.concatenate([words_to_mask(S.collect().keep_bits, S.n) for S in states])
        assert torch.equal(codes, one.codes)
        np.testing.assert_array_equal(keep, words_to_mask(one.keep_bits, one_n(cfg)))


def one_n(cfg):
    return int(np.prod(cfg.shape))


# ------------------------------------------------------------------ NEXT-3 keep-largest in the pipeline
@pytest.mark.parametrize("cfg", [synth.CONFIGS["C1"], synth.scaled("C4", 0.0625), synth.scaled("C3", 0.25, frames=4)],
                         ids=lambda c: c.name)
def test_pipeline_keep_largest_vs_oracle(cfg):
    x = synth.generate(cfg)
    p = Pipeline(cfg.shape, cfg.dtype, eb=cfg.eb, rel_eb=cfg.rel_eb, conn=cfg.conn, se=cfg.se,
                 min_size=cfg.min_size, polarity=cfg.polarity, keep="largest")
    res = p.run(x)
    ref = _check(cfg, p, x, res, keep="largest")
    assert res.n_kept == 1 and ref["kept"].sum() == 1


def test_sharded_keep_largest_g_invariant():
    """The largest component crosses slab faces (C5's z-elongated objects): the merged sizes decide."""
    from paper_2602_15917_b200.sharded import run_simulated

    cfg = synth.scaled("C5", 0.0625)
    x = synth.generate(cfg)
    kw = dict(eb=cfg.eb, conn=cfg.conn, se=cfg.se, min_size=cfg.min_size, keep="largest")
    one = Pipeline(cfg.shape, cfg.dtype, **kw).run(x)
    ref = oracle.pipeline(synth.to_numpy(x, cfg), eb=cfg.eb, conn=cfg.conn, se=cfg.se, keep="largest")
    np.testing.assert_array_equal(words_to_mask(one.keep_bits, one_n(cfg)).reshape(cfg.shape), ref["K"])
    for G in (2, 4, 8):
        states = run_simulated(x, G, **kw)
        keep = np.concatenate([words_to_mask(S.collect().keep_bits, S.n) for S in states])
        np.testing.assert_array_equal(keep.reshape(cfg.shape), ref["K"])
        assert torch.equal(torch.cat([S.collect().codes for S in states]), one.codes)
        assert sum(S.scalars().n_kept for S in states) == 1


# ------------------------------------------------------------------ NEXT-3 per-frame thresholds
@pytest.mark.parametrize("classes", [2, 3])
def test_pipeline_frames_vs_oracle(classes):
    """C3-style detector frames (LOW polarity, se = 4, conn = 8) with per-frame thresholds, end to end."""
    cfg = synth.scaled("C3", 0.25, frames=6)
    x = synth.generate(cfg)
    p = Pipeline(cfg.shape, cfg.dtype, eb=cfg.eb, conn=cfg.conn, se=cfg.se, min_size=cfg.min_size,
                 polarity=cfg.polarity, classes=classes, frames=True)
    res = p.run(x)
    x_np = synth.to_numpy(x, cfg)
    ref = oracle.pipeline(x_np, eb=cfg.eb, conn=cfg.conn, se=cfg.se, min_size=cfg.min_size, polarity=cfg.polarity,
                          classes=classes, frames=True)
    assert res.scalars.err == 0
    got = p.frame_thresholds()
    assert [(f.i_max, f.t8) for f in got] == [(imax, t8) for imax, _, t8 in ref["frames"]]
    np.testing.assert_array_equal(words_to_mask(res.keep_bits, p.n).reshape(cfg.shape), ref["K"])
    np.testing.assert_array_equal(res.comp_min.cpu().numpy(), ref["comp_min"].astype(np.int64))
    c = res.codes.cpu().numpy()
    np.testing.assert_array_equal(c.view(np.uint16), ref["stream"])


def test_sharded_frames_g_invariant():
    from paper_2602_15917_b200.sharded import run_simulated

    cfg = synth.scaled("C3", 0.125, frames=8)
    x = synth.generate(cfg)
    kw = dict(eb=cfg.eb, conn=cfg.conn, se=cfg.se, min_size=cfg.min_size, polarity=cfg.polarity, frames=True)
    one = Pipeline(cfg.shape, cfg.dtype, **kw).run(x)
    for G in (2, 4):
        states = run_simulated(x, G, **kw)
        keep = np.concatenate([words_to_mask(S.collect().keep_bits, S.n) for S in states])
        np.testing.assert_array_equal(keep, words_to_mask(one.keep_bits, one_n(cfg)))
        assert torch.equal(torch.cat([S.collect().codes for S in states]), one.codes)


# ------------------------------------------------------------------ NEXT-3 background subtraction
@pytest.mark.parametrize("frames", [False, True])
def test_pipeline_background_vs_oracle(frames):
    """C3 detector frames with the flat field subtracted (REV: B - I, the sample's shadow turns bright,
    polarity HIGH), per-frame thresholds or not; the reconstruction adds the background back;
    segmentation quality against the phantom's ground truth."""
    cfg = synth.scaled("C3", 0.25, frames=4)
    tw = torch.empty(synth.truth_words(cfg) + 4, dtype=torch.int32, device="cuda")
    x = synth.generate(cfg, truth=tw)
    B = synth.flat_field(cfg)
    p = Pipeline(cfg.shape, cfg.dtype, eb=cfg.eb, conn=cfg.conn, se=cfg.se, min_size=cfg.min_size, polarity=0,
                 frames=frames, background=B, bg="rev", spans=True)
    res = p.run(x)
    x_np = synth.to_numpy(x, cfg)
    B_np = B.cpu().numpy().view(np.uint16)
    ref = oracle.pipeline(x_np, eb=cfg.eb, conn=cfg.conn, se=cfg.se, min_size=cfg.min_size, polarity=0,
                          frames=frames, background_ref=B_np, bg="rev")
    assert res.scalars.err == 0
    np.testing.assert_array_equal(words_to_mask(res.keep_bits, p.n).reshape(cfg.shape), ref["K"])
    np.testing.assert_array_equal(res.codes.cpu().numpy().view(np.uint16), ref["stream"])
    xh = p.decode()
    torch.cuda.synchronize()
    want = oracle.background(oracle.decode_mask(ref["K"], ref["stream"], oracle.step(cfg.eb), np.uint16), B_np, "rev")
    np.testing.assert_array_equal(xh.cpu().numpy().view(np.uint16), want)
    q = p.quality(tw)
    assert q["dsc"] > 0.95, q


def test_edge_cases_next_rows():
    """NEXT-3 edge cases: multi-Otsu with only two populated norm8 bins is DEGENERATE; keep-
    largest on an empty ROI keeps nothing; per-frame thresholds with a constant frame is DEGENERATE;
    SUB background with its reconstruction (min(65535, M + B)) against the oracle."""
    v = np.full((4, 8, 40), 100, np.uint16)
    v[1:3, 2:6, 5:30] = 3000
    with pytest.raises(L.RoixError):
        Pipeline(v.shape, "u16", eb=1.0, classes=3).run(dev(v))
    z, y, xx = np.indices((4, 8, 40))
    cb = np.where((z + y + xx) % 2 == 0, 1000, 10).astype(np.uint16)   # opens to nothing
    r = Pipeline(cb.shape, "u16", eb=1.0, keep="largest").run(dev(cb))
    assert r.count == 0 and r.n_kept == 0
    fr = np.stack([v[1], np.full((8, 40), 7, np.uint16)])
    with pytest.raises(L.RoixError):
        Pipeline(fr.shape, "u16", eb=1.0, frames=True, se=4, conn=8).run(dev(fr))
    rng = np.random.default_rng(4)
    B = rng.integers(50, 150, (8, 40)).astype(np.uint16)
    x = (v.astype(np.int64) + B[None]).clip(0, 65535).astype(np.uint16)
    p = Pipeline(x.shape, "u16", eb=2.0, min_size=8, background=dev(B), bg="sub")
    res = p.run(dev(x))
    ref = oracle.pipeline(x, eb=2.0, min_size=8, background_ref=B, bg="sub")
    np.testing.assert_array_equal(words_to_mask(res.keep_bits, p.n).reshape(x.shape), ref["K"])
    np.testing.assert_array_equal(res.codes.cpu().numpy().view(np.uint16), ref["stream"])
    xh = p.decode().cpu().numpy().view(np.uint16)
    want = oracle.background(oracle.decode_mask(ref["K"], ref["stream"], oracle.step(2.0), np.uint16), B, "add")
    np.testing.assert_array_equal(xh, want)
