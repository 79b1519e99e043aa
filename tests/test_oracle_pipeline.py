"""End-to-end sanity of the composed oracle (S:218 / AC5 S:566 analogue): on a phantom with well
separated bright objects on a noisy dark background the kept mask recovers the ground truth with
DSC >= 0.99, every kept voxel's code reconstructs within eb, and small objects are removed."""
import numpy as np


def _phantom(rng, shape=(24, 48, 56)):
    z, y, x = np.indices(shape)
    truth = np.zeros(shape, bool)
    for c, r in [((12, 14, 16), 8.5), ((10, 30, 38), 7.0)]:
        truth |= (z - c[0]) ** 2 + (y - c[1]) ** 2 + (x - c[2]) ** 2 <= r * r
    speck = np.zeros(shape, bool)
    speck[2:4, 40:42, 4:6] = True                      # 8-voxel object: below min_size
    lam = np.where(truth | speck, 2500.0, 400.0)
    vol = rng.normal(lam, np.sqrt(lam)).clip(0, 4095).astype(np.uint16)
    return vol, truth, speck


def test_pipeline_sphere_phantom(oracle_mod):
    rng = np.random.default_rng(0)
    vol, truth, speck = _phantom(rng)
    r = oracle_mod.pipeline(vol, eb=2.0, conn=6, se=6, min_size=64)
    K = r["K"].astype(bool)
    dsc = 2 * np.sum(K & truth) / (K.sum() + truth.sum())
    assert dsc >= 0.99
    assert not np.any(K & speck)
    assert r["count"] == K.sum() == r["comp_size"][r["kept"].astype(bool)].sum()
    xhat = r["stream"].astype(np.float64) * 4.0
    assert np.all(np.abs(vol[K].astype(np.float64) - xhat) <= 2.0)
    assert np.all(r["o"] <= r["m"]) and np.all(r["K"] <= r["o"])
    assert int(r["h8"].sum()) == vol.size


def test_pipeline_f32_low_polarity(oracle_mod):
    rng = np.random.default_rng(1)
    vol, truth, _ = _phantom(rng)
    x = (1.0 - vol.astype(np.float32) / 4095.0).astype(np.float32)   # dark objects on bright field
    r = oracle_mod.pipeline(x, rel_eb=1e-3, conn=26, se=6, min_size=64, polarity=1)
    K = r["K"].astype(bool)
    assert 2 * np.sum(K & truth) / (K.sum() + truth.sum()) >= 0.99
    s = np.float64(np.float32(2 * np.float32(r["eb"])))
    assert np.all(np.abs(x[K].astype(np.float64) - r["stream"] * s) <= np.float64(np.float32(r["eb"])))
