"""Pins of the NEXT-3 per-frame thresholds (oracle.frame_thresholds / pipeline(frames=True)): each
frame of a uint16 stack is thresholded as its own image, as in the paper's 2-D pipeline.

Anchors: a one-frame stack reduces to the whole-volume path; Eq. 1 is scale-free (norm8(c v) with
I_max c I equals norm8(v) with I_max I, the same rational 255 v / I), so frames that are integer
multiples of one frame get identical masks -- which a global threshold does not give; and with
in-plane morphology and labelling (se = 4, conn = 8) the stack's K is the concatenation of the
per-image pipelines' K."""
import numpy as np
import pytest

import oracle


def _frame(rng, Y=40, X=56, hi=6000):
    f = rng.normal(400, 40, (Y, X))
    yy, xx = np.indices((Y, X))
    f[(yy - Y / 2) ** 2 / (Y / 3) ** 2 + (xx - X / 2) ** 2 / (X / 4) ** 2 < 1] = rng.normal(hi, 150)
    return np.clip(f, 0, 65535).astype(np.uint16)


def test_single_frame_reduces_to_volume():
    rng = np.random.default_rng(1)
    x = _frame(rng)[None]
    for classes in (2, 3):
        a = oracle.pipeline(x, eb=2.0, conn=8, se=4, min_size=8, classes=classes, frames=True)
        b = oracle.pipeline(x, eb=2.0, conn=8, se=4, min_size=8, classes=classes)
        assert a["frames"][0][2] == b["t8"]
        np.testing.assert_array_equal(a["K"], b["K"])
        np.testing.assert_array_equal(a["stream"], b["stream"])


def test_scaled_frames_get_identical_masks():
    rng = np.random.default_rng(2)
    base = (_frame(rng, hi=3000) // 4).astype(np.uint16)
    x = np.stack([base * c for c in (1, 2, 3, 5)]).astype(np.uint16)
    ft = oracle.frame_thresholds(x)
    assert len({t8 for _, _, t8 in ft}) == 1
    r = oracle.pipeline(x, eb=1.0, conn=8, se=4, min_size=8, frames=True)
    for z in range(1, 4):
        np.testing.assert_array_equal(r["m"][z], r["m"][0])
    g = oracle.pipeline(x, eb=1.0, conn=8, se=4, min_size=8)
    assert not all(np.array_equal(g["m"][z], g["m"][0]) for z in range(1, 4))   # a global threshold differs


@pytest.mark.parametrize("polarity", [0, 1])
def test_stack_equals_per_image_pipelines(polarity):
    rng = np.random.default_rng(3 + polarity)
    x = np.stack([_frame(rng, hi=h) for h in (2500, 5000, 9000)])
    if polarity:
        x = (65535 - x).astype(np.uint16)
    r = oracle.pipeline(x, eb=2.0, conn=8, se=4, min_size=8, polarity=polarity, frames=True)
    per = [oracle.pipeline(x[z:z + 1], eb=2.0, conn=8, se=4, min_size=8, polarity=polarity) for z in range(3)]
    np.testing.assert_array_equal(r["K"], np.concatenate([p["K"] for p in per]))
    np.testing.assert_array_equal(r["stream"], np.concatenate([p["stream"] for p in per]))
    assert [t8 for _, _, t8 in r["frames"]] == [p["t8"] for p in per]


def test_degenerate_frame_raises():
    rng = np.random.default_rng(5)
    x = np.stack([_frame(rng), np.full((40, 56), 9, np.uint16)])
    with pytest.raises(oracle.Degenerate):
        oracle.frame_thresholds(x)
