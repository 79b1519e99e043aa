"""-m gpu: the z-slab sharded path (paper_2602_15917_b200.sharded, all exchanges simulated in one
process on one GPU) is G-invariant: for G = 2..8 slabs the concatenated outputs equal the 1-GPU
pipeline bit for bit (threshold, mask, component table, code stream), and the 1-GPU pipeline
equals the oracle (test_gpu_pipeline)."""
import numpy as np
import pytest
import torch

import oracle
import synth
from gpu_util import words_to_mask
from paper_2602_15917_b200 import Pipeline
from paper_2602_15917_b200.sharded import run_simulated

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _build():
    from paper_2602_15917_b200 import build

    build.build()
    synth.build()
    oracle.build()


CASES = [synth.CONFIGS["C1"], synth.scaled("C2", 0.25), synth.scaled("C4", 0.0625), synth.scaled("C5", 0.0625),
         synth.scaled("C3", 0.1, frames=8), synth.scaled("C1", 0.37)]


def _kw(cfg):
    return dict(eb=cfg.eb, rel_eb=cfg.rel_eb, conn=cfg.conn, se=cfg.se, min_size=cfg.min_size, polarity=cfg.polarity)


@pytest.mark.parametrize("cfg", CASES, ids=lambda c: c.name)
@pytest.mark.parametrize("G", [2, 3, 4, 8])
def test_sharded_equals_single(cfg, G):
    if cfg.shape[0] < 2 * G:
        pytest.skip("slabs need >= 2 planes")
    x = synth.generate(cfg)
    ref = Pipeline(cfg.shape, cfg.dtype, **_kw(cfg)).run(x)
    states = run_simulated(x, G, **_kw(cfg))
    n = int(np.prod(cfg.shape))
    masks, codes, cmin, csz, ckept = [], [], [], [], []
    for S in states:
        s = S.scalars()
        assert s.err == 0, hex(s.err)
        assert s.t8 == ref.t8 and s.i_max == ref.i_max and s.eb == ref.eb
        r = S.collect(s)
        masks.append(words_to_mask(r.keep_bits, S.n))
        codes.append(r.codes.cpu().numpy())
        cmin.append(r.comp_min.cpu().numpy())
        csz.append(r.comp_size.cpu().numpy())
        ckept.append(r.comp_kept.cpu().numpy())
        assert S.global_count == ref.count
    np.testing.assert_array_equal(np.concatenate(masks), words_to_mask(ref.keep_bits, n))
    np.testing.assert_array_equal(np.concatenate(codes), ref.codes.cpu().numpy())
    np.testing.assert_array_equal(np.concatenate(cmin), ref.comp_min.cpu().numpy())
    np.testing.assert_array_equal(np.concatenate(csz), ref.comp_size.cpu().numpy())
    np.testing.assert_array_equal(np.concatenate(ckept), ref.comp_kept.cpu().numpy())
    offs = [S.offset for S in states]
    assert offs == list(np.cumsum([0] + [int(S.scalars().count) for S in states[:-1]]))


def test_component_spanning_every_slab():
    """A rod along z through every slab plus small blobs cut by slab faces (G-31, H-6)."""
    v = np.full((32, 20, 64), 100, np.uint16)
    v[:, 8:12, 10:14] = 3000                     # spans all slabs
    v[7:9, 2:5, 40:44] = 3000                    # 2x3x4 blob straddling the 8-plane slab face
    v[15:18, 14:18, 50:55] = 3000
    x = torch.from_numpy(v.view(np.int16)).cuda()
    for conn in (6, 26):
        kw = dict(eb=2.0, conn=conn, se=6, min_size=20)
        ref = oracle.pipeline(v, eb=2.0, conn=conn, se=6, min_size=20)
        states = run_simulated(x, 4, **kw)
        got = np.concatenate([words_to_mask(S.collect().keep_bits, S.n) for S in states])
        np.testing.assert_array_equal(got.reshape(v.shape), ref["K"])
        tab = np.concatenate([S.collect().comp_min.cpu().numpy() for S in states])
        np.testing.assert_array_equal(tab, ref["comp_min"].astype(np.int64))
