"""-m gpu: BASELINE.json's full-size configs (C3 128x9700x13900 frames, C4 2048^3, C5 4096x4096x2048),
run in the launch configuration bench.py times (Pipeline defaults: run capacity n/256, 16 K-run union
blocks), compared bit for bit with the streaming oracle (oracle/stream.py):
the histogram, I_max and t8, the opened mask o, the whole component table (min index, size, kept),
the kept mask K, the count and the code stream -- o, K and the stream as BLAKE2b digests of every
256 MiB chunk of their byte layouts.

The oracle's result is stored in tests/golden/fullsize_<cfg>.json, written by
scripts/make_fullsize_golden.py (synth + oracle only) and valid for the oracle and generator sources
it names (their hashes are checked here).  The output contract checked end to end is the paper's
|Q - D| <= E through a1's exact quantiser, on the volumes the paper's multi-GB stacks
 stand in for."""
import ctypes
import gc
import json
import os

import numpy as np
import pytest
import torch

import synth
from gpu_util import ptr, st
from oracle.digest import digest_buffer, first_mismatch, source_hashes, table_digest
from paper_2602_15917_b200 import Pipeline
from paper_2602_15917_b200 import _lib as L

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module", autouse=True)
def _build():
    from paper_2602_15917_b200 import build

    build.build()
    synth.build()


def _golden(name):
    path = os.path.join(GOLDEN, "fullsize_%s.json" % name)
    assert os.path.exists(path), "missing %s: run scripts/make_fullsize_golden.py --config %s" % (path, name)
    g = json.load(open(path))
    assert g["sources"] == source_hashes(), (
        "%s was written for other oracle / generator sources: re-run scripts/make_fullsize_golden.py" % path)
    return g


def _host_bytes(t, nbytes):
    return t.view(torch.uint8)[:nbytes].cpu().numpy()


def _same(got, want, what):
    k = first_mismatch(got, want)
    assert k is None, "%s differs from the oracle at chunk %s (256 MiB chunks)" % (what, k)


@pytest.mark.parametrize("name", ["C3", "C4", "C5"])
def test_fullsize_bitexact(name):
    g = _golden(name)
    cfg = synth.CONFIGS[name]
    assert g["shape"] == list(cfg.shape) and g["seed"] == cfg.seed
    gc.collect()
    torch.cuda.empty_cache()
    free, _ = torch.cuda.mem_get_info()
    if cfg.nbytes * 2.3 > free:
        pytest.skip("not enough device memory on this GPU")
    x = synth.generate(cfg)
    p = Pipeline(cfg.shape, cfg.dtype, eb=cfg.eb, conn=cfg.conn, se=cfg.se, min_size=cfg.min_size,
                 polarity=cfg.polarity)
    r = p.run(x)
    assert p.run_capacity >= 1 << 23             # the 16 K-run union blocks of the timed configuration
    n = cfg.n
    # a2, a3
    h = p.hist.cpu().numpy().view(np.uint64)
    assert int(h.sum()) == g["hist_sum"] == n
    assert table_digest(h, np.zeros(0, np.uint64), np.zeros(0, np.uint8)) == g["hist_digest"]
    assert r.i_max == g["i_max"] and r.t8 == g["t8"]
    # a4 + a5: o, recomputed into its own buffer (the pipeline's o became K in place)
    o = torch.full_like(p.o, -1)
    L.roix_morph(ptr(x), p.cdtype, ctypes.byref(p.geom), p.se, None, None, ptr(p.sc), ptr(o), None,
                 ptr(p.morph_ws), p.morph_ws.numel(), st())
    torch.cuda.synchronize()
    _same(digest_buffer(_host_bytes(o, n // 8)), g["o"], "o")
    del o
    # a6 + a7: the whole component table
    assert r.n_components == g["n_components"] and r.n_kept == g["n_kept"]
    cmin = r.comp_min.cpu().numpy().view(np.uint64)
    csz = r.comp_size.cpu().numpy().view(np.uint64)
    kept = r.comp_kept.cpu().numpy()
    if g["table"] is not None:
        np.testing.assert_array_equal(cmin, np.array(g["table"]["min_index"], np.uint64))
        np.testing.assert_array_equal(csz, np.array(g["table"]["size"], np.uint64))
        np.testing.assert_array_equal(kept, np.array(g["table"]["kept"], np.uint8))
    assert table_digest(cmin, csz, kept) == g["table_digest"]
    # K and a1 + a8: the kept mask and the code stream
    _same(digest_buffer(_host_bytes(r.keep_bits, n // 8)), g["K"], "K")
    assert r.count == g["count"]
    _same(digest_buffer(_host_bytes(r.codes, 2 * r.count)), g["stream"], "stream")
    del x, p, r
    gc.collect()
    torch.cuda.empty_cache()
