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


def test_distcomm_nccl_single_rank():
    """The torch.distributed (NCCL) exchange layer on the GPU: a one-rank process group runs
    ShardedPipeline through DistComm (histogram all-reduce, min/max, counts all-gather) and matches
    the 1-GPU pipeline.  (Several ranks need several GPUs; their exchanges are covered by the gloo
    test in test_sharded_host.py and by the simulated G-invariance above.)"""
    import socket

    import torch.distributed as dist

    from paper_2602_15917_b200.sharded import ShardedPipeline

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("nccl", init_method="tcp://127.0.0.1:%d" % port, rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        for cfg in (synth.scaled("C2", 0.25), synth.scaled("C4", 0.0625)):
            x = synth.generate(cfg)
            one = Pipeline(cfg.shape, cfg.dtype, **_kw(cfg)).run(x)
            sp = ShardedPipeline(cfg.shape, cfg.dtype, z0=0, nz=cfg.shape[0], group=dist.group.WORLD,
                                 device=torch.device("cuda", 0), **_kw(cfg))
            r = sp.run(x)
            assert torch.equal(r.codes, one.codes) and torch.equal(r.keep_bits, one.keep_bits)
            assert sp.local_count() == one.count
    finally:
        dist.destroy_process_group()


def test_bench_sharded_path_one_rank():
    """bench.py's multi-GPU code path (ShardedPipeline over NCCL, barriers, max over ranks, e2e with
    host buffers) on one rank: one clean JSON line on stdout."""
    import json
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, MASTER_PORT="29537")
    r = subprocess.run([sys.executable, "bench.py", "--sharded", "--config", "C1", "--steps", "3", "--warmup", "3",
                        "--no-cpu-baseline"], cwd=root, capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.strip()]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["config"]["parallelism"] == "zslab1" and d["value"] > 0 and d["e2e"]["value"] > 0


@pytest.mark.parametrize("G", [1, 2, 3, 8])
def test_merge_device_vs_host(G):
    """roix_merge_device (X4 on the device, every rank the same input) equals the host union-by-min
    roix_merge on random boundary tables: G blocks of ascending labels in disjoint ranges, random
    pairs between labels of neighbouring ranks, including a chain across every block."""
    import ctypes

    from gpu_util import new_sc, ptr, read_sc, st
    from paper_2602_15917_b200 import _lib as L

    rng = np.random.default_rng(G)
    pair_cap, root_cap = 64, 40
    W = 2 + 2 * pair_cap + 2 * root_cap
    blocks, all_pairs, all_lab, all_size = [], [], [], []
    prev_labels = None
    for r in range(G):
        nr = int(rng.integers(1, root_cap + 1))
        labels = np.sort(rng.choice(1 << 30, nr, replace=False)).astype(np.uint64) + np.uint64(r << 32)
        sizes = rng.integers(1, 10 ** 6, nr).astype(np.uint64)
        pairs = np.zeros((0, 2), np.uint64)
        if prev_labels is not None:
            k = int(rng.integers(1, pair_cap + 1))
            pairs = np.stack([labels[rng.integers(0, nr, k)], prev_labels[rng.integers(0, prev_labels.size, k)]], 1)
            pairs[0] = (labels[0], prev_labels[-1])          # a chain across all blocks
        b = np.zeros(W, np.uint64)
        b[0], b[1] = pairs.shape[0], nr
        b[2:2 + 2 * pairs.shape[0]] = pairs.reshape(-1)
        b[2 + 2 * pair_cap:2 + 2 * pair_cap + nr] = labels
        b[2 + 2 * pair_cap + root_cap:2 + 2 * pair_cap + root_cap + nr] = sizes
        blocks.append(b)
        all_pairs.append(pairs)
        all_lab.append(labels)
        all_size.append(sizes)
        prev_labels = labels
    gathered = torch.from_numpy(np.concatenate(blocks).view(np.int64)).cuda()
    M = G * root_cap
    out = torch.full((3, M), -1, dtype=torch.int64, device="cuda")
    nmap = torch.zeros(1, dtype=torch.int64, device="cuda")
    ws = torch.empty(L.roix_merge_workspace(G, root_cap), dtype=torch.uint8, device="cuda")
    sc = new_sc(1.0)
    L.roix_merge_device(ptr(gathered), G, pair_cap, root_cap, ptr(out[0]), ptr(out[1]), ptr(out[2]), ptr(nmap),
                        ptr(ws), ws.numel(), ptr(sc), st())
    assert read_sc(sc).err == 0
    ol, of, ot = L.roix_merge(np.concatenate(all_pairs), np.concatenate(all_lab), np.concatenate(all_size))
    m = int(nmap.item())
    assert m == ol.size
    got = out[:, :m].cpu().numpy().view(np.uint64)
    np.testing.assert_array_equal(got[0], ol)
    np.testing.assert_array_equal(got[1], of)
    np.testing.assert_array_equal(got[2], ot)
    # a count beyond its capacity is an error, not a silent truncation
    bad = gathered.clone()
    bad[1] = root_cap + 1
    sc2 = new_sc(1.0)
    L.roix_merge_device(ptr(bad), G, pair_cap, root_cap, ptr(out[0]), ptr(out[1]), ptr(out[2]), ptr(nmap),
                        ptr(ws), ws.numel(), ptr(sc2), st())
    assert read_sc(sc2).err & L.ERR_CAPACITY
