"""CPU (no GPU): the host side of the sharded path -- the host union-by-min merge of slab-boundary
components (roix_merge, C++ in libroix; the device merge roix_merge_device is checked against it in
tests/test_gpu_sharded.py) and the torch.distributed exchanges over gloo with world_size 2, on the
device-layout buffers the GPU path exchanges (packed boundary runs, merge blocks, counts)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


@pytest.fixture(scope="module")
def L():
    from paper_2602_15917_b200 import build

    build.build()
    from paper_2602_15917_b200 import _lib

    _lib.load()
    return _lib


def _brute_merge(pairs, labels, sizes):
    lab = sorted(set(int(v) for v in labels))
    size = {}
    for a, s in zip(labels, sizes):
        size.setdefault(int(a), int(s))
    comp = {a: {a} for a in lab}
    for a, b in pairs:
        ca, cb = comp[int(a)], comp[int(b)]
        if ca is not cb:
            u = ca | cb
            for v in u:
                comp[v] = u
    fin = [min(comp[a]) for a in lab]
    tot = [sum(size[v] for v in comp[a]) for a in lab]
    return lab, fin, tot


def test_merge_vs_brute_force(L):
    rng = np.random.default_rng(0)
    for trial in range(50):
        m = int(rng.integers(1, 60))
        labels = rng.choice(10 ** 12, m, replace=False).astype(np.uint64)
        sizes = rng.integers(1, 1000, m).astype(np.uint64)
        k = int(rng.integers(0, 3 * m))
        pairs = labels[rng.integers(0, m, (k, 2))] if k else np.zeros((0, 2), np.uint64)
        ol, of, ot = L.roix_merge(pairs, labels, sizes)
        bl, bf, bt = _brute_merge(pairs, labels, sizes)
        assert ol.tolist() == bl and of.tolist() == bf and ot.tolist() == bt
        # order independence: shuffled pairs and tables give the same answer
        perm = rng.permutation(m)
        ol2, of2, ot2 = L.roix_merge(pairs[::-1], labels[perm], sizes[perm])
        assert (ol2 == ol).all() and (of2 == of).all() and (ot2 == ot).all()


def test_merge_rejects_unknown_label(L):
    with pytest.raises(L.RoixError):
        L.roix_merge(np.array([[1, 99]], np.uint64), np.array([1, 2], np.uint64), np.array([5, 6], np.uint64))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class _FakeSlab:
    """The fields DistComm touches, on the CPU, in the layouts of SlabState."""

    def __init__(self, rank, world):
        from paper_2602_15917_b200 import _lib as L

        self.device = torch.device("cpu")
        self.sc = torch.zeros(L.scalars_size(), dtype=torch.uint8)
        self.brun_cap = 4
        self.brun = torch.arange(1 + 3 * self.brun_cap, dtype=torch.int64) + 1000 * rank   # [count, runs]
        self.brun[0] = 3 + rank
        self.brun_prev = torch.full_like(self.brun, -1)
        self.pair_cap, self.root_cap = 3, 2
        W = 2 + 2 * self.pair_cap + 2 * self.root_cap
        # block: [npairs, nroots, pairs (2 pair_cap), labels (root_cap), sizes (root_cap)]
        self.block = torch.tensor([2, 1 + rank, 10 * rank, 10 * rank + 1, 10 * rank + 2, 10 * rank + 3, 0, 0,
                                   100 + rank, 200 + rank, 7, 8], dtype=torch.int64)
        assert self.block.numel() == W
        self.gathered = torch.zeros(world * W, dtype=torch.int64)
        self.counts_all = torch.zeros(world, dtype=torch.int64)


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2602_15917_b200 import _lib as L
        from paper_2602_15917_b200.sharded import DistComm

        comm = DistComm()
        S = _FakeSlab(rank, world)
        out = {}
        # X1: histogram sum
        h = torch.arange(8, dtype=torch.int64) * (rank + 1)
        comm._do(("sum", h), S)
        out["sum"] = h.tolist()
        # X2: ordered-int min / max (values above 2^31 included)
        vals = [(0x80000010, 0x90000000), (0x7FFFFFF0, 0xC0000001)][rank]
        S.sc[4:12].copy_(torch.from_numpy(np.array(vals, np.uint32).view(np.uint8)))
        comm._do(("minmax", S.sc), S)
        out["minmax"] = S.sc[4:12].numpy().view(np.uint32).tolist()
        # X3: halo planes to / from the z-neighbours
        send = torch.full((2, 6), rank, dtype=torch.int32)
        send[1] += 10
        recv = torch.full((2, 6), -1, dtype=torch.int32)
        comm._do(("halo", send, recv), S)
        out["halo"] = recv.tolist()
        # X4a: the packed last-plane runs, point to point to the next rank
        comm._do(("shift", S), S)
        out["shift"] = S.brun_prev.tolist()
        # X4b: every rank's merge block, in rank order
        comm._do(("gather_tables", S), S)
        out["gathered"] = S.gathered.tolist()
        # X5: counts
        off = L.Scalars.count.offset
        S.sc[off:off + 8].view(torch.int64).fill_(5 + rank)
        comm._do(("counts", S), S)
        out["counts"] = S.counts_all.tolist()
        # X4c / X4d: keep-largest (size MAX, then label MIN; 2^63 - 1 = "no component of that size")
        best = torch.tensor([[40, 0], [55, 0]][rank], dtype=torch.int64)
        comm._do(("best_max", best), S)
        best[1] = [(1 << 63) - 1, 777][rank]
        comm._do(("best_min", best), S)
        out["best"] = best.tolist()
        out["block"] = S.block.tolist()
        out["brun"] = S.brun.tolist()
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_distcomm_exchanges_gloo(L):
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    for r in range(world):
        o = res[r]
        assert o["sum"] == [3 * k for k in range(8)]
        assert o["minmax"] == [0x7FFFFFF0, 0xC0000001]
        assert o["counts"] == [5, 6]
        assert o["best"] == [55, 777]
        assert o["gathered"] == res[0]["block"] + res[1]["block"]
    assert res[0]["halo"][1] == [1] * 6 and res[0]["halo"][0] == [-1] * 6   # rank 0 <- rank 1's first planes
    assert res[1]["halo"][0] == [10] * 6 and res[1]["halo"][1] == [-1] * 6  # rank 1 <- rank 0's last planes
    assert res[1]["shift"] == res[0]["brun"]                                  # rank 1 <- rank 0's runs
    assert res[0]["shift"] == [-1] * 13                                       # rank 0 receives none
