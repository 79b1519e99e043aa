"""The ROIX hot path on a z-slab sharded volume.

Slab g of G holds planes [floor(g Z / G), floor((g+1) Z / G)).  Every global dependency of the path
is one exchange step:

  X2  fp32 range       all-reduce MIN / MAX of the slab ranges           (relative eb, I_max)
  X1  histogram        all-reduce SUM of the slab histograms             (identical Otsu threshold)
  X3  morphology halo  each slab sends its first / last two binarised planes to its z-neighbours
  X4  CCL merge        each slab sends its last plane's runs to the next slab (point to point), which
                       links them with its first plane; every slab's pair list and boundary-component
                       table are all-gathered and every rank runs the same device union-by-min
                       (roix_merge_device), so merged labels and sizes agree everywhere; small-object
                       removal then uses the merged sizes
  X5  stream offsets   all-gather of the slab counts (rank g's codes start at sum_{r<g} count_r)

Every exchange moves device buffers of host-known (capacity) size, so no step reads anything back to
the host: the whole sharded step is one enqueue sequence that a CUDA graph can capture.  A count that
exceeds its capacity sets ROIX_ERR_CAPACITY; ``run`` then grows the capacities and runs again.

The per-slab work is a generator (``slab_program``) that yields at each exchange; ``DistComm`` runs one
slab per process over torch.distributed (NCCL on B200s, gloo on CPU), ``SimComm`` runs all slabs in one
process on one GPU, in lockstep (the G-invariance tests).  Every compute step is a libroix call.
"""
import ctypes

import numpy as np
import torch

from . import _lib as L
from .pipeline import Pipeline, _ptr


def slab_bounds(Z, G, g):
    return g * Z // G, (g + 1) * Z // G


class SlabState(Pipeline):
    """Pipeline buffers for one slab, plus the exchange buffers of the sharded path."""

    def __init__(self, shape, dtype, *, z0, nz, rank, world, **kw):
        Z, Y, X = shape
        self.global_shape = tuple(shape)
        self.rank, self.world, self.z0, self.nz = rank, world, z0, nz
        super().__init__((nz, Y, X), dtype, **kw)
        if self.frames and self.se == 6 and world > 1:
            raise ValueError("per-frame thresholds on a sharded stack need in-plane morphology (se = 4)")
        self.geom = L.Geom(nz, Y, X, z0, Z)            # slab geometry in the global volume
        wsb = L.roix_histogram_binarize_workspace(self.geom) if self.fused else L.roix_morph_workspace(self.geom)
        self.morph_ws = torch.empty(wsb, dtype=torch.uint8, device=self.device)
        self.ws_bytes = L.roix_label_workspace(self.geom, self.run_capacity)
        self.label_ws = torch.empty(self.ws_bytes, dtype=torch.uint8, device=self.device)
        self.plane_w = (Y * X + 31) // 32
        dev = self.device
        self.halo_send = torch.zeros(2, 2 * self.plane_w + 4, dtype=torch.int32, device=dev)   # [lo, hi]
        self.halo_recv = torch.zeros(2, 2 * self.plane_w + 4, dtype=torch.int32, device=dev)
        self._alloc_exchange(min(Y * ((X + 1) // 2) + 1, 1 << 16))
        self.best = torch.zeros(2, dtype=torch.int64, device=dev)     # keep-largest: (size, label)
        self.counts_all = torch.zeros(world, dtype=torch.int64, device=dev)   # X5

    def _alloc_exchange(self, brun_cap):
        """X4 buffers.  brun: [count, roix_brun x brun_cap] (24-byte runs); block: this rank's merge
        input [npairs, nroots, pairs (2 pair_cap), labels (root_cap), sizes (root_cap)] (roix.h
        roix_merge_device); gathered: every rank's block; the map and its device length."""
        dev, G = self.device, self.world
        self.brun_cap = int(brun_cap)
        self.pair_cap = 2 * self.brun_cap
        self.root_cap = self.brun_cap
        self.brun = torch.zeros(1 + 3 * self.brun_cap, dtype=torch.int64, device=dev)
        self.brun_prev = torch.zeros_like(self.brun)
        W = 2 + 2 * self.pair_cap + 2 * self.root_cap
        self.block = torch.zeros(W, dtype=torch.int64, device=dev)
        self.gathered = torch.zeros(G * W, dtype=torch.int64, device=dev)
        self.map = torch.zeros(3, G * self.root_cap, dtype=torch.int64, device=dev)
        self.nmap = torch.zeros(1, dtype=torch.int64, device=dev)
        self.merge_ws = torch.empty(L.roix_merge_workspace(G, self.root_cap), dtype=torch.uint8, device=dev)

    def block_views(self):
        pc, rc = self.pair_cap, self.root_cap
        b = self.block
        return b[0:1], b[1:2], b[2:2 + 2 * pc], b[2 + 2 * pc:2 + 2 * pc + rc], b[2 + 2 * pc + rc:2 + 2 * pc + 2 * rc]

    @property
    def offset(self):
        """Global stream offset of this slab's codes (host read of the X5 all-gather)."""
        return int(self.counts_all[: self.rank].sum().item())

    @property
    def global_count(self):
        return int(self.counts_all.sum().item())

    def _alloc_label(self, cap):
        super()._alloc_label(cap)
        if hasattr(self, "global_shape"):
            self.ws_bytes = L.roix_label_workspace(self.geom, cap)
            self.label_ws = torch.empty(self.ws_bytes, dtype=torch.uint8, device=self.device)



def slab_program(S, x, stream=None, mark=None):
    """Generator: enqueue this slab's work; yield at every exchange (see module doc).  mark(stage) is
    called after each stage is enqueued (bench.py records CUDA events there)."""
    mark = mark or (lambda stage: None)
    st = ctypes.c_void_p((stream or torch.cuda.current_stream(S.device)).cuda_stream)
    sc, xp, n = _ptr(S.sc), _ptr(x), S.n
    G, g = S.world, S.rank
    if S.bg_ref is not None:
        L.roix_background(xp, _ptr(S.bg_ref), ctypes.byref(S.geom), S.bg_op, _ptr(S.xb), st)
        xp = _ptr(S.xb)
        mark("background")
    L.roix_scalars_init(sc, S.eb, st)
    if S.cdtype == L.F32:
        L.roix_range(xp, n, sc, st)
        yield ("minmax", S.sc)                                    # X2
        mark("range")
    L.roix_resolve(sc, S.cdtype, S.rel_eb, st)
    L.roix_histogram_clear(_ptr(S.hist), S.hist.numel(), st)
    mark("setup")
    mws, mwsb = _ptr(S.morph_ws), S.morph_ws.numel()
    frames = S.frames
    if frames:
        # per-frame thresholds (NEXT-3): frames never span slabs, so no histogram exchange
        L.roix_histogram_frames(xp, ctypes.byref(S.geom), sc, _ptr(S.hist), st)
        mark("histogram")
        L.roix_threshold_frames(_ptr(S.hist), S.nz, S.polarity, S.classes, sc, _ptr(S.frame_thr), st)
        mark("threshold")
    elif S.fused:
        L.roix_histogram_binarize(xp, S.cdtype, ctypes.byref(S.geom), S.polarity, sc, _ptr(S.hist), S.nbins, mws,
                                  mwsb, st)
    else:
        L.roix_histogram(xp, S.cdtype, n, sc, _ptr(S.hist), S.nbins, st)
    if not frames:
        yield ("sum", S.hist)                                     # X1
        mark("histogram")
        L.roix_threshold_multi(_ptr(S.hist), S.nbins, S.cdtype, S.polarity, S.classes, sc, st)
        mark("threshold")
    halo_lo = halo_hi = None
    if S.se == 6 and G > 1:
        if S.nz < 2:
            raise ValueError("every slab needs >= 2 planes for the opening's halo")
        pw = S.plane_w
        L.roix_binarize_planes(xp, S.cdtype, ctypes.byref(S.geom), 0, 2, sc, _ptr(S.halo_send[0]), st)
        L.roix_binarize_planes(xp, S.cdtype, ctypes.byref(S.geom), S.nz - 2, 2, sc, _ptr(S.halo_send[1]), st)
        yield ("halo", S.halo_send, S.halo_recv)                  # X3
        if g > 0:
            halo_lo = _ptr(S.halo_recv[0])
        if g < G - 1:
            halo_hi = _ptr(S.halo_recv[1])
        assert pw > 0
    if frames:
        L.roix_morph_frames(xp, ctypes.byref(S.geom), S.se, halo_lo, halo_hi, _ptr(S.frame_thr), sc, _ptr(S.o),
                            _ptr(S.row_runs), mws, mwsb, st)
    else:
        if S.fused:
            L.roix_morph_prebinarized(xp, S.cdtype, ctypes.byref(S.geom), S.se, halo_lo, halo_hi, sc, _ptr(S.o),
                                      _ptr(S.row_runs), mws, mwsb, st)
        else:
            L.roix_morph_slots(xp, S.cdtype, ctypes.byref(S.geom), S.se, halo_lo, halo_hi, sc, _ptr(S.o),
                               _ptr(S.row_runs), _ptr(S.run_slots), S.rs, mws, mwsb, st)
    mark("morph")
    out = L.LabelOut(S.o.data_ptr(), S.comp_min.data_ptr(), S.comp_size.data_ptr(), S.comp_kept.data_ptr(),
                     S.comp_cap, S.labels.data_ptr() if S.labels is not None else None)
    geo = ctypes.byref(S.geom)
    if S.conn in (6, 18, 26) and G > 1:
        ws, wsb, cap = _ptr(S.label_ws), S.ws_bytes, S.run_capacity
        npairs, nroots, pairs, rlab, rsize = S.block_views()
        L.roix_label_local_slots(_ptr(S.o), _ptr(S.row_runs), _ptr(S.run_slots), S.rs, geo, S.conn, cap, ws, wsb, sc,
                                 st)
        L.roix_label_boundary(ws, geo, cap, 1, _ptr(S.brun[1:]), S.brun_cap, _ptr(S.brun[0:1]), sc, st)
        yield ("shift", S)                                        # X4a: last-plane runs -> next slab
        if g > 0:
            L.roix_label_link(ws, geo, cap, S.conn, _ptr(S.brun_prev[1:]), _ptr(S.brun_prev[0:1]), _ptr(pairs),
                              S.pair_cap, _ptr(npairs), sc, st)
        L.roix_label_boundary_roots(ws, geo, cap, _ptr(rlab), _ptr(rsize), S.root_cap, _ptr(nroots), sc, st)
        yield ("gather_tables", S)                                # X4b: every slab's block
        L.roix_merge_device(_ptr(S.gathered), G, S.pair_cap, S.root_cap, _ptr(S.map[0]), _ptr(S.map[1]),
                            _ptr(S.map[2]), _ptr(S.nmap), _ptr(S.merge_ws), S.merge_ws.numel(), sc, st)
        mp = (_ptr(S.map[0]), _ptr(S.map[1]), _ptr(S.map[2]), _ptr(S.nmap))
        if S.keep == "largest":
            # NEXT-3 keep-largest over the whole volume: the largest size, then the smallest label of
            # that size, each reduced over the ranks (X4c, X4d)
            L.roix_label_largest(ws, geo, cap, *mp, 0, _ptr(S.best), sc, st)
            yield ("best_max", S.best)
            L.roix_label_largest(ws, geo, cap, *mp, 1, _ptr(S.best), sc, st)
            yield ("best_min", S.best)
            L.roix_label_finish_keep(_ptr(S.o), geo, cap, ws, wsb, *mp, _ptr(S.best), ctypes.byref(out), sc, st)
        else:
            L.roix_label_finish(_ptr(S.o), geo, S.min_size, cap, ws, wsb, *mp, ctypes.byref(out), sc, st)
    else:
        L.roix_label_slots(_ptr(S.o), _ptr(S.row_runs), _ptr(S.run_slots), S.rs, geo, S.conn, S.label_min_size,
                           S.run_capacity, _ptr(S.label_ws), S.ws_bytes, ctypes.byref(out), sc, st)
    mark("label")
    if S.extract == "runs":
        L.roix_extract_runs(xp, S.cdtype, geo, S.run_capacity, _ptr(S.label_ws), S.ws_bytes, sc, _ptr(S.codes),
                            S.code_capacity, None, st)
    else:
        L.roix_extract(xp, S.cdtype, n, _ptr(S.o), sc, _ptr(S.codes), S.code_capacity, None, _ptr(S.ex_ws),
                       S.ex_ws.numel(), st)
    yield ("counts", S)                                           # X5 (device: S.counts_all)
    mark("extract")


def _count_of(S):
    off = L.Scalars.count.offset
    return S.sc[off:off + 8].view(torch.int64)


# ------------------------------------------------------------------------------------- comms
class SimComm:
    """All slabs in one process on one device, advanced in lockstep (no kernel waits on another)."""

    def run(self, states, xs):
        gens = [slab_program(S, x) for S, x in zip(states, xs)]
        msgs = [next(gen) for gen in gens]
        while True:
            kind = msgs[0][0]
            assert all(m[0] == kind for m in msgs), "slabs diverged"
            replies = self._do(kind, msgs, states)
            nxt = []
            done = 0
            for gen, rep in zip(gens, replies):
                try:
                    nxt.append(gen.send(rep))
                except StopIteration:
                    done += 1
            if done:
                assert done == len(gens)
                return
            msgs = nxt

    def _do(self, kind, msgs, states):
        G = len(msgs)
        if kind == "minmax":
            lo = min(int(m[1][4:8].view(torch.int32).cpu().numpy().view(np.uint32)[0]) for m in msgs)
            hi = max(int(m[1][8:12].view(torch.int32).cpu().numpy().view(np.uint32)[0]) for m in msgs)
            for m in msgs:
                m[1][4:12].copy_(torch.from_numpy(np.array([lo, hi], np.uint32).view(np.uint8)).to(m[1].device))
            return [None] * G
        if kind == "sum":
            tot = sum(m[1] for m in msgs)
            for m in msgs:
                m[1].copy_(tot)
            return [None] * G
        if kind == "halo":
            for g, m in enumerate(msgs):
                if g > 0:
                    m[2][0].copy_(msgs[g - 1][1][1])    # previous slab's last two planes
                if g < G - 1:
                    m[2][1].copy_(msgs[g + 1][1][0])    # next slab's first two planes
            return [None] * G
        if kind == "shift":
            for g in range(1, G):
                states[g].brun_prev.copy_(states[g - 1].brun)
            return [None] * G
        if kind == "gather_tables":
            allb = torch.cat([S.block for S in states])
            for S in states:
                S.gathered.copy_(allb)
            return [None] * G
        if kind == "counts":
            c = torch.cat([_count_of(S) for S in states])
            for S in states:
                S.counts_all.copy_(c)
            return [None] * G
        if kind in ("best_max", "best_min"):
            k = 0 if kind == "best_max" else 1
            vals = torch.stack([m[1][k] for m in msgs])
            v = vals.max() if k == 0 else vals.min()
            for m in msgs:
                m[1][k].copy_(v)
            return [None] * G
        raise ValueError(kind)


class DistComm:
    """One slab per process over torch.distributed (NCCL between B200s; gloo on CPU for tests)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist, self.group = dist, group
        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)

    def run(self, S, x, mark=None):
        gen = slab_program(S, x, mark=mark)
        rep = None
        try:
            msg = next(gen)
            while True:
                rep = self._do(msg, S)
                msg = gen.send(rep)
        except StopIteration:
            return

    def _do(self, msg, S):
        d, grp = self.dist, self.group
        kind = msg[0]
        if kind == "minmax":
            v = msg[1][4:12].view(torch.int32).to(torch.int64) & 0xFFFFFFFF
            lo, hi = v[0:1].clone(), v[1:2].clone()
            d.all_reduce(lo, op=d.ReduceOp.MIN, group=grp)
            d.all_reduce(hi, op=d.ReduceOp.MAX, group=grp)
            v = torch.cat([lo, hi])
            msg[1][4:12].view(torch.int32).copy_(torch.where(v >= 2 ** 31, v - 2 ** 32, v).to(torch.int32))
            return None
        if kind == "sum":
            d.all_reduce(msg[1], group=grp)
            return None
        if kind == "halo":
            send, recv = msg[1], msg[2]
            ops = []
            g, G = self.rank, self.world
            if g > 0:
                ops += [d.P2POp(d.isend, send[0], g - 1, grp), d.P2POp(d.irecv, recv[0], g - 1, grp)]
            if g < G - 1:
                ops += [d.P2POp(d.isend, send[1], g + 1, grp), d.P2POp(d.irecv, recv[1], g + 1, grp)]
            if ops:
                for r in d.batch_isend_irecv(ops):
                    r.wait()
            return None
        if kind == "shift":
            # the packed last-plane runs (count + capacity) to the next rank, point to point
            ops = []
            g, G = self.rank, self.world
            if g < G - 1:
                ops.append(d.P2POp(d.isend, S.brun, g + 1, grp))
            if g > 0:
                ops.append(d.P2POp(d.irecv, S.brun_prev, g - 1, grp))
            if ops:
                for r in d.batch_isend_irecv(ops):
                    r.wait()
            return None
        if kind == "gather_tables":
            d.all_gather_into_tensor(S.gathered, S.block, group=grp)
            return None
        if kind in ("best_max", "best_min"):
            k = 0 if kind == "best_max" else 1
            v = msg[1][k:k + 1].clone()
            d.all_reduce(v, op=d.ReduceOp.MAX if k == 0 else d.ReduceOp.MIN, group=grp)
            msg[1][k:k + 1].copy_(v)
            return None
        if kind == "counts":
            d.all_gather_into_tensor(S.counts_all, _count_of(S).clone(), group=grp)
            return None
        raise ValueError(kind)


class ShardedPipeline:
    """One rank's slab of a z-sharded volume over a torch.distributed group (used by bench.py)."""

    def __init__(self, shape, dtype, *, z0, nz, group=None, device=None, **kw):
        self.comm = DistComm(group)
        self.S = SlabState(shape, dtype, z0=z0, nz=nz, rank=self.comm.rank, world=self.comm.world, device=device, **kw)

    @property
    def extract(self):   # the resolved a8 form of the slab pipeline
        return self.S.extract

    def enqueue(self, x, mark=None):
        self.comm.run(self.S, x, mark=mark)

    def run(self, x):
        """Enqueue, synchronise and collect.  A capacity error on any rank (the exchange buffers or the
        labelling workspace) grows the capacities on every rank and runs again (ranks agree through a
        MAX all-reduce of the error bits, so all of them retry or none does)."""
        S, d = self.S, self.comm.dist
        for attempt in range(6):
            self.enqueue(x)
            torch.cuda.synchronize(S.device)
            s = S.scalars()
            e = torch.tensor([int(s.err)], dtype=torch.int64, device=S.device)
            d.all_reduce(e, op=d.ReduceOp.MAX, group=self.comm.group)
            err = int(e.item())
            if err & L.ERR_CAPACITY and s.count <= S.code_capacity and attempt < 5:
                S._alloc_exchange(2 * S.brun_cap)
                S._alloc_label(int(max(s.n_runs, 2 * S.run_capacity)))
                continue
            break
        if err:
            raise L.RoixError("device error bits 0x%x" % err)
        return S.collect(s)

    def scalars(self):
        return self.S.scalars()

    def local_count(self):
        return int(self.S.scalars().count)

    def launches(self):
        # the unsharded count, plus: halo binarisation (2 x 2 kernels), boundary runs (1), link (1),
        # boundary roots (5), device merge (5), finish instead of label (-0)
        return self.S.launches() + 14


def run_simulated(x_full, G, *, shape=None, dtype=None, **kw):
    """All G slabs of a volume on this GPU, in lockstep -- the G-invariance tests."""
    Z = x_full.shape[0]
    dtype = dtype or ("f32" if x_full.dtype == torch.float32 else "u16")
    states, xs = [], []
    for g in range(G):
        z0, z1 = slab_bounds(Z, G, g)
        states.append(SlabState(tuple(x_full.shape), dtype, z0=z0, nz=z1 - z0, rank=g, world=G,
                                device=x_full.device, **kw))
        xs.append(x_full[z0:z1].clone())   # fresh (16-byte aligned) allocation per slab
    SimComm().run(states, xs)
    torch.cuda.synchronize()
    return states
