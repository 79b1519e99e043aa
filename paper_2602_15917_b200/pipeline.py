"""The ROIX hot path on one GPU, composed from the libroix C ABI (include/roix.h).

    histogram -> Otsu threshold -> binarise + opening -> CCL + filter -> quantise + compact
    (Fig. 2 P:210-217 order; BASELINE.json north_star)

PyTorch provides device memory and the stream; every step runs in libroix's kernels, enqueued on
one stream without host synchronisation (so the whole step can be captured in a CUDA graph).
"""
import ctypes
import math
import dataclasses

import numpy as np
import torch

from . import _lib as L

# kernels libroix launches per call (used for the bench's gpu_launches count)
LAUNCHES = {"scalars_init": 2, "range": 1, "resolve": 1, "histogram": 1, "threshold": 1, "morph": 2,
            "label": 9, "extract": 4, "extract_runs": 5}


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


@dataclasses.dataclass
class Result:
    codes: torch.Tensor        # dense code stream (count,), uint16 bits in int16 storage or int32
    keep_bits: torch.Tensor    # packed K, int32 words (bit i%32 of word i//32)
    count: int
    t8: int
    i_max: float
    eb: float
    thr: float
    n_components: int
    n_kept: int
    n_runs: int
    comp_min: torch.Tensor
    comp_size: torch.Tensor
    comp_kept: torch.Tensor
    scalars: L.Scalars


# run records per row the opening writes (roix_morph_slots, 1..64): with the opening hidden beside the
# binarisation, 64 (fewer rows left to a6's mask reader) measured 0.05 ms faster than 32 at C3
RUN_SLOTS = 64


def morph_chunks(shape, se, prebinarized=False):
    """Plane chunks of roix_morph (k_morph.cu open2d_pipelined / open3d_pipelined: binarised on the
    caller's stream, opened on a second one) for slabs of >= 2^30 voxels: in-plane SE, register-row
    opening: 8 chunks of whole planes, each starting on a word boundary; 3-D SE, whole-row opening
    (X = 32 W, W a power of two <= 32, 64 or 128): 16 chunks of >= 8 planes, at least 3; else 1."""
    Z, Y, X = shape
    W = (X + 31) // 32
    if prebinarized or Z * Y * X < (1 << 30):
        return 1
    if se == 6:
        if not (X % 32 == 0 and ((W <= 32 and W & (W - 1) == 0) or W in (64, 128))):
            return 1
        cp = max(8, -(-Z // 16))
        nch = -(-Z // cp)
        return nch if nch >= 3 else 1
    if X < 32 or W + 1 > 512:
        return 1
    pa = (Y * X) % 32
    quantum = 32 // math.gcd(pa if pa else 32, 32)
    cp = -(-Z // 8)
    cp = -(-cp // quantum) * quantum
    nch = -(-Z // cp)
    return nch if nch >= 2 else 1


def run_slots_for(shape, se):
    """Run records per row the opening writes for this slab shape: the in-plane openings (X >= 64);
    0 where the opening writes none (a6 then reads every row from o).  The 3-D opening writes none:
    records from k_open3d_rows measured slower overall (C5: opening +2.1 ms, labelling -0.9 ms)."""
    return RUN_SLOTS if (se == 4 and shape[2] >= 64) else 0


class Pipeline:
    """Preallocated buffers + the enqueue sequence for volumes of one shape / dtype / parameter set."""

    def __init__(self, shape, dtype, *, eb=0.0, rel_eb=0.0, conn=6, se=6, min_size=64, polarity=0,
                 run_capacity=None, code_capacity=None, device=None, labels=False, fused=False, extract="auto",
                 spans=False, classes=2, keep="size", frames=False, background=None, bg="sub"):
        L.load()
        self.shape = tuple(int(v) for v in shape)
        Z, Y, X = self.shape
        self.n = Z * Y * X
        self.dtype = dtype
        self.cdtype = L.U16 if dtype == "u16" else L.F32
        if (eb > 0) == (rel_eb > 0):
            raise ValueError("give exactly one of eb (absolute) and rel_eb (relative, fp32)")
        self.eb, self.rel_eb = float(eb), float(rel_eb)
        self.conn, self.se, self.min_size, self.polarity = int(conn), int(se), int(min_size), int(polarity)
        # a3 class count: 2 (Otsu, G-9) or 3 (multi-Otsu, NEXT-3: ROI above the lowest threshold / at or
        # below the highest for LOW, G-39)
        if classes not in (2, 3):
            raise ValueError("classes must be 2 or 3")
        if classes == 3 and fused:
            raise ValueError("the fused speculative histogram+binarisation supports classes = 2 only")
        self.classes = int(classes)
        # a7 filter: "size" drops components smaller than min_size (G-13); "largest" keeps only the
        # largest component (NEXT-3)
        if keep not in ("size", "largest"):
            raise ValueError("keep must be 'size' or 'largest'")
        self.keep = keep
        self.label_min_size = L.KEEP_LARGEST if keep == "largest" else self.min_size
        # a2-a4 per frame (NEXT-3, uint16 frame stacks): each z-plane its own image -- own histogram,
        # I_max and threshold (roix_histogram_frames / roix_threshold_frames / roix_morph_frames)
        self.frames = bool(frames)
        if self.frames and (dtype != "u16" or fused):
            raise ValueError("per-frame thresholds need uint16 input and the unfused path")
        # background subtraction first (NEXT-3): the path runs on max(0, I - B) ("sub") or
        # max(0, B - I) ("rev", transmission frames); B is one (Y, X) uint16 frame for every z
        self.bg_ref = None
        if background is not None:
            if dtype != "u16" or bg not in ("sub", "rev"):
                raise ValueError("background subtraction: uint16 input, bg 'sub' or 'rev'")
            assert tuple(background.shape) == tuple(shape[1:]) and background.is_contiguous()
            self.bg_ref = background
            self.bg_op = L.BG_SUB if bg == "sub" else L.BG_REV
            self.xb = torch.empty(tuple(shape), dtype=torch.int16, device=device or "cuda")
        self.device = torch.device(device or "cuda")
        dev = self.device
        self.geom = L.Geom(Z, Y, X, 0, Z)
        self.nwords = (self.n + 31) // 32
        self.sc = torch.zeros(L.scalars_size(), dtype=torch.uint8, device=dev)
        self.nbins = 65536 if dtype == "u16" else 256
        self.hist = torch.zeros(self.nbins * (Z if frames else 1), dtype=torch.int64, device=dev)
        self.frame_thr = torch.zeros(4 * max(Z, 1), dtype=torch.int32, device=dev) if frames else None   # roix_frame
        self.o = torch.empty(self.nwords + 4, dtype=torch.int32, device=dev)   # o, then K in place
        self.row_runs = torch.empty(Z * Y, dtype=torch.int32, device=dev)
        # run records of every row (x0, x1) written by the opening for rows of <= rs runs, so a6 does
        # not re-read those rows of o (roix_morph_slots / roix_label_slots)
        # (C3 rows hold ~11 runs on average: noise specks)
        self.rs = run_slots_for((Z, Y, X), se)
        self.run_slots = torch.empty(max(1, Z * Y * self.rs * 2), dtype=torch.int32, device=dev) if self.rs else None
        # fused (speculative) histogram + binarisation: one read of x for a2 + a4 (roix_histogram_binarize);
        # off by default: on B200 the histogram pass is bound by shared-memory atomics, and the fused pass
        # (3x slower than the plain histogram at C4) loses to histogram + streaming binarisation
        self.fused = bool(fused)
        # a8 form: "mask" = roix_extract over K (1024-voxel chunks of the kept mask), "runs" =
        # roix_extract_runs over the labelling's kept runs (reads neither K nor x outside them).  "auto":
        # runs for uint16 volumes labelled in 3-D (C1, C4, C5: kept runs shorter than a chunk, or cut by
        # chunk ends, where the per-chunk work of the mask form dominates), the mask form for in-plane
        # frame stacks (C3: long kept runs, mostly fully kept chunks) and fp32
        if extract not in ("mask", "runs", "auto"):
            raise ValueError("extract must be 'mask', 'runs' or 'auto'")
        if extract == "auto":
            extract = "runs" if dtype == "u16" and self.conn in (6, 18, 26) else "mask"
        self.extract = extract
        wsb = L.roix_histogram_binarize_workspace(self.geom) if self.fused else L.roix_morph_workspace(self.geom)
        self.morph_ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
        rows = Z * Y
        worst = rows * ((X + 1) // 2)
        if run_capacity is None:
            run_capacity = min(worst, max(1 << 22, self.n // 256))
        self._alloc_label(max(1, min(int(run_capacity), worst if worst > 0 else 1)))
        self.code_capacity = self.n if code_capacity is None else int(code_capacity)
        cdt = torch.int16 if dtype == "u16" else torch.int32
        self.codes = torch.empty(max(self.code_capacity, 8), dtype=cdt, device=dev)
        self.ex_ws = torch.empty(L.roix_extract_workspace(self.n), dtype=torch.uint8, device=dev)
        # NEXT-1 (optional): the paper's row-span representation of K (roix_row_spans)
        self.spans_on = bool(spans)
        if self.spans_on:
            self.span_ws = torch.empty(L.roix_row_spans_workspace(self.geom), dtype=torch.uint8, device=dev)
            self.span_rec = torch.empty(2 * Z * Y + 2, dtype=torch.int64, device=dev)   # roix_span: 16 bytes
            self.span_codes = torch.empty(max(self.n, 8), dtype=cdt, device=dev)
            self.span_counts = torch.zeros(2, dtype=torch.int64, device=dev)
        self.labels = torch.empty(self.n, dtype=torch.int64, device=dev) if labels else None

    def _alloc_label(self, cap):
        self.run_capacity = cap
        self.ws_bytes = L.roix_label_workspace(self.geom, cap)
        self.label_ws = torch.empty(self.ws_bytes, dtype=torch.uint8, device=self.device)
        self.comp_cap = cap
        dev = self.device
        self.comp_min = torch.empty(cap, dtype=torch.int64, device=dev)
        self.comp_size = torch.empty(cap, dtype=torch.int64, device=dev)
        self.comp_kept = torch.empty(cap, dtype=torch.uint8, device=dev)

    # -------------------------------------------------------------------------------- enqueue
    def enqueue(self, x, stream=None, mark=None):
        """Enqueue the whole path for x (device tensor, shape (Z, Y, X); u16 bits in int16/uint16
        storage or float32) on `stream` (default: torch's current stream).  No host sync.
        mark(stage) is called after each stage is enqueued (the bench records CUDA events there)."""
        assert x.is_cuda and x.numel() == self.n and x.is_contiguous()
        if stream is not None and stream != torch.cuda.current_stream(self.device):
            with torch.cuda.stream(stream):
                return self.enqueue(x, None, mark)
        mark = mark or (lambda stage: None)
        st = ctypes.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)
        sc, xp, n = _ptr(self.sc), _ptr(x), self.n
        if self.bg_ref is not None:
            L.roix_background(xp, _ptr(self.bg_ref), ctypes.byref(self.geom), self.bg_op, _ptr(self.xb), st)
            xp = _ptr(self.xb)
            mark("background")
        L.roix_scalars_init(sc, self.eb, st)
        if self.cdtype == L.F32:
            L.roix_range(xp, n, sc, st)
            mark("range")
        L.roix_resolve(sc, self.cdtype, self.rel_eb, st)
        L.roix_histogram_clear(_ptr(self.hist), self.hist.numel(), st)
        mark("setup")
        ws, wsb = _ptr(self.morph_ws), self.morph_ws.numel()
        if self.frames:
            L.roix_histogram_frames(xp, ctypes.byref(self.geom), sc, _ptr(self.hist), st)
            mark("histogram")
            L.roix_threshold_frames(_ptr(self.hist), self.shape[0], self.polarity, self.classes, sc,
                                    _ptr(self.frame_thr), st)
            mark("threshold")
            L.roix_morph_frames(xp, ctypes.byref(self.geom), self.se, None, None, _ptr(self.frame_thr), sc,
                                _ptr(self.o), _ptr(self.row_runs), ws, wsb, st)
            mark("morph")
            self._label_extract(xp, sc, st, mark)
            return
        if self.fused:
            L.roix_histogram_binarize(xp, self.cdtype, ctypes.byref(self.geom), self.polarity, sc, _ptr(self.hist),
                                      self.nbins, ws, wsb, st)
        else:
            L.roix_histogram(xp, self.cdtype, n, sc, _ptr(self.hist), self.nbins, st)
        mark("histogram")
        L.roix_threshold_multi(_ptr(self.hist), self.nbins, self.cdtype, self.polarity, self.classes, sc, st)
        mark("threshold")
        if self.fused:
            L.roix_morph_prebinarized(xp, self.cdtype, ctypes.byref(self.geom), self.se, None, None, sc, _ptr(self.o),
                                      _ptr(self.row_runs), ws, wsb, st)
        else:
            L.roix_morph_slots(xp, self.cdtype, ctypes.byref(self.geom), self.se, None, None, sc, _ptr(self.o),
                               _ptr(self.row_runs), _ptr(self.run_slots), self.rs, ws, wsb, st)
        mark("morph")
        self._label_extract(xp, sc, st, mark)

    def _label_extract(self, xp, sc, st, mark):
        n = self.n
        out = L.LabelOut(self.o.data_ptr(), self.comp_min.data_ptr(), self.comp_size.data_ptr(),
                         self.comp_kept.data_ptr(), self.comp_cap,
                         self.labels.data_ptr() if self.labels is not None else None)
        L.roix_label_slots(_ptr(self.o), _ptr(self.row_runs), _ptr(self.run_slots), self.rs, ctypes.byref(self.geom),
                           self.conn, self.label_min_size, self.run_capacity, _ptr(self.label_ws), self.ws_bytes,
                           ctypes.byref(out), sc, st)
        mark("label")
        if self.extract == "runs":
            # a1+a8 from the kept runs of a6/a7 (reads exactly the kept voxels of x; K is not re-read)
            L.roix_extract_runs(xp, self.cdtype, ctypes.byref(self.geom), self.run_capacity, _ptr(self.label_ws),
                                self.ws_bytes, sc, _ptr(self.codes), self.code_capacity, None, st)
        else:
            L.roix_extract(xp, self.cdtype, n, _ptr(self.o), sc, _ptr(self.codes), self.code_capacity, None,
                           _ptr(self.ex_ws), self.ex_ws.numel(), st)
        mark("extract")
        if self.spans_on:
            Z, Y, X = self.shape
            L.roix_row_spans(_ptr(self.o), xp, self.cdtype, ctypes.byref(self.geom), sc, _ptr(self.span_rec), Z * Y,
                             _ptr(self.span_codes), self.span_codes.numel(), _ptr(self.span_counts),
                             _ptr(self.span_ws), self.span_ws.numel(), st)
            mark("spans")

    def frame_thresholds(self):
        """Per-frame results of the last run (frames=True): list of roix_frame records."""
        a = self.frame_thr.cpu().numpy().view(np.uint32).reshape(-1, 4)
        return [L.Frame(*map(int, r)) for r in a]

    def row_spans(self):
        """(records (m, 3) int64: row, x_start, x_end; section codes) of the last run (spans=True)."""
        ns, nc = (int(v) for v in self.span_counts.cpu())
        sp = self.span_rec[: 2 * ns].view(-1, 2).cpu()
        rec = torch.stack([sp[:, 0], sp[:, 1] & 0xffffffff, sp[:, 1] >> 32], dim=1)
        return rec, self.span_codes[:nc]

    # ------------------------------------------------------------------ NEXT-4 reconstruction / quality
    def _stream(self, stream):
        return ctypes.c_void_p((stream or torch.cuda.current_stream(self.device)).cuda_stream)

    def decode(self, out=None, stream=None, from_spans=False):
        """Reconstruct the last run's volume: x^ = code * s on the ROI, 0 elsewhere; with a
        background reference, x^ is then combined with it: min(65535, x^ + B) for "sub",
        max(0, B - x^) for "rev".
        from_spans=False decodes the kept mask + dense code stream (roix_decode); True decodes the
        paper's row spans (roix_decode_spans, needs spans=True): every column of a span's
        [x_start, x_end) is restored, interior gaps included.  Returns out (shape, input dtype)."""
        tdt = torch.int16 if self.dtype == "u16" else torch.float32
        if out is None:
            out = torch.empty(self.shape, dtype=tdt, device=self.device)
        assert out.is_contiguous() and out.numel() == self.n and out.dtype in (tdt, torch.uint16)
        st = self._stream(stream)
        if from_spans:
            if not self.spans_on:
                raise ValueError("from_spans needs Pipeline(spans=True)")
            if not hasattr(self, "dspan_ws"):
                self.dspan_ws = torch.empty(max(1, L.roix_decode_spans_workspace(self.geom)), dtype=torch.uint8,
                                            device=self.device)
            Z, Y, _ = self.shape
            L.roix_decode_spans(_ptr(self.span_rec), Z * Y, _ptr(self.span_codes), self.span_codes.numel(),
                                _ptr(self.span_counts), self.cdtype, ctypes.byref(self.geom), _ptr(self.sc),
                                _ptr(out), _ptr(self.dspan_ws), self.dspan_ws.numel(), st)
        else:
            if not hasattr(self, "dec_ws"):
                self.dec_ws = torch.empty(max(1, L.roix_decode_workspace(self.n)), dtype=torch.uint8,
                                          device=self.device)
            L.roix_decode(_ptr(self.o), _ptr(self.codes), self.code_capacity, self.cdtype, self.n, _ptr(self.sc),
                          _ptr(out), _ptr(self.dec_ws), self.dec_ws.numel(), st)
        if self.bg_ref is not None:
            op = L.BG_ADD if self.bg_op == L.BG_SUB else L.BG_REV
            L.roix_background(_ptr(out), _ptr(self.bg_ref), ctypes.byref(self.geom), op, _ptr(out), st)
        return out

    def confusion(self, truth_words, stream=None, counts=None):
        """Enqueue roix_confusion of the last run's K against a packed ground-truth mask (e.g. from
        synth.generate(..., truth=...)); returns the device int64[4] (tp, fp, fn, tn)."""
        if counts is None:
            counts = torch.empty(4, dtype=torch.int64, device=self.device)
        assert truth_words.numel() >= self.nwords
        L.roix_confusion(_ptr(self.o), _ptr(truth_words), self.n, _ptr(counts), self._stream(stream))
        return counts

    def quality(self, truth_words):
        """Eqs. 7-14 of the last run's K against ground truth, plus the spatial reduction
        N / kept (Fig. 4) and, with spans=True, the paper's (rows * X) / sum(x_end - x_start)."""
        c = tuple(int(v) for v in self.confusion(truth_words).cpu())
        m = L.roix_overlap_metrics(c)
        m["counts"] = dict(zip(("tp", "fp", "fn", "tn"), c))
        kept = c[0] + c[1]
        m["spatial_reduction_voxels"] = self.n / kept if kept else float("nan")
        if self.spans_on:
            area = int(self.span_counts[1].item())
            m["spatial_reduction"] = self.n / area if area else float("nan")
        return m

    def launches(self):
        k = 4 if self.spans_on else 0   # roix_row_spans: extent, 2 scans, write
        k += 3 if self.keep == "largest" else 0   # reset + two reduction phases
        k += 1 if self.bg_ref is not None else 0
        k += sum(LAUNCHES[s] for s in ("scalars_init", "resolve", "histogram", "threshold", "morph", "label",
                                       "extract" if self.extract == "mask" else "extract_runs"))
        k += 1 if self.rs else 0          # k_runs_slots (the opening's run records)
        k += 2 * (morph_chunks(self.shape, self.se, self.fused) - 1)   # a4 + a5 per plane chunk
        return k + (LAUNCHES["range"] if self.cdtype == L.F32 else 0)

    def scalars(self):
        return L.Scalars.from_buffer_copy(bytes(self.sc.cpu().numpy()))

    def run(self, x, stream=None, check=True):
        """Enqueue, synchronise and collect.  Grows the run capacity and retries once if the
        labelling workspace was too small."""
        self.enqueue(x, stream)
        torch.cuda.synchronize(self.device)
        s = self.scalars()
        if s.err & L.ERR_CAPACITY and s.count <= self.code_capacity:
            # the labelling workspace (runs, or the cross-block pair queue sized from it) was too small
            self._alloc_label(int(max(s.n_runs, 2 * self.run_capacity)))
            self.enqueue(x, stream)
            torch.cuda.synchronize(self.device)
            s = self.scalars()
        if check and s.err:
            raise L.RoixError("device error bits 0x%x" % s.err)
        return self.collect(s)

    def collect(self, s=None):
        s = s or self.scalars()
        cnt = int(s.count)
        nc = int(min(s.n_components, self.comp_cap))
        thr = float(s.thr_u16) if self.cdtype == L.U16 else float(s.thr_f32)
        return Result(codes=self.codes[:cnt], keep_bits=self.o[: self.nwords], count=cnt, t8=int(s.t8),
                      i_max=float(s.i_max), eb=float(s.eb), thr=thr, n_components=int(s.n_components),
                      n_kept=int(s.n_kept), n_runs=int(s.n_runs), comp_min=self.comp_min[:nc],
                      comp_size=self.comp_size[:nc], comp_kept=self.comp_kept[:nc], scalars=s)


def run(x, **kw):
    """One-shot convenience: Pipeline(x.shape, dtype, **kw).run(x)."""
    dtype = "f32" if x.dtype == torch.float32 else "u16"
    return Pipeline(tuple(x.shape), dtype, device=x.device, **kw).run(x)


def unpack_bits(words, n):
    """Host helper: packed int32 words -> uint8 mask of n voxels (LSB-first, G-16)."""
    w = words.detach().cpu().numpy().view(np.uint8)
    return np.unpackbits(w, bitorder="little")[:n]
