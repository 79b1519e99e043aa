"""Seeded synthetic inputs for the ROIX hot path (DESIGN.md §5 "Input recipe").

The paper's seven datasets are not available; BASELINE.json's configs C1..C5 stand in
for them.  This module holds the config table and the phantom generator, and NONE of the method's
arithmetic: both the product's tests/bench and the oracle's tests draw inputs from it.

Object lists (centres, semi-axes, rotations, intensities) are drawn on the host with
``numpy.random.Generator(PCG64(seed))`` in the documented order; voxel values are produced on the
GPU by ``synth.cu`` as a pure function of (config, seed, objects, global linear index), so every
z-slab is bit-identical to the same planes of the whole volume, whatever the GPU count.
"""
import ctypes
import dataclasses
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "synth.cu")
_LIB = os.path.join(_HERE, "libroixsynth.so")
_lib = None


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    shape: tuple          # (Z, Y, X), x fastest
    dtype: str            # "u16" | "f32"
    eb: float = 0.0       # absolute eb (input units); 0 when rel_eb is used
    rel_eb: float = 0.0   # value-range-relative eb (G-6)
    conn: int = 6
    se: int = 6
    min_size: int = 64
    polarity: int = 0     # 0 HIGH, 1 LOW (G-10)
    seed: int = 0
    scale: float = 1.0    # lengths of the phantom relative to the BASELINE.json config
    frames: int = 0       # C3: frames of the full stack the rotation angle refers to

    @property
    def n(self):
        return int(np.prod(self.shape, dtype=np.int64))

    @property
    def itemsize(self):
        return 2 if self.dtype == "u16" else 4

    @property
    def nbytes(self):
        return self.n * self.itemsize


# BASELINE.json configs[0..4] (C1..C5); bold decisions of SURVEY.md §8.0 (G-12, G-15, G-10)
CONFIGS = {
    "C1": Config("C1", (64, 256, 256), "u16", eb=2.0, conn=6, se=6, min_size=64, seed=0),
    "C2": Config("C2", (512, 512, 512), "f32", rel_eb=1e-3, conn=6, se=6, min_size=64, seed=1),
    "C3": Config("C3", (128, 9700, 13900), "u16", eb=1.0, conn=8, se=4, min_size=64, polarity=1, seed=2, frames=128),
    "C4": Config("C4", (2048, 2048, 2048), "u16", eb=4.0, conn=26, se=6, min_size=512, seed=3),
    "C5": Config("C5", (4096, 4096, 2048), "u16", eb=2.0, conn=6, se=6, min_size=64, seed=4),
}


def scaled(name, scale, frames=None):
    """A smaller phantom of the same recipe: every length (and the volume) scaled by `scale`.
    C3 keeps its frame count unless `frames` is given (the rotation stays that of the full stack)."""
    c = CONFIGS[name]
    Z, Y, X = c.shape
    if name == "C3":
        shape = (frames or Z, max(1, round(Y * scale)), max(1, round(X * scale)))
    else:
        shape = (max(1, round(Z * scale)), max(1, round(Y * scale)), max(1, round(X * scale)))
    return dataclasses.replace(c, name="%s@%g" % (name, scale), shape=shape, scale=scale)


# ------------------------------------------------------------------------------- object lists
_OBJ = np.dtype([("c", "<f4", 3), ("R", "<f4", 9), ("inv_r2", "<f4", 3), ("mu", "<f4"), ("bbox", "<f4", 6)])


def _quat_rot(q):
    q = q / np.linalg.norm(q)
    w, a, b, c = q
    return np.array([[1 - 2 * (b * b + c * c), 2 * (a * b - c * w), 2 * (a * c + b * w)],
                     [2 * (a * b + c * w), 1 - 2 * (a * a + c * c), 2 * (b * c - a * w)],
                     [2 * (a * c - b * w), 2 * (b * c + a * w), 1 - 2 * (a * a + b * b)]])


def _obj(c, radii, R, mu):
    o = np.zeros((), _OBJ)
    o["c"] = c
    o["R"] = R.reshape(-1)
    o["inv_r2"] = 1.0 / np.square(radii)
    o["mu"] = mu
    half = np.sqrt(np.sum(np.square(R * np.asarray(radii)[None, :]), axis=1))  # world half-extents
    lo, hi = np.asarray(c) - half - 1.0, np.asarray(c) + half + 1.0
    o["bbox"] = [lo[0], hi[0], lo[1], hi[1], lo[2], hi[2]]
    return o


def objects(cfg):
    """The object list of a config, in painter's order (later objects win), as a numpy record array."""
    rng = np.random.Generator(np.random.PCG64(cfg.seed))
    Z, Y, X = cfg.shape
    s = cfg.scale
    base = cfg.name.split("@")[0]
    objs = []
    if base == "C1":
        for _ in range(6):
            c = rng.uniform([0, 0, 0], [Z, Y, X])
            r = rng.uniform(10, 60, 3) * s
            R = _quat_rot(rng.normal(size=4))
            objs.append(_obj(c, r, R, rng.uniform(1800, 3200)))
    elif base == "C2":
        for k in range(40):
            c = rng.uniform([0, 0, 0], [Z, Y, X])
            if k % 2 == 0:
                r = np.full(3, rng.uniform(16, 96) * s)
                R = np.eye(3)
            else:
                r = rng.uniform(16, 96, 3) * s
                R = _quat_rot(rng.normal(size=4))
            objs.append(_obj(c, r, R, rng.uniform(0.3, 1.2)))
    elif base == "C4":
        cy = cx = (Y - 1) / 2.0
        rad = 900.0 * s
        npores = 5000
        for _ in range(npores):
            z = rng.uniform(0, Z)
            rr = rad * math.sqrt(rng.uniform(0, 1))
            th = rng.uniform(0, 2 * math.pi)
            r = rng.uniform(2, 40) * s
            objs.append(_obj([z, cy + rr * math.sin(th), cx + rr * math.cos(th)], np.full(3, r), np.eye(3), 300.0))
        objs.sort(key=lambda o: float(o["c"][0]))   # pores all share one value law: order is free
    elif base == "C5":
        for k in range(200):
            if k < 56:
                j = 1 + k % 7
                cz = 512 * j * (Z / 4096.0) + rng.uniform(-64, 64) * s
                c = np.array([cz, rng.uniform(0, Y), rng.uniform(0, X)])
            else:
                c = rng.uniform([0, 0, 0], [Z, Y, X])
            if 56 <= k < 64:     # elongated along z: cross >= 3 slabs at G = 8
                r = np.array([rng.uniform(600, 1000), rng.uniform(32, 128), rng.uniform(32, 128)]) * s
                th = rng.uniform(0, 2 * math.pi)
                R = np.array([[1, 0, 0], [0, math.cos(th), -math.sin(th)], [0, math.sin(th), math.cos(th)]])
            else:
                r = rng.uniform(32, 256, 3) * s
                R = _quat_rot(rng.normal(size=4))
            objs.append(_obj(c, r, R, rng.uniform(1500, 4000)))
    if not objs:
        return np.zeros(0, _OBJ)
    return np.array(objs, dtype=_OBJ)


def rings(cfg):
    """C2 ring artefacts: 12 bands (R_j ~ U(8,360), w_j ~ U(1,3), sigma_j = +-1), drawn after the objects."""
    rng = np.random.Generator(np.random.PCG64(cfg.seed + 1000))
    s = cfg.scale
    out = []
    for _ in range(12):
        out += [rng.uniform(8, 360) * s, rng.uniform(1, 3) * max(s, 0.34), float(rng.choice([-1.0, 1.0]))]
    return np.array(out, np.float32)


# ------------------------------------------------------------------------------- GPU generation
class _Params(ctypes.Structure):
    _fields_ = [("mode", ctypes.c_int), ("seed", ctypes.c_uint32), ("gz", ctypes.c_uint64), ("ny", ctypes.c_uint64),
                ("nx", ctypes.c_uint64), ("z0", ctypes.c_uint64), ("nz", ctypes.c_uint64), ("nobj", ctypes.c_int),
                ("obj", ctypes.c_void_p), ("p", ctypes.c_float * 16), ("nring", ctypes.c_int), ("ring", ctypes.c_void_p),
                ("truth", ctypes.c_void_p)]


def build(force=False):
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + ".tmp%d" % os.getpid()
        subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17",
                               "-Xcompiler", "-fPIC", "-shared", "-cudart", "static", "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        lib.synth_generate.restype = ctypes.c_int
        lib.synth_generate.argtypes = [ctypes.POINTER(_Params), ctypes.c_void_p, ctypes.c_void_p]
        assert lib.synth_obj_size() == _OBJ.itemsize
        _lib = lib
    return _lib


_MODE = {"C1": 1, "C5": 2, "C2": 3, "C3": 4, "C4": 5}


def truth_words(cfg, nz=None):
    """uint32 words of a packed ground-truth mask of nz planes (default: the whole volume)."""
    Z, Y, X = cfg.shape
    return ((Z if nz is None else nz) * Y * X + 31) // 32


def generate(cfg, z0=0, nz=None, out=None, device="cuda", truth=None):
    """Generate planes [z0, z0+nz) of cfg's volume on the GPU into a torch tensor (nz, Y, X).

    truth (optional): an int32 device tensor of truth_words(cfg, nz) words, overwritten with the
    slab's ground-truth region of interest, bit-packed like the product's masks (bit i % 32 of word
    i // 32, LSB first, pad bits 0; i slab-local).  Ground truth = the voxel lies inside an object
    (C1, C2, C5: the ellipsoids; painter's order does not matter, every object is foreground), inside
    the sample's shadow (C3), or in the porous cylinder's solid matrix, pores excluded (C4)."""
    import torch

    Z, Y, X = cfg.shape
    nz = Z - z0 if nz is None else nz
    tdt = torch.int16 if cfg.dtype == "u16" else torch.float32     # u16 bits carried in int16 storage
    if out is None:
        out = torch.empty((nz, Y, X), dtype=tdt, device=device)
    base = cfg.name.split("@")[0]
    objs = objects(cfg)
    obj_t = torch.from_numpy(objs.view(np.uint8).copy()).to(device) if objs.size else None
    P = _Params()
    P.mode, P.seed = _MODE[base], cfg.seed
    P.gz, P.ny, P.nx, P.z0, P.nz = Z, Y, X, z0, nz
    P.nobj = int(objs.size)
    P.obj = obj_t.data_ptr() if obj_t is not None else None
    s = cfg.scale
    p = [0.0] * 16
    ring_t = None
    if base == "C1":
        p[:4] = [400.0, 60.0, 80.0, 4095.0]
    elif base == "C5":
        p[:2] = [350.0, 70.0]
    elif base == "C2":
        p[:6] = [0.02, 0.005, 0.05, (Y - 1) / 2.0, (X - 1) / 2.0, 0.01]
        r = rings(cfg)
        ring_t = torch.from_numpy(r).to(device)
        P.nring, P.ring = r.size // 3, ring_t.data_ptr()
    elif base == "C3":
        p[:10] = [float(cfg.frames or Z), 0.30 * X, 0.18 * X, 0.35 * Y, (Y - 1) / 2.0, (X - 1) / 2.0,
                  500.0, 350.0, 700.0, 1023.0]
    elif base == "C4":
        p[0] = p[1] = (Y - 1) / 2.0
        p[2] = 900.0 * s
        p[5] = 40.0 * s + 1.0
    for k, v in enumerate(p):
        P.p[k] = v
    if truth is not None:
        assert truth.dtype == torch.int32 and truth.numel() >= truth_words(cfg, nz) and truth.is_contiguous()
        truth.zero_()
        P.truth = truth.data_ptr()
    stream = torch.cuda.current_stream(out.device).cuda_stream
    rc = _load().synth_generate(ctypes.byref(P), ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(stream))
    if rc != 0:
        raise RuntimeError("synth_generate failed: cuda error %d" % rc)
    torch.cuda.current_stream(out.device).synchronize()   # keep obj/ring buffers alive until done
    del obj_t, ring_t
    return out


def flat_field(cfg, device="cuda"):
    """C3's background reference B(y, x) ("calibration scans without sample"): the gain-varied
    open-beam frame of the recipe, noise-free (an average of many calibration frames), uint16 bits in
    an int16 tensor (Y, X)."""
    import torch

    base = cfg.name.split("@")[0]
    assert base == "C3", "only the detector-frame config has a flat field"
    one = dataclasses.replace(cfg, shape=(1,) + tuple(cfg.shape[1:]))
    out = torch.empty((1,) + tuple(cfg.shape[1:]), dtype=torch.int16, device=device)
    Z, Y, X = one.shape
    P = _Params()
    P.mode, P.seed = 6, cfg.seed
    P.gz, P.ny, P.nx, P.z0, P.nz = 1, Y, X, 0, 1
    p = [0.0] * 16
    p[8], p[9] = 700.0, 1023.0
    for k, v in enumerate(p):
        P.p[k] = v
    stream = torch.cuda.current_stream(out.device).cuda_stream
    rc = _load().synth_generate(ctypes.byref(P), ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(stream))
    if rc != 0:
        raise RuntimeError("synth_generate failed: cuda error %d" % rc)
    return out[0]


def to_numpy(t, cfg):
    """Host copy with the config's numpy dtype (u16 bits reinterpreted from int16 storage)."""
    a = t.cpu().numpy()
    return a.view(np.uint16) if cfg.dtype == "u16" else a
