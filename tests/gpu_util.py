"""Helpers for the -m gpu parity tests: device buffers, scalars read/write, calls through the C ABI."""
import ctypes

import numpy as np
import torch

from paper_2602_15917_b200 import _lib as L


def ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def st():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def dev(a):
    a = np.ascontiguousarray(a)
    if a.dtype == np.uint16:
        return torch.from_numpy(a.view(np.int16).copy()).cuda()
    return torch.from_numpy(a.copy()).cuda()


def host_u16(t):
    return t.cpu().numpy().view(np.uint16)


def dtype_code(a):
    return L.U16 if a.dtype == np.uint16 else L.F32


def ord2f(o):
    """Host decode of roix_scalars.min_ord / max_ord (ordered-integer fp32 encoding)."""
    b = (o & 0x7FFFFFFF) if (o & 0x80000000) else (~o & 0xFFFFFFFF)
    return float(np.array([b], np.uint32).view(np.float32)[0])


def new_sc(eb=0.0):
    sc = torch.zeros(L.scalars_size(), dtype=torch.uint8, device="cuda")
    L.roix_scalars_init(ptr(sc), eb, st())
    return sc


def read_sc(sc):
    torch.cuda.synchronize()
    return L.Scalars.from_buffer_copy(bytes(sc.cpu().numpy()))


def write_sc(sc, s):
    sc.copy_(torch.frombuffer(bytearray(bytes(s)), dtype=torch.uint8).cuda())


def words_to_mask(words, n):
    w = words.cpu().numpy().astype(np.int32).view(np.uint8)
    return np.unpackbits(w, bitorder="little")[:n]


def mask_to_words(mask):
    import oracle

    w = oracle.pack_bits(mask).view(np.int32)
    return torch.from_numpy(np.concatenate([w, np.zeros(4, np.int32)])).cuda()


def gpu_threshold(x_np, eb=1.0, rel_eb=0.0, polarity=0):
    """Scalars after range/resolve/histogram/threshold on x (all through the C ABI)."""
    x = dev(x_np)
    dt = dtype_code(x_np)
    sc = new_sc(0.0 if rel_eb else eb)
    n = x_np.size
    if dt == L.F32:
        L.roix_range(ptr(x), n, ptr(sc), st())
    L.roix_resolve(ptr(sc), dt, rel_eb, st())
    nb = 65536 if dt == L.U16 else 256
    h = torch.zeros(nb, dtype=torch.int64, device="cuda")
    L.roix_histogram(ptr(x), dt, n, ptr(sc), ptr(h), nb, st())
    L.roix_threshold(ptr(h), nb, dt, polarity, ptr(sc), st())
    return x, sc, h
