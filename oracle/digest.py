"""Chunked byte-stream digests -- TEST INFRASTRUCTURE ONLY (no method arithmetic).

Full-size outputs (the kept mask K and the code stream of C3-C5: gigabytes) are compared by digest:
the byte stream is cut into fixed chunks of CHUNK bytes and each chunk hashed with BLAKE2b-128
(digests per 256 MiB chunk).  A mismatch names the first differing chunk.
The same class digests the oracle's streamed output (fed plane by plane) and the GPU's buffers."""
import concurrent.futures
import hashlib

import numpy as np

CHUNK = 256 << 20


def _h(b):
    return hashlib.blake2b(b, digest_size=16).hexdigest()


class ChunkDigest:
    """Feed bytes in any pieces; chunk k is bytes [k*CHUNK, (k+1)*CHUNK) of the concatenation."""

    def __init__(self, chunk=CHUNK):
        self.chunk = chunk
        self.cur = hashlib.blake2b(digest_size=16)
        self.fill = 0
        self.total = 0
        self.digests = []

    def feed(self, data):
        mv = memoryview(np.ascontiguousarray(data)).cast("B")
        i = 0
        while i < len(mv):
            take = min(self.chunk - self.fill, len(mv) - i)
            self.cur.update(mv[i:i + take])
            self.fill += take
            i += take
            if self.fill == self.chunk:
                self.digests.append(self.cur.hexdigest())
                self.cur = hashlib.blake2b(digest_size=16)
                self.fill = 0
        self.total += len(mv)
        return self

    def result(self):
        d = list(self.digests)
        if self.fill:
            d.append(self.cur.hexdigest())
        return {"bytes": self.total, "chunks": d}


def digest_buffer(arr, chunk=CHUNK, threads=16):
    """The same result as ChunkDigest().feed(arr).result(), chunks hashed in parallel (hashlib
    releases the GIL on large buffers)."""
    mv = memoryview(np.ascontiguousarray(arr)).cast("B")
    n = len(mv)
    starts = list(range(0, n, chunk))
    with concurrent.futures.ThreadPoolExecutor(max_workers=threads) as ex:
        d = list(ex.map(lambda s: _h(mv[s:s + chunk]), starts))
    return {"bytes": n, "chunks": d}


def first_mismatch(a, b):
    """Index of the first differing chunk of two digest results (None when equal)."""
    if a["bytes"] != b["bytes"]:
        return "bytes %d != %d" % (a["bytes"], b["bytes"])
    for k, (x, y) in enumerate(zip(a["chunks"], b["chunks"])):
        if x != y:
            return k
    return None


def table_digest(cmin, csize, kept):
    """Digest of a component table (min index, size, kept) as little-endian uint64 / uint64 / uint8."""
    h = hashlib.blake2b(digest_size=16)
    h.update(np.ascontiguousarray(cmin, dtype="<u8").tobytes())
    h.update(np.ascontiguousarray(csize, dtype="<u8").tobytes())
    h.update(np.ascontiguousarray(kept, dtype=np.uint8).tobytes())
    return h.hexdigest()


def source_hashes():
    """Provenance of a stored full-size result: BLAKE2b of the oracle sources the streaming mode
    runs and of the phantom generator's sources.  A stored result is valid only for these."""
    import os

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

    def h(files):
        d = hashlib.blake2b(digest_size=16)
        for f in files:
            with open(os.path.join(root, f), "rb") as fh:
                d.update(fh.read())
        return d.hexdigest()

    return {"oracle": h(["oracle/roix_oracle.c", "oracle/otsu.py", "oracle/stream.py", "oracle/digest.py"]),
            "synth": h(["synth/synth.cu", "synth/__init__.py"])}
