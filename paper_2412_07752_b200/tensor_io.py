"""RTN1 named-tensor files (the reference's golden-vector / parameter container,
rnnkit tensor_io.hpp:11-35), numpy side.  The C++ side is
include/flashrnn/tensor_io.hpp.

Layout (little-endian): b"RTN1", u32 count, then per tensor: u16 name length,
name bytes, u8 dtype tag (0 = float64), u8 rank, u64 dims[rank], f64 payload
row-major.  Entries are written in name order (the reference stores a
std::map), so files round-trip byte-identically with the reference writer.
"""
from __future__ import annotations

import struct

import numpy as np

MAGIC = b"RTN1"


def save_tensors(path: str, tensors: dict) -> None:
    with open(path, "wb") as f:
        f.write(MAGIC)
        f.write(struct.pack("<I", len(tensors)))
        for name in sorted(tensors, key=lambda s: s.encode()):
            a = np.ascontiguousarray(tensors[name], dtype="<f8")
            nb = name.encode()
            f.write(struct.pack("<H", len(nb)) + nb + struct.pack("<BB", 0, a.ndim))
            f.write(struct.pack(f"<{a.ndim}Q", *a.shape))
            f.write(a.tobytes())


def load_tensors(path: str) -> dict:
    with open(path, "rb") as f:
        buf = f.read()
    if buf[:4] != MAGIC:
        raise ValueError(f"not a tensor file: {path}")
    (count,) = struct.unpack_from("<I", buf, 4)
    off, out = 8, {}
    for _ in range(count):
        (n,) = struct.unpack_from("<H", buf, off)
        off += 2
        name = buf[off:off + n].decode()
        off += n
        tag, rank = struct.unpack_from("<BB", buf, off)
        off += 2
        if tag != 0:
            raise ValueError(f"unsupported dtype tag in {path}")
        dims = struct.unpack_from(f"<{rank}Q", buf, off)
        off += 8 * rank
        count_el = int(np.prod(dims, dtype=np.int64)) if rank else 1
        if off + 8 * count_el > len(buf):
            raise ValueError(f"truncated tensor payload in {path}")
        out[name] = np.frombuffer(buf, dtype="<f8", count=count_el, offset=off).reshape(dims).copy()
        off += 8 * count_el
    return out
