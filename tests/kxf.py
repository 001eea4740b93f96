"""Reader for the KXF1 golden-fixture format written by oracle/gen_golden.cpp.

Layout: b"KXF1", u32 count, then per array: u32 name_len, name, 1-byte dtype
code, u64 byte count, raw little-endian data.
"""
from __future__ import annotations

import struct
from pathlib import Path

import numpy as np

_CODES = {"f": np.float64, "q": np.int64, "Q": np.uint64, "i": np.int32, "I": np.uint32,
          "B": np.uint8}

GOLDEN = Path(__file__).resolve().parent / "golden"


def read(path) -> dict[str, np.ndarray]:
    p = Path(path)
    if not p.is_absolute() and not p.exists():
        p = GOLDEN / p
    b = p.read_bytes()
    assert b[:4] == b"KXF1", p
    (count,) = struct.unpack_from("<I", b, 4)
    off = 8
    out = {}
    for _ in range(count):
        (nl,) = struct.unpack_from("<I", b, off)
        off += 4
        name = b[off:off + nl].decode()
        off += nl
        code = chr(b[off])
        off += 1
        (nb,) = struct.unpack_from("<Q", b, off)
        off += 8
        out[name] = np.frombuffer(b[off:off + nb], dtype=_CODES[code]).copy()
        off += nb
    return out
