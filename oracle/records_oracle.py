"""Record-dump format restated in numpy (records.py:149-202).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  A dump is a 16-byte
header -- magic b"SSR1", key_width u16, value_width u16, n u64, little
endian (records.py:147-149, 165) -- then n packed rows, key bytes first
(records.py:166-169).  Pinned by tests/test_io_cli.py against dumps written
by the unmodified reference (tests/golden/make_golden_io.py).
"""

from __future__ import annotations

import struct

import numpy as np

MAGIC = b"SSR1"


def pack_rows(keys: np.ndarray, values) -> np.ndarray:
    """(n, row_bytes) uint8 matrix: key bytes then value bytes (records.py:122-127)."""
    n = len(keys)

    def mat(a):
        width = a.dtype.itemsize * int(np.prod(a.shape[1:], dtype=np.int64))
        return np.ascontiguousarray(a.astype(a.dtype.newbyteorder("<"))).view(np.uint8).reshape(n, width)

    parts = [mat(keys)] + ([] if values is None else [mat(values)])
    return parts[0] if len(parts) == 1 else np.hstack(parts)


def dump_bytes(keys: np.ndarray, values, key_width: int) -> bytes:
    """records.py:152-169 as a byte string."""
    rows = pack_rows(keys, values)
    vw = 0 if values is None else (rows.shape[1] - key_width // 8) * 8
    return MAGIC + struct.pack("<HHQ", key_width, vw, len(keys)) + rows.tobytes()


def parse_dump(blob: bytes):
    """records.py:172-202: (keys, values, key_kind); ValueError on bad input."""
    if len(blob) < 16 or blob[:4] != MAGIC:
        raise ValueError("not a record dump")
    kw, vw, n = struct.unpack("<HHQ", blob[4:16])
    row = (kw + vw) // 8
    payload = blob[16:]
    if kw not in (32, 64, 128) or len(payload) != n * row:
        raise ValueError("corrupt record dump header")
    mat = np.frombuffer(payload, np.uint8).reshape(n, row) if n else np.zeros((0, row), np.uint8)
    kb = kw // 8
    kcol = mat[:, :kb].copy()
    if kw == 32:
        keys, kind = kcol.view("<u4").reshape(n), "u32"
    elif kw == 64:
        keys, kind = kcol.view("<u8").reshape(n), "u64"
    else:
        keys, kind = kcol.view("<u8").reshape(n, 2), "u128"
    values = None
    if vw:
        vcol = mat[:, kb:].copy()
        values = vcol.view("<u4").reshape(n) if vw == 32 else (
            vcol.view("<u8").reshape(n) if vw == 64 else vcol.view("<u8").reshape(n, vw // 64))
    return keys, values, kind
