"""CPU oracle for byte-view keys (TEST INFRASTRUCTURE ONLY; see __init__).

Restates hashing.py:56-66 (hash_bytes: mix64(poly(bytes) ^ mix64(len)), poly
the wrapping polynomial with multiplier 0x100000001B3) and the byte-view
semisort of core.py:566-598 with BytesKeyAdapter (adapters.py:200-275)
through its defining property: bucket ids depend only on the content hash,
heavy detection and leaf grouping only on content equality, and the lt
base case only on content order -- so the semisort of 128-bit identity keys
(hash, length) resp. (hash, exact content rank) is the byte-view semisort.
Pinned against the reference's own outputs (tests/golden/make_golden_bytes.py).
"""

from __future__ import annotations

import numpy as np

from .semisort_oracle import OracleParams, mix64_int, semisort

U64 = (1 << 64) - 1
POLY_MULT = 0x100000001B3


def hash_bytes(b: bytes) -> int:
    acc = 0
    for x in b:
        acc = (acc * POLY_MULT + x) & U64
    return mix64_int(acc ^ mix64_int(len(b)))


def contents(arena: np.ndarray, views: np.ndarray) -> list:
    buf = np.asarray(arena, dtype=np.uint8).tobytes()
    return [buf[int(o):int(o) + int(n)] for o, n in np.asarray(views, dtype=np.uint64).reshape(-1, 2)]


def semisort_bytes(arena, views, values, P: OracleParams, mode: str = "eq"):
    """(views_out, values_out, telemetry) of the reference's byte-view semisort."""
    cs = contents(arena, views)
    n = len(cs)
    keys = np.zeros((n, 2), dtype=np.uint64)
    keys[:, 0] = np.array([hash_bytes(c) for c in cs], dtype=np.uint64)
    if mode == "lt":
        order = {c: i for i, c in enumerate(sorted(set(cs)))}
        keys[:, 1] = np.array([order[c] for c in cs], dtype=np.uint64)
    else:
        keys[:, 1] = np.array([len(c) for c in cs], dtype=np.uint64)
    _, perm, tel = semisort(keys, np.arange(n, dtype=np.uint64), P, mode, True)
    p = perm.astype(np.int64)
    v = np.asarray(views, dtype=np.uint64).reshape(-1, 2)[p]
    vals = None if values is None else np.asarray(values)[p]
    return v, vals, tel
