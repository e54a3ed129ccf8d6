"""CPU restatement of the reference graph transpose / CSR build.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Follows graphs.py:59-105:
``csr_from_edges`` = bincount + cumsum offsets, stable argsort by source
(graphs.py:59-71); ``transpose`` = expand sources by degree, semisort the
(target, source) records with the identity hash (the oracle semisort,
core.py:566-598), then rebuild the offsets from in-degrees and place each
run of equal targets at its offset (graphs.py:77-105).
"""

from __future__ import annotations

import numpy as np

from .semisort_oracle import OracleParams, semisort

__all__ = ["csr_from_edges", "transpose"]


def csr_from_edges(n: int, sources, targets):
    """graphs.py:59-71 -> (offsets u64[n+1], targets u32[m])."""
    s = np.asarray(sources, dtype=np.uint32)
    t = np.asarray(targets, dtype=np.uint32)
    m = len(s)
    counts = np.bincount(s, minlength=n) if m else np.zeros(n, dtype=np.int64)
    off = np.zeros(n + 1, dtype=np.uint64)
    np.cumsum(counts, out=off[1:])
    return off, t[np.argsort(s, kind="stable")]


def transpose(n: int, offsets, targets, params: OracleParams | None = None):
    """graphs.py:77-105 -> (offsets u64[n+1], targets u32[m])."""
    off = np.asarray(offsets, dtype=np.uint64)
    tg = np.asarray(targets, dtype=np.uint32)
    m = len(tg)
    deg = np.diff(off.astype(np.int64))
    src = np.repeat(np.arange(n, dtype=np.uint32), deg)
    P = params if params is not None else OracleParams.derive(m)
    keys, vals, _ = semisort(tg.copy(), src, P, "eq", identity=True)
    counts = np.bincount(tg, minlength=n) if m else np.zeros(n, dtype=np.int64)
    new_off = np.zeros(n + 1, dtype=np.uint64)
    np.cumsum(counts, out=new_off[1:])
    out = np.empty(m, dtype=np.uint32)
    if m:
        start = np.flatnonzero(np.concatenate([[True], keys[1:] != keys[:-1]]))
        size = np.diff(np.append(start, m))
        base = new_off[keys[start]].astype(np.int64)
        within = np.arange(m, dtype=np.int64) - np.repeat(start, size)
        out[np.repeat(base, size) + within] = vals
    return new_off, out
