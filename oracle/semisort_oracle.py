"""Numpy restatement of the reference semisort / collect-reduce algorithm.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).  This is an
independent re-statement of the reference's *algorithm* — written as an
explicit work-list instead of the reference's recursion — so that tests can
compare the CUDA path against it byte for byte.  Every function names the
reference file:line it follows (paths relative to
``/root/reference/pkg/src/semisort/``).  The only third-party arithmetic is
numpy, exactly as in the reference (``pyproject.toml:10``): Philox4x64-10
``Generator.integers`` for sampling, stable argsort, bincount, cumsum.

Parity pin: ``tests/test_oracle_golden.py`` checks this module against the
fixtures ``tests/golden/make_golden.py`` produced by running the reference.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "M64", "mix64_int", "mix64_np", "mix64_pair_int", "OracleParams",
    "OracleTelemetry", "key_hash", "light_slice", "sample_heavy",
    "bucket_ids", "count_rows", "col_scan", "scatter_positions",
    "eq_leaf_order", "lt_leaf_order", "semisort", "local_refine", "collect_reduce",
    "DEPTH_LIMIT",
]

M64 = (1 << 64) - 1
_GAMMA = 0x9E3779B97F4A7C15          # hashing.py:14
_MUL1 = 0xBF58476D1CE4E5B9           # hashing.py:15
_MUL2 = 0x94D049BB133111EB           # hashing.py:16
DEPTH_LIMIT = 64                     # core.py:39


# --------------------------------------------------------------------------
# hashing (hashing.py:25-53)
# --------------------------------------------------------------------------

def mix64_int(x: int) -> int:
    """splitmix64 finalizer on a Python int (hashing.py:25-30)."""
    z = (x + _GAMMA) & M64
    z = ((z ^ (z >> 30)) * _MUL1) & M64
    z = ((z ^ (z >> 27)) * _MUL2) & M64
    return z ^ (z >> 31)


def mix64_np(a: np.ndarray) -> np.ndarray:
    """Vector form, uint64 wrap-around (hashing.py:33-42)."""
    z = np.asarray(a).astype(np.uint64) + np.uint64(_GAMMA)
    z = (z ^ (z >> np.uint64(30))) * np.uint64(_MUL1)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(_MUL2)
    return z ^ (z >> np.uint64(31))


def mix64_pair_int(a: int, b: int) -> int:
    """hashing.py:45-47: mix64(a ^ mix64(b))."""
    return mix64_int(a ^ mix64_int(b))


# --------------------------------------------------------------------------
# parameters (params.py:36-123)
# --------------------------------------------------------------------------

@dataclass(frozen=True)
class OracleParams:
    n: int
    n_light: int
    bits: int
    sub_len: int
    alpha: int
    max_heavy: int
    sample_factor: int
    seed: int
    samples: int
    threshold: float

    @staticmethod
    def derive(n, *, light_buckets=1 << 10, subarray_len=None,
               base_case_cutoff=1 << 14, max_heavy=500, sample_factor=500,
               seed=1) -> "OracleParams":
        """params.py:64-103 (for_input)."""
        if subarray_len is None:
            subarray_len = max(max(1, -(-n // 5000)), light_buckets)
        log_n = math.log2(max(n, 2))
        return OracleParams(n, light_buckets, light_buckets.bit_length() - 1,
                            subarray_len, base_case_cutoff, max_heavy,
                            sample_factor, seed,
                            max(1, round(sample_factor * log_n)), log_n)

    @property
    def rounds(self) -> int:
        """params.py:120-123."""
        return max(1, 64 // max(self.bits, 1))

    def nsub(self, m: int) -> int:
        """params.py:117-118."""
        return -(-m // self.sub_len)


@dataclass
class OracleTelemetry:
    """Counter semantics of core.py:42-61."""
    max_depth: int = 0
    nodes: int = 0
    scratch_allocations: int = 0
    scratch_moves: int = 0
    bucket_assignments: int = 0
    matrix_cells_by_level: dict = field(default_factory=dict)

    def seen(self, level: int, count: int = 1) -> None:
        self.nodes += count
        self.max_depth = max(self.max_depth, level)

    def cells(self, level: int, c: int) -> None:
        self.matrix_cells_by_level[level] = self.matrix_cells_by_level.get(level, 0) + c


# --------------------------------------------------------------------------
# bucket ids (core.py:139-213, adapters.py:112-119)
# --------------------------------------------------------------------------

def key_hash(keys: np.ndarray, identity: bool) -> np.ndarray:
    """adapters.py:112-116: u64 widening, then mix64 unless identity.

    128-bit keys ((n, 2) u64 rows, column 0 = lo; records.py:8-10) hash as
    mix64(mix64(hi) ^ lo), or lo in identity mode (adapters.py:155-159).
    """
    k = np.asarray(keys)
    if k.ndim == 2:
        lo, hi = k[:, 0].astype(np.uint64), k[:, 1].astype(np.uint64)
        return lo.copy() if identity else mix64_np(mix64_np(hi) ^ lo)
    k = k.astype(np.uint64)
    return k if identity else mix64_np(k)


def _kv(keys: np.ndarray) -> np.ndarray:
    """1-D view usable for equality / np.unique: 128-bit rows become void16."""
    k = np.asarray(keys)
    if k.ndim == 1:
        return k.astype(np.uint64)
    return np.ascontiguousarray(k, dtype=np.uint64).view(np.dtype((np.void, 16))).ravel()


def _key_obj(row):
    """Canonical key (adapters.py:161-166): an int, or (lo, hi) for 128-bit."""
    return (int(row[0]), int(row[1])) if np.ndim(row) else int(row)


def light_slice(h: np.ndarray, depth: int, P: OracleParams) -> np.ndarray:
    """core.py:146-151: b-bit slice of the (round-remixed) hash."""
    rnd, slot = divmod(depth, P.rounds)
    h = np.asarray(h, dtype=np.uint64)
    if rnd:
        h = mix64_np(h ^ np.uint64(mix64_int(rnd)))
    return ((h >> np.uint64(slot * P.bits)) & np.uint64(P.n_light - 1)).astype(np.int64)


def sample_heavy(keys: np.ndarray, P: OracleParams, rng_key: int) -> list:
    """core.py:221-260 restated with numpy set operations.

    Draw min(m, |S|) positions from Philox(key=rng_key) (core.py:238-239),
    count sampled keys in stream order, keep keys with count >= threshold,
    cap to max_heavy by (-count, first stream position), return them in
    discovery (first stream position) order.
    """
    m = len(keys)
    draws = min(m, P.samples)
    if draws == 0 or P.max_heavy == 0:
        return []
    pos = np.random.Generator(np.random.Philox(key=rng_key)).integers(0, m, size=draws)
    s = np.asarray(keys)[pos].astype(np.uint64)
    _, first, cnt = np.unique(_kv(s), return_index=True, return_counts=True)
    keep = cnt >= P.threshold
    first, cnt = first[keep], cnt[keep]
    if len(first) > P.max_heavy:
        sel = np.lexsort((first, -cnt))[: P.max_heavy]
        first = first[sel]
    first = np.sort(first)
    return [_key_obj(s[f]) for f in first]


def bucket_ids(keys: np.ndarray, heavy: list, P: OracleParams, depth: int,
               identity: bool) -> np.ndarray:
    """core.py:169-213: light slice, overridden by heavy id n_L + slot."""
    k = np.asarray(keys).astype(np.uint64)
    ids = light_slice(key_hash(k, identity), depth, P)
    if heavy and k.ndim == 2:   # 128-bit: match row by row (adapters.py:187-191)
        kv = _kv(k)
        tv = _kv(np.asarray(heavy, dtype=np.uint64).reshape(-1, 2))
        for slot in range(len(tv)):
            ids[kv == tv[slot]] = P.n_light + slot
    elif heavy:
        table = np.asarray(heavy, dtype=np.uint64)
        order = np.argsort(table, kind="stable")
        st = table[order]
        at = np.searchsorted(st, k)
        at_c = np.minimum(at, len(st) - 1)
        hit = (at < len(st)) & (st[at_c] == k)
        ids[hit] = P.n_light + order[at_c[hit]]
    return ids


# --------------------------------------------------------------------------
# blocked distributing (core.py:268-380)
# --------------------------------------------------------------------------

def count_rows(ids: np.ndarray, sub_len: int, n_buckets: int) -> np.ndarray:
    """core.py:268-291: C[i][j] = #records of subarray i in bucket j."""
    m = len(ids)
    rows = -(-m // sub_len)
    flat = (np.arange(m, dtype=np.int64) // sub_len) * n_buckets + np.asarray(ids, np.int64)
    return np.bincount(flat, minlength=rows * n_buckets).reshape(rows, n_buckets).astype(np.int64)


def col_scan(C: np.ndarray):
    """core.py:302-318: column-major exclusive scan -> (X, offsets)."""
    rows, nb = C.shape
    run = np.concatenate([[0], np.cumsum(C.T.reshape(-1), dtype=np.int64)])
    X = run[:-1].reshape(nb, rows).T.copy()
    off = np.empty(nb + 1, dtype=np.int64)
    off[:nb] = X[0] if rows else 0
    off[nb] = run[-1]
    return X, off


def scatter_positions(ids: np.ndarray, X: np.ndarray, sub_len: int) -> np.ndarray:
    """core.py:321-362: dest = X[sub][b] + stable rank within (sub, b)."""
    m = len(ids)
    ids = np.asarray(ids, np.int64)
    sub = np.arange(m, dtype=np.int64) // sub_len
    comp = sub * X.shape[1] + ids
    order = np.argsort(comp, kind="stable")
    sc = comp[order]
    start = np.ones(m, dtype=bool)
    start[1:] = sc[1:] != sc[:-1]
    first_idx = np.maximum.accumulate(np.where(start, np.arange(m), 0))
    rank = np.empty(m, dtype=np.int64)
    rank[order] = np.arange(m) - first_idx
    return X[sub, ids] + rank


# --------------------------------------------------------------------------
# base cases (core.py:388-429, adapters.py:81-135)
# --------------------------------------------------------------------------

def eq_leaf_order(keys: np.ndarray, identity: bool) -> np.ndarray:
    """Permutation of the chained-hash base case (core.py:388-422).

    Groups (distinct keys) are ordered by (hash & (cap-1), first index)
    with cap the smallest power of two >= 2m; records keep input order
    inside a group.
    """
    k = np.asarray(keys).astype(np.uint64)
    m = len(k)
    if m < 2:
        return np.arange(m)
    uniq, first, inv = np.unique(_kv(k), return_index=True, return_inverse=True)
    cap = 1 << max(1, 2 * m - 1).bit_length()
    cell = (key_hash(k[first], identity) & np.uint64(cap - 1)).astype(np.int64)
    grank = np.empty(len(uniq), dtype=np.int64)
    grank[np.lexsort((first, cell))] = np.arange(len(uniq))
    return np.argsort(grank[inv.reshape(-1)], kind="stable")


def lt_leaf_order(keys: np.ndarray) -> np.ndarray:
    """core.py:425-429 / adapters.py:132-135: stable sort by key; 128-bit
    keys by (hi, lo) (adapters.py:178-182)."""
    k = np.asarray(keys)
    if k.ndim == 2:
        return np.lexsort((k[:, 0], k[:, 1]))
    return np.argsort(k, kind="stable")


# --------------------------------------------------------------------------
# semisort (core.py:437-598), as an explicit work-list
# --------------------------------------------------------------------------

def _stall(P, size, parent_size, depth, stalled):
    """core.py:452-458 safety valve."""
    if parent_size is not None and 2 * size > parent_size:
        stalled += 1
        if stalled == 1:
            depth = (depth // P.rounds + 1) * P.rounds
    return depth, stalled


def semisort(keys, values, P: OracleParams, mode: str = "eq", identity: bool = False):
    """Return (keys, values, telemetry) after the reference semisort.

    Same output bytes as core.semisort (core.py:566-598) for the same
    params: node processing order does not affect any node's result.
    """
    if mode not in ("eq", "lt"):
        raise ValueError(mode)
    A = [np.array(keys, copy=True), None if values is None else np.array(values, copy=True)]
    n = len(A[0])
    if P.n != n:
        raise ValueError("params bound to another n")
    S = [np.empty_like(A[0]), None if A[1] is None else np.empty_like(A[1])]
    tel = OracleTelemetry(scratch_allocations=1)
    _drive(A, S, [(0, n, 1, 0, True, 0, None, 0)], P, mode, identity, tel)
    return A[0], A[1], tel


def local_refine(primary, scratch, offsets, live_in_primary: bool, P: OracleParams, mode: str = "eq",
                 identity: bool = False, depth: int = 0):
    """core.py:533-563: refine the light buckets of a node already
    distributed into the live buffer; returns (primary keys, values, tel).
    primary / scratch: (keys, values) arrays of the node's size."""
    A = [np.array(primary[0], copy=True), None if primary[1] is None else np.array(primary[1], copy=True)]
    S = [np.array(scratch[0], copy=True), None if scratch[1] is None else np.array(scratch[1], copy=True)]
    tel = OracleTelemetry()
    off = [int(x) for x in offsets]
    total = off[-1]
    if not live_in_primary and off[P.n_light] < total:      # heavy buckets are final
        h0 = off[P.n_light]
        A[0][h0:total] = S[0][h0:total]
        if A[1] is not None:
            A[1][h0:total] = S[1][h0:total]
    smalls, bigs = [], []
    for b in range(P.n_light):
        lo, hi = off[b], off[b + 1]
        if hi > lo:
            (smalls if hi - lo < P.alpha else bigs).append((b, lo, hi))
    work = [(lo, hi, 1, depth + 1, live_in_primary, mix64_pair_int(P.seed, b + 1), total, 0)
            for b, lo, hi in reversed(bigs)]
    _drive(A, S, work, P, mode, identity, tel, first_leaves=[(lo, hi) for _, lo, hi in smalls],
           leaves_in_a=live_in_primary)
    return A[0], A[1], tel


def _drive(A, S, work, P, mode, identity, tel, first_leaves=(), leaves_in_a=True):
    """The recursion (core.py:437-530) as an explicit work list over
    (lo, hi, level, depth, in_a, path, parent_size, stalled) nodes."""

    def buf(in_a):
        return A if in_a else S

    def move(dst, dpos, src, spos):
        dst[0][dpos] = src[0][spos]
        if src[1] is not None:
            dst[1][dpos] = src[1][spos]

    def leaf(lo, hi, in_a):
        B = buf(in_a)
        if hi - lo >= 2:
            kk = B[0][lo:hi]
            perm = lt_leaf_order(kk) if mode == "lt" else eq_leaf_order(kk, identity)
            move(B, slice(lo, hi), B, lo + perm)
        if not in_a:
            move(A, slice(lo, hi), S, slice(lo, hi))

    if first_leaves:
        tel.seen(1, len(first_leaves))
        for lo, hi in first_leaves:
            leaf(lo, hi, leaves_in_a)
    while work:
        lo, hi, level, depth, in_a, path, parent, stalled = work.pop()
        size = hi - lo
        tel.seen(level)
        depth, stalled = _stall(P, size, parent, depth, stalled)
        if size < P.alpha or stalled >= 2 or level >= DEPTH_LIMIT:
            leaf(lo, hi, in_a)
            continue
        src, dst = buf(in_a), buf(not in_a)
        wk = src[0][lo:hi]
        heavy = sample_heavy(wk, P, mix64_pair_int(P.seed, path))
        nb = P.n_light + len(heavy)
        ids = bucket_ids(wk, heavy, P, depth, identity)
        tel.bucket_assignments += size
        C = count_rows(ids, P.sub_len, nb)
        tel.cells(level, C.size)
        X, off = col_scan(C)
        move(dst, lo + scatter_positions(ids, X, P.sub_len), src, slice(lo, hi))
        if in_a:  # dst is the scratch: heavy buckets are final, copy them back
            tel.scratch_moves += size
            if off[P.n_light] < size:
                move(A, slice(lo + int(off[P.n_light]), hi), S, slice(lo + int(off[P.n_light]), hi))
        smalls, bigs = [], []
        for b in range(P.n_light):
            b_lo, b_hi = int(off[b]), int(off[b + 1])
            if b_hi == b_lo:
                continue
            (smalls if b_hi - b_lo < P.alpha else bigs).append((b, lo + b_lo, lo + b_hi))
        if smalls:
            tel.seen(level + 1, len(smalls))
            for _, c_lo, c_hi in smalls:
                leaf(c_lo, c_hi, not in_a)
        for b, c_lo, c_hi in reversed(bigs):
            work.append((c_lo, c_hi, level + 1, depth + 1, not in_a,
                         mix64_pair_int(path, b + 1), size, stalled))


# --------------------------------------------------------------------------
# collect-reduce / histogram (aggregate.py:133-299)
# --------------------------------------------------------------------------

def _as_u64_values(values):
    """aggregate.py:197-203 (_map_u64): first word, widened to uint64."""
    if values is None:
        raise ValueError("summing64 needs a value column")
    v = np.asarray(values)
    if v.ndim == 2:
        v = v[:, 0]
    return v.astype(np.uint64)


def collect_reduce(keys, values, P: OracleParams, kind: str, identity: bool = False):
    """Return (pairs, telemetry); pairs in the reference's DFS order.

    kind is "count" (histogram, aggregate.py:293-299) or "sum64"
    (ReduceSpec.summing64, aggregate.py:67-79).  Output order follows
    aggregate.py:10-12: heavy pairs of a node, then its light buckets
    ascending, depth-first; leaves emit in chained-hash order.
    """
    keys = np.asarray(keys)
    n = len(keys)
    if P.n != n:
        raise ValueError("params bound to another n")
    tel = OracleTelemetry()
    out: list = []

    def fold_leaf(k, v):
        m = len(k)
        if m == 0:
            return
        ku = k.astype(np.uint64)
        uniq, first, inv = np.unique(ku, return_index=True, return_inverse=True)
        inv = inv.reshape(-1)
        cap = 1 << max(1, 2 * m - 1).bit_length()
        cell = (key_hash(uniq, identity) & np.uint64(cap - 1)).astype(np.int64)
        order = np.lexsort((first, cell))
        if kind == "count":
            agg = np.bincount(inv, minlength=len(uniq)).astype(np.uint64)
        else:
            agg = np.zeros(len(uniq), dtype=np.uint64)
            np.add.at(agg, inv, _as_u64_values(v))
        out.extend((int(uniq[g]), int(agg[g])) for g in order)

    # explicit DFS stack; each frame emits before its children (pre-order)
    stack = [(keys, values, 1, 0, 0, None, 0)]
    while stack:
        k, v, level, depth, path, parent, stalled = stack.pop()
        size = len(k)
        tel.seen(level)
        depth, stalled = _stall(P, size, parent, depth, stalled)
        if size < P.alpha or stalled >= 2 or level >= DEPTH_LIMIT:
            fold_leaf(k, v)
            continue
        heavy = sample_heavy(k, P, mix64_pair_int(P.seed, path))
        nl = P.n_light
        ids = bucket_ids(k, heavy, P, depth, identity)
        tel.bucket_assignments += size
        C = count_rows(ids, P.sub_len, nl + len(heavy))
        tel.cells(level, C.size)
        if heavy:
            if kind == "count":
                tot = C[:, nl:].sum(axis=0)
            else:
                tot = np.zeros(len(heavy), dtype=np.uint64)
                hp = np.flatnonzero(ids >= nl)
                np.add.at(tot, ids[hp] - nl, _as_u64_values(v)[hp])
            out.extend((heavy[t], int(tot[t])) for t in range(len(heavy)))
        X, off = col_scan(C[:, :nl])
        total = int(off[-1])
        if total == 0:
            continue
        light = np.flatnonzero(ids < nl)
        # light-only stable scatter (aggregate.py:172-193): subarray of each
        # light record is that of its position in the window.
        sub = light // P.sub_len
        comp = sub * nl + ids[light]
        order = np.argsort(comp, kind="stable")
        sc = comp[order]
        start = np.ones(len(sc), dtype=bool)
        start[1:] = sc[1:] != sc[:-1]
        first_idx = np.maximum.accumulate(np.where(start, np.arange(len(sc)), 0))
        rank = np.empty(len(sc), dtype=np.int64)
        rank[order] = np.arange(len(sc)) - first_idx
        dest = X[sub, ids[light]] + rank
        ck = np.empty(total, dtype=k.dtype)
        ck[dest] = k[light]
        cv = None
        if v is not None:
            cv = np.empty((total,) + np.asarray(v).shape[1:], dtype=np.asarray(v).dtype)
            cv[dest] = np.asarray(v)[light]
        tel.scratch_moves += total
        frames = []
        for b in range(nl):
            b_lo, b_hi = int(off[b]), int(off[b + 1])
            if b_hi > b_lo:
                frames.append((ck[b_lo:b_hi], None if cv is None else cv[b_lo:b_hi],
                               level + 1, depth + 1, mix64_pair_int(path, b + 1), size, stalled))
        stack.extend(reversed(frames))
    return out, tel
