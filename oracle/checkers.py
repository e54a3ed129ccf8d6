"""Validators restating the reference oracle (oracle.py:61-160).

TEST INFRASTRUCTURE ONLY.  ``semisort_valid`` restates validate_semisort's
three properties by definition (permutation, contiguity, stability);
``semisort_valid_indexed`` is the O(n) form for value == record index
 used at sizes where the definition-level check does not
fit; ``reduce_by_key`` is the sort + reduceat fold equivalent to
oracle_collect_reduce (oracle.py:128-141) for count / sum64.
"""

from __future__ import annotations

import numpy as np

__all__ = ["semisort_valid", "semisort_valid_indexed", "reduce_by_key",
           "pairs_multiset_equal"]


def semisort_valid(keys_in, vals_in, keys_out, vals_out):
    """(is_permutation, is_contiguous, is_stable), oracle.py:61-125 semantics."""
    ki, ko = np.asarray(keys_in), np.asarray(keys_out)
    n = len(ki)
    if len(ko) != n:
        return False, False, False
    if n == 0:
        return True, True, True
    # contiguity: every key value forms exactly one run
    run_start = np.ones(n, dtype=bool)
    run_start[1:] = ko[1:] != ko[:-1]
    contiguous = len(np.unique(ko[run_start])) == int(run_start.sum())
    # stability: per-key subsequences of whole records are equal
    oi = np.argsort(ki, kind="stable")
    oo = np.argsort(ko, kind="stable")
    same = np.array_equal(ki[oi], ko[oo])
    if same and vals_in is not None:
        same = np.array_equal(np.asarray(vals_in)[oi], np.asarray(vals_out)[oo])
    if same:
        return True, contiguous, True
    # not stable; is it at least a permutation of records?
    def rows(k, v):
        cols = [np.asarray(k).astype(np.uint64)]
        if v is not None:
            vv = np.asarray(v)
            vv = vv.reshape(len(vv), -1).astype(np.uint64)
            cols.extend(vv[:, j] for j in range(vv.shape[1]))
        return np.stack(cols, axis=1)
    ri, ro = rows(ki, vals_in), rows(ko, vals_out)
    ri = ri[np.lexsort(ri.T[::-1])]
    ro = ro[np.lexsort(ro.T[::-1])]
    return bool(np.array_equal(ri, ro)), contiguous, False


def semisort_valid_indexed(keys_in, keys_out, vals_out):
    """O(n) check when the input values are 0..n-1."""
    ki, ko, vo = np.asarray(keys_in), np.asarray(keys_out), np.asarray(vals_out).astype(np.int64)
    n = len(ki)
    if len(ko) != n or len(vo) != n:
        return False
    if n == 0:
        return True
    if vo.min() < 0 or vo.max() >= n:
        return False
    seen = np.zeros(n, dtype=bool)
    seen[vo] = True
    if not seen.all():
        return False                       # permutation of record indices
    if not np.array_equal(ko, ki[vo]):
        return False                       # records intact
    brk = np.ones(n, dtype=bool)
    brk[1:] = ko[1:] != ko[:-1]
    if int(brk.sum()) != len(np.unique(ki)):
        return False                       # one run per distinct key
    inside = ~brk[1:]
    return bool(np.all(vo[1:][inside] > vo[:-1][inside]))   # stable


def reduce_by_key(keys, values, kind: str) -> dict:
    """Per-key count or wrapping uint64 sum (oracle.py:128-141 semantics)."""
    k = np.asarray(keys).astype(np.uint64)
    if len(k) == 0:
        return {}
    order = np.argsort(k, kind="stable")
    ks = k[order]
    start = np.flatnonzero(np.concatenate([[True], ks[1:] != ks[:-1]]))
    if kind == "count":
        agg = np.diff(np.append(start, len(ks)))
    else:
        v = np.asarray(values)
        if v.ndim == 2:
            v = v[:, 0]
        agg = np.add.reduceat(v.astype(np.uint64)[order], start)
    return dict(zip(ks[start].tolist(), np.asarray(agg, dtype=np.uint64).tolist()))


def pairs_multiset_equal(a, b) -> bool:
    """oracle.py:150-160: order-insensitive, no duplicate keys."""
    if len(a) != len(b):
        return False
    da = dict(a)
    if len(da) != len(a):
        return False
    return all(k in da and da[k] == v for k, v in b)
