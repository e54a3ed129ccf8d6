"""Golden fixtures for 128-bit keys, made by the UNMODIFIED reference.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden_u128.py

Runs the reference's ``semisort`` with ``UInt128KeyAdapter`` (adapters.py:
147-198; keys stored as (n, 2) uint64 rows, column 0 = lo, records.py:8-10)
on seeded inputs and writes ``golden_u128.npz``: inputs, outputs and the
heavy keys the reference's sampler returns.  Nothing at test time reads
/root/reference.
"""

from __future__ import annotations

import os
import sys

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
HERE = os.path.dirname(os.path.abspath(__file__))

import semisort as S  # noqa: E402

A = S.UInt128KeyAdapter()
AI = S.UInt128KeyAdapter(identity=True)


def rows(lo, hi):
    k = np.empty((len(lo), 2), dtype=np.uint64)
    k[:, 0] = lo
    k[:, 1] = hi
    return k


def cases():
    r = np.random.default_rng(128)
    out = []
    # the reference test's shape (test_semisort.py:132-143)
    out.append(("reftest", rows(r.integers(0, 50, 5000), r.integers(0, 3, 5000)),
                dict(light_buckets=8, base_case_cutoff=64, max_heavy=4)))
    # distinct wide keys, default params
    out.append(("wide", rows(r.integers(0, 2**64 - 1, 6000, dtype=np.uint64, endpoint=True),
                             r.integers(0, 2**64 - 1, 6000, dtype=np.uint64, endpoint=True)), {}))
    # same lo, different hi: one identity-hash bucket, distinct keys
    out.append(("samelo", rows(np.full(4000, 7, np.uint64), r.integers(0, 300, 4000)),
                dict(light_buckets=16, base_case_cutoff=32, subarray_len=64)))
    # skewed: a few heavy keys differing only in hi, plus a uniform tail
    m = 20000
    lo = r.integers(0, 2**40, m).astype(np.uint64)
    hi = r.integers(0, 2**40, m).astype(np.uint64)
    hot = r.random(m) < 0.6
    lo[hot] = 99
    hi[hot] = r.integers(0, 3, int(hot.sum()))
    out.append(("skew", rows(lo, hi), dict(light_buckets=32, base_case_cutoff=128, max_heavy=8)))
    # recursion at small n (the reference tests' recursive_params shape)
    out.append(("recur", rows(r.integers(0, 40, 3000), r.integers(0, 2, 3000)),
                dict(light_buckets=4, subarray_len=8, base_case_cutoff=8, max_heavy=2)))
    out.append(("one", rows(np.array([5], np.uint64), np.array([9], np.uint64)), {}))
    out.append(("empty", np.zeros((0, 2), np.uint64), {}))
    return out


def main():
    z: dict[str, np.ndarray] = {}
    names = []
    for name, keys, kw in cases():
        n = len(keys)
        for mode in ("eq", "lt"):
            for ident in (False, True):
                for with_v in (False, True):
                    if mode == "lt" and ident:
                        continue   # identity only changes hashing: lt output is the same
                    tag = f"{name}_{mode}_{int(ident)}_{int(with_v)}"
                    vals = np.arange(n, dtype=np.uint64) * 3 + 1 if with_v else None
                    data = S.RecordArray(keys.copy(), None if vals is None else vals.copy())
                    params = S.TuningParams.for_input(n, **kw)
                    S.semisort(data, AI if ident else A, mode, params)
                    z[f"{tag}_out_k"] = np.asarray(data.keys)
                    if with_v:
                        z[f"{tag}_out_v"] = np.asarray(data.values)
                    names.append(tag)
        z[f"{name}_keys"] = keys
        z[f"{name}_params"] = np.array([kw.get(k, -1) for k in
                                        ("light_buckets", "subarray_len", "base_case_cutoff", "max_heavy")],
                                       dtype=np.int64)
        if n:
            params = S.TuningParams.for_input(n, **kw)
            for ident in (False, True):
                t = S.sample_and_bucket(S.RecordArray(keys.copy()), AI if ident else A, params, 0,
                                        np.random.Generator(np.random.Philox(key=1234)))
                z[f"{name}_heavy_{int(ident)}"] = np.asarray(t.keys, dtype=np.uint64).reshape(-1, 2)
    z["tags"] = np.array(names)
    z["cases"] = np.array([c[0] for c in cases()])
    np.savez_compressed(os.path.join(HERE, "golden_u128.npz"), **z)
    print(len(names), "semisort cases")


if __name__ == "__main__":
    main()
