"""Golden fixtures for local_refine and for _distribute_ids on a window with
base > 0, produced by the UNMODIFIED reference (run in the build container):

    python tests/golden/make_golden_refine.py   ->  tests/golden/golden_refine.npz

local_refine cases follow the reference test's flow
(test_semisort.py:226-245): sample_and_bucket with a Philox(key) stream ->
assign_bucket_ids -> _counts_from_ids -> column_major_exclusive_scan ->
_distribute_ids into the other buffer -> local_refine; stored: the inputs,
the heavy keys and the refined primary buffer with the telemetry.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
HERE = os.path.dirname(os.path.abspath(__file__))

import semisort as S  # noqa: E402
from semisort import core as C  # noqa: E402

CASES = [   # name, n, key range, params, philox key, live_in_primary, mode, identity
    ("ref_test", 4096, 1500, dict(light_buckets=8, subarray_len=64, base_case_cutoff=128, max_heavy=4), 5, False,
     "eq", False),
    ("ref_test_live", 4096, 1500, dict(light_buckets=8, subarray_len=64, base_case_cutoff=128, max_heavy=4), 5, True,
     "eq", False),
    ("ref_test_lt", 4096, 1500, dict(light_buckets=8, subarray_len=64, base_case_cutoff=128, max_heavy=4), 5, False,
     "lt", False),
    ("identity", 6000, 3000, dict(light_buckets=16, subarray_len=128, base_case_cutoff=64, max_heavy=8), 9, False,
     "eq", True),
    ("deep", 50000, 40000, dict(light_buckets=8, subarray_len=256, base_case_cutoff=256, max_heavy=4), 11, False,
     "eq", False),
    ("skewed_live", 30000, None, dict(light_buckets=16, subarray_len=512, base_case_cutoff=512, max_heavy=16), 13,
     True, "eq", False),
    ("default_params", 1 << 16, 1 << 14, dict(), 21, False, "eq", False),
]


def keys_for(rng, n, rng_max):
    if rng_max is None:   # Zipf-ish with a few very frequent keys
        return np.minimum(rng.zipf(1.3, n), 10**6).astype(np.uint64)
    return rng.integers(0, rng_max, n).astype(np.uint64)


def main():
    out, meta = {}, {"refine": [], "window": []}
    for name, n, kr, kw, pk, live, mode, ident in CASES:
        rng = np.random.default_rng(n + pk)
        keys = keys_for(rng, n, kr)
        vals = np.arange(n, dtype=np.uint64)
        adp = S.UIntKeyAdapter(identity=ident)
        P = S.TuningParams.for_input(n, **kw)
        data = S.RecordArray(keys.copy(), vals.copy())
        heavy = C.sample_and_bucket(data, adp, P, 0, np.random.Generator(np.random.Philox(key=pk)))
        ids = C.assign_bucket_ids(data, heavy, adp, P, 0)
        nb = P.light_buckets + len(heavy)
        counts = C._counts_from_ids(ids, P, nb)
        prefix, offsets = C.column_major_exclusive_scan(counts)
        other = data.empty_like()
        C._distribute_ids(data, other, 0, ids, prefix, P, nb)
        if live:
            bufs = C.WorkBuffers(primary=other, scratch=data.empty_like(), live_in_primary=True)
        else:
            bufs = C.WorkBuffers(primary=data, scratch=other, live_in_primary=False)
        tel = C.Telemetry()
        C.local_refine(bufs, C.BucketPlan(heavy, counts, prefix, offsets), adp, mode, P, depth=0, telemetry=tel)
        p = f"rf_{name}_"
        out[p + "keys"], out[p + "heavy"] = keys, np.asarray(heavy.keys, dtype=np.uint64)
        out[p + "out_keys"], out[p + "out_vals"] = bufs.primary.keys.copy(), bufs.primary.values.copy()
        meta["refine"].append({"name": name, "params": kw, "philox_key": pk, "live_in_primary": live, "mode": mode,
                               "identity": ident,
                               "telemetry": {"max_depth": tel.max_depth, "nodes": tel.nodes,
                                             "scratch_moves": tel.scratch_moves,
                                             "bucket_assignments": tel.bucket_assignments,
                                             "matrix_cells_by_level": {str(k): v for k, v in
                                                                       tel.matrix_cells_by_level.items()}}})
    # _distribute_ids on a window [base, base + m) of larger arrays (core.py:339-362)
    for name, total, base, m, kw in (("mid", 20000, 7000, 5000, dict(light_buckets=8, subarray_len=64)),
                                     ("tail", 9000, 8000, 1000, dict(light_buckets=4, subarray_len=16)),
                                     ("head_part", 9000, 0, 3000, dict(light_buckets=16, subarray_len=256))):
        rng = np.random.default_rng(total + base)
        keys = rng.integers(0, 10**6, total).astype(np.uint64)
        vals = rng.integers(0, 2**63, total).astype(np.uint64)
        P = S.TuningParams.for_input(m, **kw)
        ids = rng.integers(0, P.light_buckets, m).astype(np.int32)
        counts = C._counts_from_ids(ids, P, P.light_buckets)
        prefix, _ = C.column_major_exclusive_scan(counts)
        src = S.RecordArray(keys.copy(), vals.copy())
        dst = S.RecordArray(np.full(total, 7, np.uint64), np.full(total, 9, np.uint64))
        C._distribute_ids(src, dst, base, ids, prefix, P, P.light_buckets)
        p = f"win_{name}_"
        out[p + "keys"], out[p + "vals"], out[p + "ids"] = keys, vals, ids
        out[p + "dst_keys"], out[p + "dst_vals"] = dst.keys.copy(), dst.values.copy()
        meta["window"].append({"name": name, "total": total, "base": base, "m": m, "params": kw})
    out["meta"] = np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8)
    np.savez_compressed(os.path.join(HERE, "golden_refine.npz"), **out)
    print("wrote", len(out), "arrays")


if __name__ == "__main__":
    main()
