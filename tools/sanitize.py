"""Small end-to-end workload for compute-sanitizer (measurement / evidence).

    compute-sanitizer --tool {memcheck,racecheck,synccheck,initcheck} python tools/sanitize.py

Runs every kernel family of the hot path once on small inputs: c1-shaped
semisort (2^20 uniform, eq, both layouts), a Zipf semisort with heavy keys
(copy-back, mid leaves), lt mode, collect_reduce / histogram through both the
node-fold path and the level path (SS_NODE_FOLD=0 in a second process), the
packed partition, and the fallback kernels (SS_HW_RANK=0, SS_DIST_KERNEL=radix)
when SANITIZE_FALLBACKS=1.  Exits non-zero if any result disagrees with an
independent torch check, so a sanitizer run is also a correctness run.
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2304_10078_b200 as S  # noqa: E402
from paper_2304_10078_b200.validate import validate_semisort  # noqa: E402


def check_sort(before, after, adp, what):
    v = validate_semisort(before, after, adp)
    assert v.valid, f"{what}: invalid semisort"


def check_agg(keys, vals, res, count, what):
    k = torch.from_numpy(keys.astype(np.int64))
    uniq, inv = torch.unique(k, return_inverse=True)
    if count:
        agg = torch.bincount(inv, minlength=uniq.numel())
    else:
        agg = torch.zeros(uniq.numel(), dtype=torch.int64).index_add_(0, inv, torch.from_numpy(vals.view(np.int64)))
    rk, ra = res.to_numpy()
    order = np.argsort(rk.astype(np.int64))
    assert np.array_equal(rk.astype(np.int64)[order], uniq.numpy()), f"{what}: keys"
    assert np.array_equal(ra.view(np.int64)[order], agg.numpy()), f"{what}: aggregates"


def main():
    rng = np.random.default_rng(1)
    n = 1 << 20
    adp = S.UIntKeyAdapter()
    # c1: uniform keys over [0, 2^20), value = index
    keys = rng.integers(0, n, n).astype(np.uint64)
    vals = np.arange(n, dtype=np.uint64)
    for mode in ("eq", "lt"):
        d = S.RecordArray(keys, vals)
        before = d.copy()
        S.semisort(d, adp, mode)
        check_sort(before, d, adp, f"c1 {mode}")
    # Zipf with heavy keys (copy-back, warp / smem / mid leaves)
    z = (rng.zipf(1.2, n) % 100_000).astype(np.uint64)
    d = S.RecordArray(z, vals)
    before = d.copy()
    S.semisort(d, adp, "eq")
    check_sort(before, d, adp, "zipf eq")
    # u32 keys without values
    d = S.RecordArray(rng.integers(0, 5000, n).astype(np.uint32))
    before = d.copy()
    S.semisort(d, S.UIntKeyAdapter(identity=True), "eq")
    check_sort(before, d, S.UIntKeyAdapter(identity=True), "u32 identity")
    # aggregation: node folds (c4-like counts, c3-like sums) or the level path
    hk = rng.integers(0, 200_000, n).astype(np.uint32)
    check_agg(hk, None, S.histogram(S.RecordArray(hk), adp), True, "histogram")
    ck = np.floor(rng.exponential(2000.0, n)).astype(np.uint64)
    cv = rng.integers(0, 2**32, n).astype(np.uint64)
    check_agg(ck, cv, S.collect_reduce(S.RecordArray(ck, cv), adp, S.ReduceSpec.summing64()), False, "sum64")
    # packed partition (multi-GPU data path, one device)
    from paper_2304_10078_b200.distributed import device_pack_partition
    words, counts = device_pack_partition(S.RecordArray(keys, vals), 4)
    assert sum(counts) == n
    torch.cuda.synchronize()
    print("sanitize workload ok", {k: os.environ.get(k) for k in ("SS_NODE_FOLD", "SS_HW_RANK", "SS_DIST_KERNEL")})


if __name__ == "__main__":
    main()
