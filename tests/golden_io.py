"""Loading helpers for the committed reference fixtures (tests/golden)."""
import hashlib
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def small():
    return np.load(os.path.join(GOLDEN, "golden_small.npz"))


def meta():
    with open(os.path.join(GOLDEN, "golden_digests.json")) as fh:
        return json.load(fh)


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def rp(n, **kw):
    kw.setdefault("light_buckets", 4)
    kw.setdefault("subarray_len", 8)
    kw.setdefault("base_case_cutoff", 8)
    kw.setdefault("max_heavy", 2)
    return kw
