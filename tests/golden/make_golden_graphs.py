"""Golden fixtures for graph transpose / CSR build from the UNMODIFIED reference.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden_graphs.py

Writes ``golden_graphs.npz``: for every case the input edges or CSR and the
reference ``from_edges`` / ``transpose`` outputs (graphs.py:59-105).  The
cases follow the reference's own tests (test_graphs.py: two-cycle, star,
random canonical graphs, non-canonical input, empty graph, multi-edges)
plus larger skewed graphs.  Nothing at test time reads /root/reference.
"""

from __future__ import annotations

import os
import sys

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
HERE = os.path.dirname(os.path.abspath(__file__))

from semisort.graphs import from_edges, transpose  # noqa: E402


def canonical(rng, n, m):
    src = rng.integers(0, n, m)
    dst = rng.integers(0, n, m)
    order = np.lexsort((dst, src))
    return src[order], dst[order]


def main():
    out = {}
    cases = []

    def add(name, n, src, dst):
        src = np.asarray(src, dtype=np.uint32)
        dst = np.asarray(dst, dtype=np.uint32)
        g = from_edges(n, src, dst)
        t = transpose(g)
        out[f"{name}_n"] = np.array([n], dtype=np.uint64)
        out[f"{name}_src"] = src
        out[f"{name}_dst"] = dst
        out[f"{name}_off"] = g.offsets
        out[f"{name}_tgt"] = g.targets
        out[f"{name}_toff"] = t.offsets
        out[f"{name}_ttgt"] = t.targets
        cases.append(name)

    add("two_cycle", 2, [0, 1], [1, 0])
    add("star", 10, [0] * 9, list(range(1, 10)))
    add("empty", 4, [], [])
    add("multi", 3, [0, 0, 1], [1, 1, 1])
    add("self_loops", 5, [0, 1, 1, 4, 4, 4], [0, 1, 3, 4, 4, 0])
    rng = np.random.default_rng(21)
    add("random_1e3", *(lambda s, d: (1000, s, d))(*canonical(rng, 1000, 10**4)))
    rng = np.random.default_rng(22)
    for i in range(5):
        add(f"canon_{i}", *(lambda s, d: (200, s, d))(*canonical(rng, 200, 3000)))
    rng = np.random.default_rng(23)
    add("arbitrary", 100, rng.integers(0, 100, 2000), rng.integers(0, 100, 2000))   # input order kept
    rng = np.random.default_rng(24)
    add("degrees", *(lambda s, d: (500, s, d))(*canonical(rng, 500, 8000)))
    # skewed (Zipf-like) in- and out-degrees, large enough for several semisort levels
    rng = np.random.default_rng(25)
    n = 1 << 16
    m = 1 << 20
    src = np.minimum(rng.zipf(1.4, m) - 1, n - 1)
    dst = np.minimum(rng.zipf(1.2, m) - 1, n - 1)
    add("zipf_64k_1m", n, *canonical_sorted(src, dst))
    rng = np.random.default_rng(26)
    add("isolated_tail", 5000, rng.integers(0, 100, 20000), rng.integers(0, 100, 20000))
    out["cases"] = np.array(cases)
    np.savez_compressed(os.path.join(HERE, "golden_graphs.npz"), **out)
    print(len(cases), "graph cases")


def canonical_sorted(src, dst):
    order = np.lexsort((dst, src))
    return src[order], dst[order]


if __name__ == "__main__":
    main()
