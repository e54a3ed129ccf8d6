"""Golden fixtures for collect_reduce / histogram over 128-bit keys, made by
the UNMODIFIED reference.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden_u128_agg.py

Runs the reference's ``histogram`` and ``collect_reduce(summing64)`` with
``UInt128KeyAdapter`` (adapters.py:147-198; aggregate.py:267-299) on the
inputs of make_golden_u128.py and writes ``golden_u128_agg.npz``: the result
pairs (keys as (lo, hi) rows, aggregates) and the Telemetry counters.
Nothing at test time reads /root/reference.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
HERE = os.path.dirname(os.path.abspath(__file__))

import semisort as S  # noqa: E402
from make_golden_u128 import cases  # noqa: E402


def tel_dict(t):
    return {"max_depth": t.max_depth, "nodes": t.nodes, "scratch_moves": t.scratch_moves,
            "bucket_assignments": t.bucket_assignments,
            "matrix_cells_by_level": {str(k): v for k, v in sorted(t.matrix_cells_by_level.items())}}


def main():
    z: dict[str, np.ndarray] = {}
    meta = {}
    for name, keys, kw in cases():
        n = len(keys)
        vals = (np.arange(n, dtype=np.uint64) * 0x9E3779B97F4A7C15) if n else np.zeros(0, np.uint64)
        z[f"{name}_vals"] = vals
        for ident in (False, True):
            adp = S.UInt128KeyAdapter(identity=ident)
            for kind in ("count", "sum64"):
                tag = f"{name}_{kind}_{int(ident)}"
                tel = S.Telemetry()
                params = S.TuningParams.for_input(n, **kw)
                if kind == "count":
                    res = S.histogram(S.RecordArray(keys.copy()), adp, params, telemetry=tel)
                else:
                    res = S.collect_reduce(S.RecordArray(keys.copy(), vals.copy()), adp, S.ReduceSpec.summing64(),
                                           params, telemetry=tel)
                pairs = list(res)
                z[f"{tag}_k"] = np.array([k for k, _ in pairs], dtype=np.uint64).reshape(-1, 2)
                z[f"{tag}_a"] = np.array([a for _, a in pairs], dtype=np.uint64)
                meta[tag] = tel_dict(tel)
    z["tags"] = np.array(sorted(meta))
    z["meta"] = np.array(json.dumps(meta, sort_keys=True))
    np.savez_compressed(os.path.join(HERE, "golden_u128_agg.npz"), **z)
    print(len(meta), "aggregate cases")


if __name__ == "__main__":
    main()
