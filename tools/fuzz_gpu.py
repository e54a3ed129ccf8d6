"""Differential fuzz of the GPU path against the oracle (measurement / QA
helper, run on a GPU box): random sizes, bucket counts (odd totals
included), heavy caps, cut-offs, key widths and key distributions;
semisort compared byte for byte with every Telemetry counter, collect_reduce /
histogram per key.

    python tools/fuzz_gpu.py [cases] [seed]
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402
import paper_2304_10078_b200 as S  # noqa: E402

cases = int(sys.argv[1]) if len(sys.argv) > 1 else 40
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 7)
bad = 0
for c in range(cases):
    n = int(rng.integers(1 << 15, 1 << 20))
    kdt = rng.choice([np.uint32, np.uint64])
    lb = int(rng.choice([16, 64, 256, 1024, 4096]))
    mh = int(rng.choice([0, 1, 7, 37, 100, 500]))
    alpha = int(rng.choice([256, 1024, 4096, 16384]))
    kind = rng.choice(["uniform_small", "uniform_wide", "zipf", "few", "runs"])
    if kind == "uniform_small":
        keys = rng.integers(0, max(2, n // 8), n)
    elif kind == "uniform_wide":
        keys = rng.integers(0, 1 << 31, n)
    elif kind == "zipf":
        keys = np.minimum(rng.zipf(1.2, n), 1 << 30)
    elif kind == "few":
        keys = rng.integers(0, 5, n)
    else:
        keys = np.repeat(rng.integers(0, 1 << 20, n // 64 + 1), 64)[:n]
    keys = keys.astype(kdt)
    vals = np.arange(n, dtype=np.uint64)
    ident = bool(rng.integers(0, 4) == 0)
    kw = {"light_buckets": lb, "base_case_cutoff": alpha, "max_heavy": mh, "seed": int(rng.integers(1, 1 << 30))}
    tag = f"case {c}: n={n} {np.dtype(kdt).name} lb={lb} mh={mh} alpha={alpha} {kind} identity={ident}"
    try:
        op = O.OracleParams.derive(n, **kw)
        ko, vo, tel_o = O.semisort(keys, vals, op, identity=ident)
        data = S.RecordArray(keys, vals)
        tel = S.Telemetry()
        adp = S.UIntKeyAdapter(identity=True) if ident else S.UIntKeyAdapter()
        S.semisort(data, adp, "eq", S.TuningParams.for_input(n, **kw), telemetry=tel)
        ok = np.array_equal(data.keys_host(), ko) and np.array_equal(data.values_host(), vo)
        ok = ok and tel.nodes == tel_o.nodes and tel.max_depth == tel_o.max_depth and \
            tel.bucket_assignments == tel_o.bucket_assignments
        v2 = rng.integers(0, 1 << 62, n).astype(np.uint64)
        res = S.collect_reduce(S.RecordArray(keys, v2), S.UIntKeyAdapter(), S.ReduceSpec.summing64(),
                               S.TuningParams.for_input(n, **kw))
        k, a = res.to_numpy()
        ok2 = dict(zip(k.tolist(), a.tolist())) == O.reduce_by_key(keys, v2, "sum64")
        print(("ok  " if ok and ok2 else "FAIL") + " " + tag + ("" if ok and ok2 else f" semisort={ok} reduce={ok2}"), flush=True)
        bad += 0 if ok and ok2 else 1
    except Exception as e:  # noqa: BLE001
        print("ERR  " + tag + f": {type(e).__name__}: {e}", flush=True)
        bad += 1
print("failures:", bad)
sys.exit(1 if bad else 0)
