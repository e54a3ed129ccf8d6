"""Generate golden fixtures by running the UNMODIFIED reference package.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports ``semisort`` from /root/reference/pkg/src (no bytecode written),
runs its public and phase-level functions on seeded inputs and writes:

* ``golden_small.npz``   — full input/output arrays for small cases;
* ``golden_digests.json`` — SHA-256 digests (+ telemetry) for cases whose
  inputs are regenerated on the GPU box by ``oracle.datagen`` (the input
  digest is stored too, so a generator drift is detected).

Nothing at test time reads /root/reference; tests read only these files.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

sys.dont_write_bytecode = True
REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)

import semisort as S  # noqa: E402
from semisort import core as C  # noqa: E402
from semisort.hashing import mix64, mix64_pair  # noqa: E402

ADP = S.UIntKeyAdapter()
IDA = S.UIntKeyAdapter(identity=True)


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def tel_dict(t: C.Telemetry) -> dict:
    return {"max_depth": t.max_depth, "nodes": t.nodes,
            "scratch_allocations": t.scratch_allocations,
            "scratch_moves": t.scratch_moves,
            "bucket_assignments": t.bucket_assignments,
            "matrix_cells_by_level": {str(k): v for k, v in t.matrix_cells_by_level.items()}}


def rp(n, **kw):
    """The reference tests' recursive_params (test_semisort.py:34-40)."""
    kw.setdefault("light_buckets", 4)
    kw.setdefault("subarray_len", 8)
    kw.setdefault("base_case_cutoff", 8)
    kw.setdefault("max_heavy", 2)
    return kw


def main():
    small: dict[str, np.ndarray] = {}
    meta: dict = {"cases": {}}

    # ---- mix64 known answers (hashing.py:25-47) ---------------------------
    rng = np.random.default_rng(100)
    xs = np.concatenate([np.array([0, 1, 13, 2**64 - 1, 0x0123456789ABCDEF, 2**63],
                                  dtype=np.uint64),
                         rng.integers(0, 2**64 - 1, 250, dtype=np.uint64, endpoint=True)])
    small["kat_x"] = xs
    small["kat_mix64"] = np.array([mix64(int(x)) for x in xs], dtype=np.uint64)
    small["kat_pair_b"] = xs[::-1].copy()
    small["kat_pair"] = np.array([mix64_pair(int(a), int(b)) for a, b in zip(xs, xs[::-1])],
                                 dtype=np.uint64)

    # ---- sampling / heavy tables (core.py:221-260) -------------------------
    samp_cases = []
    r = np.random.default_rng(7)
    heavy_tail = np.minimum((1.0 / r.random(50000)) ** 2.0, 10**6).astype(np.uint64)
    samp_cases.append(("tail", heavy_tail, dict(), 12345))
    samp_cases.append(("cap", np.repeat(np.arange(8, dtype=np.uint64), 512), dict(max_heavy=3), 1))
    samp_cases.append(("ten", r.integers(0, 10, 10**5).astype(np.uint64), dict(), 11))
    samp_cases.append(("tiny", r.integers(0, 8, 64).astype(np.uint64), dict(), 5))
    samp_cases.append(("lowthr", r.integers(0, 40, 3).astype(np.uint64), dict(), 99))
    samp_cases.append(("one", np.full(20000, 42, dtype=np.uint64), dict(), 7))
    samp_cases.append(("wide", r.integers(0, 2**64 - 1, 30000, dtype=np.uint64, endpoint=True),
                       dict(), mix64_pair(1, 0)))
    samp_cases.append(("mh0", np.zeros(5000, dtype=np.uint64), dict(max_heavy=0), 1))
    samp_cases.append(("manyheavy", np.repeat(r.integers(0, 2**40, 700).astype(np.uint64), 40),
                       dict(sample_factor=4000), 3))
    # a window of a larger array sampled at the *window* size (core.py:233-239)
    samp_cases.append(("sf", np.tile(np.arange(30, dtype=np.uint64), 900), dict(sample_factor=50), 77))
    meta["sampling"] = []
    for name, keys, kw, key in samp_cases:
        n = len(keys)
        params = S.TuningParams.for_input(n, **kw)
        data = S.RecordArray(keys)
        table = S.sample_and_bucket(data, ADP, params, 0,
                                    np.random.Generator(np.random.Philox(key=key)))
        small[f"samp_{name}_keys"] = keys
        small[f"samp_{name}_heavy"] = np.asarray(table.keys, dtype=np.uint64)
        meta["sampling"].append({"name": name, "params": kw, "rng_key": key})

    # ---- bucket ids (core.py:139-213) --------------------------------------
    meta["ids"] = []
    idk = r.integers(0, 2**64 - 1, 4000, dtype=np.uint64, endpoint=True)
    idk[::7] = idk[3]      # a heavy key
    idk[::11] = idk[5]     # another
    small["ids_keys"] = idk
    for nl in (1024, 8, 1, 2):
        for depth in (0, 1, 5, 6, 7, 13, 31, 32, 64):
            for ident in (False, True):
                params = S.TuningParams.for_input(len(idk), light_buckets=nl)
                adp = IDA if ident else ADP
                table = C.HeavyTable(nl)
                for k in (int(idk[3]), int(idk[5])):
                    table.insert(k, adp.hash_scalar(k))
                table.finalize(adp)
                ids = C.assign_bucket_ids(S.RecordArray(idk), table, adp, params, depth)
                tag = f"ids_{nl}_{depth}_{int(ident)}"
                small[tag] = ids.astype(np.int32)
                meta["ids"].append({"tag": tag, "n_light": nl, "depth": depth,
                                    "identity": ident, "heavy": [int(idk[3]), int(idk[5])]})

    # ---- counts / scan / distribute (core.py:268-380) ----------------------
    meta["distribute"] = []
    dcases = [("hand", np.array([1, 0, 1, 1, 0, 0, 1, 0], np.int32), 4, 2)]
    for i, (n, nb, sl) in enumerate([(1, 1, 1), (60, 6, 9), (1000, 37, 64), (5000, 1100, 1024),
                                     (777, 3, 5), (4096, 1524, 4096)]):
        dcases.append((f"r{i}", r.integers(0, nb, n).astype(np.int32), sl, nb))
    for name, ids, sl, nb in dcases:
        n = len(ids)
        params = S.TuningParams.for_input(n, light_buckets=1, subarray_len=sl)
        counts = C._counts_from_ids(ids, params, nb)
        prefix, offsets = C.column_major_exclusive_scan(counts)
        src = S.RecordArray(np.arange(n, dtype=np.uint64), np.arange(n, dtype=np.uint64) * 3)
        dst = src.empty_like()
        C._distribute_ids(src, dst, 0, ids, prefix, params, nb)
        small[f"dist_{name}_ids"] = ids
        small[f"dist_{name}_counts"] = counts
        small[f"dist_{name}_prefix"] = prefix
        small[f"dist_{name}_offsets"] = offsets
        small[f"dist_{name}_out"] = dst.keys.copy()
        meta["distribute"].append({"name": name, "sub_len": sl, "n_buckets": nb})

    # ---- base cases (core.py:388-429) --------------------------------------
    meta["base"] = []
    bcases = [("empty", np.zeros(0, np.uint64)), ("one", np.array([9], np.uint64)),
              ("same", np.array([5, 5, 5], np.uint64)), ("two", np.array([2, 1, 2], np.uint64))]
    for i, (m, u) in enumerate([(120, 13), (1000, 40), (1023, 2**64 - 1), (2048, 300),
                                (5000, 5000), (16383, 2**20), (4097, 7), (600, 600)]):
        bcases.append((f"r{i}", r.integers(0, u, m, dtype=np.uint64, endpoint=True)))
    for name, keys in bcases:
        for ident in (False, True):
            for mode in ("eq", "lt"):
                data = S.RecordArray(keys.copy(), np.arange(len(keys), dtype=np.uint64))
                adp = IDA if ident else ADP
                (C.base_case_eq if mode == "eq" else C.base_case_lt)(data, adp)
                small[f"base_{name}_{mode}_{int(ident)}"] = data.values.copy()
        small[f"base_{name}_keys"] = keys
        meta["base"].append(name)

    # ---- end-to-end semisort, small (full arrays) ---------------------------
    meta["semisort_small"] = []
    ss_cases = []
    for i in range(12):
        m = int(r.integers(0, 300))
        ss_cases.append((f"rec{i}", r.integers(0, 10, m).astype(np.uint64), rp(m), "eq", False))
    for i in range(6):
        m = int(r.integers(1, 200))
        ss_cases.append((f"wide{i}", r.integers(0, 2**64 - 1, m, dtype=np.uint64, endpoint=True),
                         rp(m), "eq", False))
    for i in range(6):
        m = int(r.integers(1, 300))
        ss_cases.append((f"lt{i}", r.integers(0, 10, m).astype(np.uint64), rp(m), "lt", False))
    ss_cases.append(("id40k", r.integers(0, 3000, 40000).astype(np.uint64),
                     dict(base_case_cutoff=512), "eq", True))
    ss_cases.append(("u32", r.integers(0, 200, 20000).astype(np.uint32),
                     dict(base_case_cutoff=256), "eq", False))
    ss_cases.append(("heavyish", np.minimum((1.0 / r.random(30000)) ** 1.5, 10**6).astype(np.uint64),
                     dict(base_case_cutoff=256, light_buckets=16, subarray_len=64), "eq", False))
    ss_cases.append(("allsame", np.zeros(20000, np.uint64), dict(), "eq", False))
    ss_cases.append(("seed7", r.integers(0, 5000, 30000).astype(np.uint64),
                     dict(base_case_cutoff=1024, seed=7), "eq", False))
    ss_cases.append(("lt20k", r.integers(0, 2**40, 20000).astype(np.uint64),
                     dict(base_case_cutoff=300), "lt", False))
    # identity hash with all-zero low bits: forces the safety valve (core.py:452-460)
    ss_cases.append(("valve", (r.integers(0, 4000, 6000).astype(np.uint64) << np.uint64(40)),
                     dict(light_buckets=8, subarray_len=32, base_case_cutoff=64, max_heavy=0),
                     "eq", True))
    for name, keys, kw, mode, ident in ss_cases:
        n = len(keys)
        vdt = np.uint32 if keys.dtype == np.uint32 else np.uint64
        data = S.RecordArray(keys.copy(), np.arange(n, dtype=vdt))
        tel = C.Telemetry()
        S.semisort(data, IDA if ident else ADP, mode, S.TuningParams.for_input(n, **kw),
                   telemetry=tel)
        small[f"ss_{name}_keys"] = keys
        small[f"ss_{name}_out"] = data.values.copy()
        meta["semisort_small"].append({"name": name, "params": kw, "mode": mode,
                                       "identity": ident, "telemetry": tel_dict(tel)})

    # ---- end-to-end semisort, digests (inputs regenerated on the box) -------
    meta["semisort_digest"] = []
    big = [
        ("c1", ("uniform", 2**20, 2**20, 64), dict(), "eq", False),
        ("c1_deep", ("uniform", 2**20, 2**20, 64), dict(base_case_cutoff=1024), "eq", False),
        ("zipf12", ("zipfian", 1.2, 2**18, 64), dict(base_case_cutoff=1024), "eq", False),
        ("zipf12_hashed", ("zipfian", 1.2, 2**18, 64), dict(base_case_cutoff=2048), "eq", False),
        ("exp", ("exponential", 1e-3, 300000, 64), dict(base_case_cutoff=700), "eq", False),
        ("u32_uniform", ("uniform", 10**5, 250000, 32), dict(base_case_cutoff=900), "eq", False),
        ("ident", ("uniform", 10**4, 200000, 64), dict(base_case_cutoff=600), "eq", True),
        ("lt_uniform", ("uniform", 10**6, 100000, 64), dict(base_case_cutoff=2000), "lt", False),
    ]
    for name, (fam, par, n, kw_bits), kw, mode, ident in big:
        g = S.generate(S.DistributionSpec(fam, par, n, kw_bits, seed=1))
        keys = g.keys.copy()
        if name == "zipf12_hashed":
            keys = S.hashing.mix64_array(keys - np.uint64(1))
        vdt = keys.dtype
        data = S.RecordArray(keys.copy(), np.arange(n, dtype=vdt))
        tel = C.Telemetry()
        S.semisort(data, IDA if ident else ADP, mode, S.TuningParams.for_input(n, **kw),
                   telemetry=tel)
        meta["semisort_digest"].append({
            "name": name, "gen": [fam, par, n, kw_bits], "params": kw, "mode": mode,
            "identity": ident, "hash_ranks": name == "zipf12_hashed",
            "input_sha": sha(g.keys, g.values), "out_sha": sha(data.keys, data.values),
            "telemetry": tel_dict(tel)})

    # ---- collect-reduce / histogram (aggregate.py) --------------------------
    meta["aggregate"] = []
    ag_cases = []
    for i in range(8):
        m = int(r.integers(0, 200))
        ag_cases.append((f"rec{i}", r.integers(0, 12, m).astype(np.uint64),
                         r.integers(0, 2**64 - 1, m, dtype=np.uint64, endpoint=True), rp(m), False))
    ag_cases.append(("wrap", r.integers(0, 30, 5000).astype(np.uint64),
                     r.integers(0, 2**63, 5000).astype(np.uint64) * np.uint64(2),
                     rp(5000, base_case_cutoff=256), False))
    ag_cases.append(("zeros", np.zeros(20000, np.uint64), np.arange(20000, dtype=np.uint64),
                     dict(), False))
    ag_cases.append(("tail", np.minimum((1.0 / r.random(60000)) ** 1.5, 10**9).astype(np.uint64),
                     r.integers(0, 2**32, 60000).astype(np.uint64), dict(base_case_cutoff=512), False))
    ag_cases.append(("wide", r.integers(0, 2**62, 50000).astype(np.uint64),
                     r.integers(0, 2**32, 50000).astype(np.uint64), dict(), False))
    ag_cases.append(("ident", r.integers(0, 4000, 50000).astype(np.uint64),
                     r.integers(0, 2**32, 50000).astype(np.uint64), dict(base_case_cutoff=512), True))
    ag_cases.append(("u32", r.integers(0, 3000, 30000).astype(np.uint32),
                     r.integers(0, 2**32, 30000).astype(np.uint32), dict(base_case_cutoff=256), False))
    for name, keys, vals, kw, ident in ag_cases:
        n = len(keys)
        params = S.TuningParams.for_input(n, **kw)
        adp = IDA if ident else ADP
        data = S.RecordArray(keys.copy(), vals.copy())
        t1, t2 = C.Telemetry(), C.Telemetry()
        hist = S.histogram(data, adp, params, telemetry=t1)
        summ = S.collect_reduce(data, adp, S.ReduceSpec.summing64(), params, telemetry=t2)
        small[f"ag_{name}_keys"] = keys
        small[f"ag_{name}_vals"] = vals
        small[f"ag_{name}_hist"] = np.array(hist.pairs, dtype=np.uint64).reshape(-1, 2)
        small[f"ag_{name}_sum"] = np.array(summ.pairs, dtype=np.uint64).reshape(-1, 2)
        meta["aggregate"].append({"name": name, "params": kw, "identity": ident,
                                  "tel_hist": tel_dict(t1), "tel_sum": tel_dict(t2)})

    meta["aggregate_digest"] = []
    for name, (fam, par, n, bits), kw, kind in [
        ("exp_sum", ("exponential", 1e-4, 300000, 64), dict(base_case_cutoff=2048), "sum64"),
        ("u32_hist", ("uniform", 10**5, 400000, 32), dict(base_case_cutoff=1024), "count"),
        ("zipf_hist", ("zipfian", 1.2, 300000, 64), dict(), "count"),
    ]:
        g = S.generate(S.DistributionSpec(fam, par, n, bits, seed=1))
        vals = g.values >> (np.uint64(32) if bits == 64 else np.uint32(0))
        params = S.TuningParams.for_input(n, **kw)
        data = S.RecordArray(g.keys.copy(), vals.copy())
        tel = C.Telemetry()
        spec = S.ReduceSpec.counting() if kind == "count" else S.ReduceSpec.summing64()
        res = S.collect_reduce(data, ADP, spec, params, telemetry=tel)
        pairs = np.array(res.pairs, dtype=np.uint64).reshape(-1, 2)
        srt = pairs[np.argsort(pairs[:, 0], kind="stable")]
        meta["aggregate_digest"].append({
            "name": name, "gen": [fam, par, n, bits], "params": kw, "kind": kind,
            "input_sha": sha(g.keys, g.values), "pairs_sha": sha(pairs),
            "sorted_pairs_sha": sha(srt), "n_pairs": len(pairs), "telemetry": tel_dict(tel)})

    np.savez_compressed(os.path.join(HERE, "golden_small.npz"), **small)
    with open(os.path.join(HERE, "golden_digests.json"), "w") as fh:
        json.dump(meta, fh, indent=1, sort_keys=True)
    print("wrote", len(small), "arrays")


if __name__ == "__main__":
    main()
