"""CUDA path vs the reference fixtures and the oracle (GPU tier).

Every case compares bytes: the GPU replays numpy's Philox sample stream and
the reference's bucket / scan / distribute / chained-hash definitions, so
semisort output must equal the reference output for the same params.
"""
import numpy as np
import pytest
import torch

import oracle as O
from golden_io import meta, sha, small
from oracle.datagen import gen_keys_values

pytestmark = pytest.mark.gpu

G = small()
M = meta()


@pytest.fixture(scope="module")
def S():
    import paper_2304_10078_b200 as S
    assert torch.cuda.is_available()
    return S


def tel_eq(tel, ref):
    assert tel.max_depth == ref["max_depth"]
    assert tel.nodes == ref["nodes"]
    assert tel.scratch_moves == ref["scratch_moves"]
    assert tel.bucket_assignments == ref["bucket_assignments"]
    assert tel.scratch_allocations == ref.get("scratch_allocations", tel.scratch_allocations)
    assert {str(k): v for k, v in tel.matrix_cells_by_level.items()} == ref["matrix_cells_by_level"]


# ---- phases ---------------------------------------------------------------

@pytest.mark.parametrize("case", M["ids"], ids=lambda c: c["tag"])
def test_bucket_ids(S, case):
    keys = G["ids_keys"]
    P = S.TuningParams.for_input(len(keys), light_buckets=case["n_light"])
    adp = S.UIntKeyAdapter(identity=case["identity"])
    table = S.HeavyTable(case["n_light"])
    for k in case["heavy"]:
        table.insert(k, adp.hash_scalar(k))
    ids = S.assign_bucket_ids(S.RecordArray(keys), table, adp, P, case["depth"])
    assert np.array_equal(ids.cpu().numpy(), G[case["tag"]])


def test_get_bucket_id_scalar(S):
    P = S.TuningParams.for_input(16, light_buckets=4, subarray_len=4)
    adp = S.UIntKeyAdapter(identity=True)
    empty = S.HeavyTable(4)
    assert S.get_bucket_id(13, empty, adp, P, depth=0) == 1      # test_core_ops.py:51-54
    assert S.get_bucket_id(13, empty, adp, P, depth=1) == 3      # test_core_ops.py:57-61
    t = S.HeavyTable(4)
    t.insert(13, 13)
    t.insert(7, 7)
    assert S.get_bucket_id(13, t, adp, P) == 4 and S.get_bucket_id(7, t, adp, P) == 5
    assert S.get_bucket_id(99, t, adp, P) == 99 % 4


@pytest.mark.parametrize("case", M["sampling"], ids=lambda c: c["name"])
def test_sampling(S, case):
    keys = G[f"samp_{case['name']}_keys"]
    P = S.TuningParams.for_input(len(keys), **case["params"])
    rng = np.random.Generator(np.random.Philox(key=case["rng_key"]))
    table = S.sample_and_bucket(S.RecordArray(keys), S.UIntKeyAdapter(), P, 0, rng)
    assert table.keys == G[f"samp_{case['name']}_heavy"].tolist()


@pytest.mark.parametrize("case", M["distribute"], ids=lambda c: c["name"])
def test_counts_scan_distribute(S, case):
    p = f"dist_{case['name']}_"
    ids = G[p + "ids"]
    n = len(ids)
    P = S.TuningParams.for_input(n, light_buckets=1, subarray_len=case["sub_len"])
    C = S.core.counts_from_ids(ids, P, case["n_buckets"])
    assert np.array_equal(C.cpu().numpy(), G[p + "counts"])
    X, off = S.column_major_exclusive_scan(C)
    assert np.array_equal(X.cpu().numpy(), G[p + "prefix"])
    assert np.array_equal(off.cpu().numpy(), G[p + "offsets"])
    src = S.RecordArray(np.arange(n, dtype=np.uint64), np.arange(n, dtype=np.uint64) * 3)
    dst = src.empty_like()
    S.core.distribute_ids(src, dst, 0, torch.from_numpy(ids).cuda(), X, P, case["n_buckets"])
    assert np.array_equal(dst.keys_host(), G[p + "out"])
    assert np.array_equal(dst.values_host(), G[p + "out"] * 3)


def test_scan_hand_examples(S):
    X, off = S.column_major_exclusive_scan(np.array([[1, 3], [3, 1]]))
    assert X.cpu().tolist() == [[0, 4], [1, 7]] and off.cpu().tolist() == [0, 4, 8]
    X, off = S.column_major_exclusive_scan(np.array([[17]]))
    assert X.cpu().tolist() == [[0]] and off.cpu().tolist() == [0, 17]


def test_count_into_matrix_from_keys(S):
    rng = np.random.default_rng(3)
    keys = rng.integers(0, 2**60, 5000).astype(np.uint64)
    P = S.TuningParams.for_input(5000, light_buckets=16, subarray_len=64)
    OP = O.OracleParams.derive(5000, light_buckets=16, subarray_len=64)
    heavy = O.sample_heavy(keys, OP, 2)
    t = S.HeavyTable(16)
    for k in heavy:
        t.insert(k, 0)
    got = S.count_into_matrix(S.RecordArray(keys), t, S.UIntKeyAdapter(), P, 3).cpu().numpy()
    ids = O.bucket_ids(keys, heavy, OP, 3, False)
    assert np.array_equal(got, O.count_rows(ids, 64, 16 + len(heavy)))


@pytest.mark.parametrize("name", M["base"])
@pytest.mark.parametrize("ident", [0, 1])
@pytest.mark.parametrize("mode", ["eq", "lt"])
def test_base_cases(S, name, ident, mode):
    keys = G[f"base_{name}_keys"]
    data = S.RecordArray(keys, np.arange(len(keys), dtype=np.uint64))
    adp = S.UIntKeyAdapter(identity=bool(ident))
    (S.base_case_eq if mode == "eq" else S.base_case_lt)(data, adp)
    exp = G[f"base_{name}_{mode}_{ident}"]
    assert np.array_equal(data.values_host(), exp)
    assert np.array_equal(data.keys_host(), keys[exp.astype(np.int64)])


# ---- whole semisort ---------------------------------------------------------

@pytest.mark.parametrize("case", M["semisort_small"], ids=lambda c: c["name"])
def test_semisort_small(S, case):
    keys = G[f"ss_{case['name']}_keys"]
    n = len(keys)
    data = S.RecordArray(keys, np.arange(n, dtype=keys.dtype))
    tel = S.Telemetry()
    S.semisort(data, S.UIntKeyAdapter(identity=case["identity"]), case["mode"],
               S.TuningParams.for_input(n, **case["params"]), telemetry=tel)
    assert np.array_equal(data.values_host(), G[f"ss_{case['name']}_out"])
    tel_eq(tel, case["telemetry"])


@pytest.mark.parametrize("case", M["semisort_digest"], ids=lambda c: c["name"])
def test_semisort_digest(S, case):
    fam, par, n, bits = case["gen"]
    keys, vals = gen_keys_values(fam, par, n, bits, seed=1)
    assert sha(keys, vals) == case["input_sha"]
    if case["hash_ranks"]:
        keys = O.mix64_np(keys - np.uint64(1))
    data = S.RecordArray(keys, np.arange(n, dtype=keys.dtype))
    tel = S.Telemetry()
    S.semisort(data, S.UIntKeyAdapter(identity=case["identity"]), case["mode"],
               S.TuningParams.for_input(n, **case["params"]), telemetry=tel)
    assert sha(data.keys_host(), data.values_host()) == case["out_sha"]
    tel_eq(tel, case["telemetry"])


@pytest.mark.parametrize("dist", ["uniform", "zipf", "few", "wide"])
def test_semisort_vs_oracle_4m(S, dist):
    rng = np.random.default_rng(42)
    n = 1 << 22
    if dist == "uniform":
        keys = rng.integers(0, 1 << 22, n).astype(np.uint64)
    elif dist == "zipf":
        keys = O.mix64_np(np.minimum(rng.zipf(1.3, n), 10**7).astype(np.uint64))
    elif dist == "few":
        keys = rng.integers(0, 300, n).astype(np.uint64)
    else:
        keys = rng.integers(0, 2**64 - 1, n, dtype=np.uint64, endpoint=True)
    vals = np.arange(n, dtype=np.uint64)
    P = O.OracleParams.derive(n)
    ko, vo, tel_o = O.semisort(keys, vals, P)
    data = S.RecordArray(keys, vals)
    tel = S.Telemetry()
    S.semisort(data, S.UIntKeyAdapter(), "eq", S.TuningParams.for_input(n), telemetry=tel)
    assert np.array_equal(data.values_host(), vo)
    assert np.array_equal(data.keys_host(), ko)
    assert tel.max_depth == tel_o.max_depth and tel.nodes == tel_o.nodes
    assert S.validate_semisort(S.RecordArray(keys, vals), data).valid


def test_semisort_value_layouts(S):
    rng = np.random.default_rng(5)
    n = 300000
    for kdt in (np.uint32, np.uint64):
        keys = rng.integers(0, 5000, n).astype(kdt)
        P = O.OracleParams.derive(n, base_case_cutoff=2048)
        _, vo, _ = O.semisort(keys, np.arange(n, dtype=np.uint64), P)
        for vals in (None, np.arange(n, dtype=np.uint32), np.arange(n, dtype=np.uint64),
                     np.stack([np.arange(n), np.arange(n) * 7], axis=1).astype(np.uint64)):
            d = S.RecordArray(keys, vals)
            S.semisort(d, S.UIntKeyAdapter(), "eq", S.TuningParams.for_input(n, base_case_cutoff=2048))
            assert np.array_equal(d.keys_host(), keys[vo.astype(np.int64)])
            if vals is not None:
                v = d.values_host()
                v0 = v[:, 0] if v.ndim == 2 else v
                assert np.array_equal(v0.astype(np.int64), vo.astype(np.int64))


def test_semisort_errors(S):
    d = S.RecordArray(np.array([1, 2], dtype=np.uint64), np.arange(2, dtype=np.uint64))
    with pytest.raises(S.ConfigurationError):
        S.semisort(d, S.UIntKeyAdapter(), "wrong")
    with pytest.raises(S.ContractError):
        S.semisort(d, S.UIntKeyAdapter(with_lt=False), "lt")
    with pytest.raises(S.ConfigurationError):
        S.semisort(d, S.UIntKeyAdapter(), "eq", S.TuningParams.for_input(7))

    class Custom(S.UIntKeyAdapter):
        def hash_scalar(self, key):
            return 0
    with pytest.raises(S.ContractError):
        S.semisort(d, Custom())


def test_all_heavy_and_tiny(S):
    d = S.RecordArray(np.zeros(10**5, dtype=np.uint64), np.arange(10**5, dtype=np.uint64))
    tel = S.Telemetry()
    S.semisort(d, S.UIntKeyAdapter(), telemetry=tel)
    assert tel.max_depth == 1 and tel.nodes == 1     # test_semisort.py:190-194
    assert np.array_equal(d.values_host(), np.arange(10**5))
    e = S.RecordArray(np.zeros(0, dtype=np.uint64), np.zeros(0, dtype=np.uint64))
    tel = S.Telemetry()
    S.semisort(e, S.UIntKeyAdapter(), telemetry=tel)
    assert tel.scratch_allocations == 1 and len(e) == 0


def test_local_refine(S):
    rng = np.random.default_rng(17)
    n = 4096
    keys = rng.integers(0, 1500, n).astype(np.uint64)
    adp = S.UIntKeyAdapter()
    P = S.TuningParams.for_input(n, light_buckets=8, subarray_len=64, base_case_cutoff=128, max_heavy=4)
    data = S.RecordArray(keys, np.arange(n, dtype=np.uint64))
    heavy = S.sample_and_bucket(data, adp, P, 0, np.random.Generator(np.random.Philox(key=5)))
    ids = S.assign_bucket_ids(data, heavy, adp, P, 0)
    nb = 8 + len(heavy)
    counts = S.core.counts_from_ids(ids, P, nb)
    prefix, offsets = S.column_major_exclusive_scan(counts)
    scratch = data.empty_like()
    S.core.distribute_ids(data, scratch, 0, ids, prefix, P, nb)
    buffers = S.WorkBuffers(primary=data, scratch=scratch, live_in_primary=False)
    S.local_refine(buffers, S.BucketPlan(heavy, counts, prefix, offsets), adp, "eq", P, depth=0)
    rep = S.validate_semisort(S.RecordArray(keys, np.arange(n, dtype=np.uint64)), data)
    assert rep.valid, rep


# ---- aggregates -----------------------------------------------------------------

def _sorted_pairs(res):
    k, v = res.to_numpy()
    o = np.argsort(k.astype(np.uint64), kind="stable")
    return np.stack([k.astype(np.uint64)[o], v.astype(np.uint64)[o]], axis=1) if len(k) else \
        np.zeros((0, 2), np.uint64)


@pytest.mark.parametrize("case", M["aggregate"], ids=lambda c: c["name"])
def test_aggregate_small(S, case):
    p = f"ag_{case['name']}_"
    keys, vals = G[p + "keys"], G[p + "vals"]
    P = S.TuningParams.for_input(len(keys), **case["params"])
    adp = S.UIntKeyAdapter(identity=case["identity"])
    data = S.RecordArray(keys, vals)
    before = (data.keys_host().copy(), data.values_host().copy())
    th, ts = S.Telemetry(), S.Telemetry()
    hist = S.histogram(data, adp, P, telemetry=th)
    summ = S.collect_reduce(data, adp, S.ReduceSpec.summing64(), P, telemetry=ts)
    for res, tag in ((hist, "hist"), (summ, "sum")):
        ref = G[p + tag]
        exp = ref[np.argsort(ref[:, 0], kind="stable")] if len(ref) else ref.reshape(0, 2)
        assert np.array_equal(_sorted_pairs(res), exp)
    tel_eq(th, case["tel_hist"])
    tel_eq(ts, case["tel_sum"])
    assert np.array_equal(data.keys_host(), before[0]) and np.array_equal(data.values_host(), before[1])


@pytest.mark.parametrize("case", M["aggregate_digest"], ids=lambda c: c["name"])
def test_aggregate_digest(S, case):
    fam, par, n, bits = case["gen"]
    keys, vals = gen_keys_values(fam, par, n, bits, seed=1)
    assert sha(keys, vals) == case["input_sha"]
    vals = vals >> (np.uint64(32) if bits == 64 else np.uint32(0))
    P = S.TuningParams.for_input(n, **case["params"])
    spec = S.ReduceSpec.counting() if case["kind"] == "count" else S.ReduceSpec.summing64()
    tel = S.Telemetry()
    res = S.collect_reduce(S.RecordArray(keys, vals), S.UIntKeyAdapter(), spec, P, telemetry=tel)
    assert len(res) == case["n_pairs"]
    assert sha(_sorted_pairs(res)) == case["sorted_pairs_sha"]
    tel_eq(tel, case["telemetry"])


def test_aggregate_examples_and_errors(S):
    adp = S.UIntKeyAdapter()
    t = lambda ks: S.RecordArray(np.asarray(ks, np.uint64), np.arange(len(ks), dtype=np.uint64))  # noqa: E731
    assert S.histogram(t([]), adp).pairs == []
    assert S.histogram(t([7, 7, 7]), adp).pairs == [(7, 3)]
    assert dict(S.histogram(t([2, 1, 2, 3]), adp).pairs) == {2: 2, 1: 1, 3: 1}
    with pytest.raises(S.ConfigurationError):
        S.collect_reduce(S.RecordArray(np.arange(10, dtype=np.uint64)), adp, S.ReduceSpec.summing64())
    with pytest.raises(S.ContractError):
        S.collect_reduce(t([1, 2]), adp, S.ReduceSpec(lambda k, v: v, lambda a, b: a + b, 0))
    tel = S.Telemetry()
    res = S.histogram(S.RecordArray(np.zeros(10**5, np.uint64)), adp, S.TuningParams.for_input(10**5), telemetry=tel)
    assert res.pairs == [(0, 10**5)] and tel.scratch_moves == 0


def test_aggregate_vs_oracle_large(S):
    rng = np.random.default_rng(8)
    n = 3_000_000
    keys = np.floor(rng.exponential(1e3, n)).astype(np.uint64)
    vals = rng.integers(0, 2**63, n).astype(np.uint64) * np.uint64(3)
    res = S.collect_reduce(S.RecordArray(keys, vals), S.UIntKeyAdapter(), S.ReduceSpec.summing64())
    ref = O.reduce_by_key(keys, vals, "sum64")
    k, v = res.to_numpy()
    assert len(k) == len(ref) and dict(zip(k.tolist(), v.tolist())) == ref
    keys32 = rng.integers(0, 10**6, n).astype(np.uint32)
    res = S.histogram(S.RecordArray(keys32), S.UIntKeyAdapter())
    k, v = res.to_numpy()
    assert dict(zip(k.tolist(), v.tolist())) == O.reduce_by_key(keys32, None, "count")


# ---- node folds (csrc/node_fold.cuh) ----------------------------------------------

def _fold_cases():
    rng = np.random.default_rng(21)
    n = 1 << 20
    u32max, u64max = np.uint32(0xFFFFFFFF), np.uint64(0xFFFFFFFFFFFFFFFF)
    zipf = np.minimum(rng.zipf(1.3, n), 10**6).astype(np.uint64)
    k32 = rng.integers(0, 20000, n).astype(np.uint32)
    k32[rng.integers(0, n, 5000)] = u32max              # the table's empty marker as a real key
    k64 = (rng.integers(0, 5000, n).astype(np.uint64) * np.uint64(0x9E3779B97F4A7C15))
    k64[rng.integers(0, n, 3000)] = u64max
    wide = rng.integers(0, 2**63, 1 << 22).astype(np.uint64)   # level-2 nodes overflow the table
    few = rng.integers(0, 1000, n).astype(np.uint64)            # children >= alpha: nodes recurse
    # one key with > 65535 records inside an eligible level-2 node: its
    # 16-bit fold count wraps, the node total catches it (level path)
    wrap = rng.integers(0, 2000, 1 << 21).astype(np.uint32)
    wrap[rng.choice(1 << 21, 70000, replace=False)] = np.uint32(12345)
    vals = lambda m: rng.integers(0, 2**64 - 1, m, dtype=np.uint64, endpoint=True)  # noqa: E731
    return [
        ("u32_marker", k32, vals(n), {"light_buckets": 64, "base_case_cutoff": 4096}, False),
        ("u64_marker", k64, vals(n), {"light_buckets": 64, "base_case_cutoff": 4096}, False),
        ("zipf_heavy", zipf, vals(n), {"light_buckets": 64, "base_case_cutoff": 2048}, False),
        ("identity", k32.astype(np.uint64), vals(n), {"light_buckets": 32, "base_case_cutoff": 4096}, True),
        ("wide_overflow", wide, vals(len(wide)), {"light_buckets": 64, "base_case_cutoff": 16384}, False),
        ("few_recurse", few, vals(n), {"light_buckets": 4, "base_case_cutoff": 16384}, False),
        ("u16_wrap", wrap, vals(len(wrap)), {"light_buckets": 16, "base_case_cutoff": 1 << 17, "max_heavy": 0}, False),
    ]


@pytest.mark.parametrize("case", _fold_cases(), ids=lambda c: c[0])
def test_node_fold_vs_oracle_and_level_path(S, case, monkeypatch):
    """Folded nodes give the reference's pairs and Telemetry; the level path
    (SS_NODE_FOLD=0) gives the same; overflowing / recursing nodes fall back."""
    name, keys, vals, kw, ident = case
    n = len(keys)
    P = S.TuningParams.for_input(n, **kw)
    OP = O.OracleParams.derive(n, **kw)
    adp = S.UIntKeyAdapter(identity=ident)
    folded = {}
    for kind, spec in (("count", S.ReduceSpec.counting()), ("sum64", S.ReduceSpec.summing64())):
        runs = {}
        for mode in ("1", "0"):
            monkeypatch.setenv("SS_NODE_FOLD", mode)
            tel = S.Telemetry()
            res = S.collect_reduce(S.RecordArray(keys, vals), adp, spec, P, telemetry=tel)
            runs[mode] = (_sorted_pairs(res), tel)
        monkeypatch.delenv("SS_NODE_FOLD")
        pairs, otel = O.collect_reduce(keys, vals if kind == "sum64" else None, OP, kind, identity=ident)
        ref = np.array(sorted(pairs), dtype=np.uint64).reshape(-1, 2)
        for mode, (got, tel) in runs.items():
            assert np.array_equal(got, ref), (name, kind, mode)
            assert tel.max_depth == otel.max_depth and tel.nodes == otel.nodes, (name, kind, mode)
            assert tel.scratch_moves == otel.scratch_moves and tel.bucket_assignments == otel.bucket_assignments
            assert {int(k): v for k, v in tel.matrix_cells_by_level.items()} == \
                {int(k): v for k, v in otel.matrix_cells_by_level.items()}
        assert runs["0"][1].nodes_folded == 0
        folded[kind] = runs["1"][1].nodes_folded
        if name == "wide_overflow":
            assert runs["1"][1].nodes_folded == 0, name   # every level-2 node overflowed
        elif name != "few_recurse":   # (its level-2 nodes recurse; deeper ones may fold)
            assert runs["1"][1].nodes_folded > 0, name
        # deterministic output order
        res2 = S.collect_reduce(S.RecordArray(keys, vals), adp, spec, P)
        k1, a1 = S.collect_reduce(S.RecordArray(keys, vals), adp, spec, P).to_numpy()
        k2, a2 = res2.to_numpy()
        assert np.array_equal(k1, k2) and np.array_equal(a1, a2)
    if name == "u16_wrap":   # the hot key's node folds with 32-bit sum-side counts, not with 16-bit ones
        assert folded["count"] == folded["sum64"] - 1, folded


# ---- leaf size classes ---------------------------------------------------------------

@pytest.mark.parametrize("kdt", [np.uint32, np.uint64])
@pytest.mark.parametrize("lb,alpha", [(512, 16384), (64, 65536)])
def test_leaf_classes_vs_oracle(S, kdt, lb, alpha):
    """Mid-size leaves (1025..4096 records: shared-memory k_leaf_eq_mid) and
    larger ones (global scratch) reproduce the reference order byte for
    byte; u32 keys also run the 8192-record distribute tiles."""
    rng = np.random.default_rng(17)
    n = 1 << 21
    keys = rng.integers(0, 1 << 20, n).astype(kdt)
    vals = np.arange(n, dtype=np.uint64)
    kw = {"light_buckets": lb, "base_case_cutoff": alpha}
    ko, vo, tel_o = O.semisort(keys, vals, O.OracleParams.derive(n, **kw))
    data = S.RecordArray(keys, vals)
    tel = S.Telemetry()
    S.semisort(data, S.UIntKeyAdapter(), "eq", S.TuningParams.for_input(n, **kw), telemetry=tel)
    assert np.array_equal(data.values_host(), vo) and np.array_equal(data.keys_host(), ko)
    assert tel.max_depth == tel_o.max_depth and tel.nodes == tel_o.nodes
    assert tel.leaves_global > 0   # the mid / global class ran
