"""The CPU oracle reproduces every reference fixture byte for byte (CPU tier)."""
import numpy as np
import pytest

import oracle as O
from oracle.datagen import gen_keys_values
from golden_io import meta, sha, small

G = small()
M = meta()


def test_mix64_kats():
    assert np.array_equal(O.mix64_np(G["kat_x"]), G["kat_mix64"])
    assert [O.mix64_int(int(x)) for x in G["kat_x"][:20]] == G["kat_mix64"][:20].tolist()
    pairs = [O.mix64_pair_int(int(a), int(b)) for a, b in zip(G["kat_x"], G["kat_pair_b"])]
    assert pairs == G["kat_pair"].tolist()
    # SURVEY.md Appendix B
    assert O.mix64_int(0) == 0xE220A8397B1DCDAF
    assert O.mix64_pair_int(1, 0) == 0x08B4FDA8C892B50E


@pytest.mark.parametrize("case", M["sampling"], ids=lambda c: c["name"])
def test_sampling(case):
    keys = G[f"samp_{case['name']}_keys"]
    P = O.OracleParams.derive(len(keys), **case["params"])
    got = O.sample_heavy(keys, P, case["rng_key"])
    assert got == G[f"samp_{case['name']}_heavy"].tolist()


@pytest.mark.parametrize("case", M["ids"], ids=lambda c: c["tag"])
def test_bucket_ids(case):
    keys = G["ids_keys"]
    P = O.OracleParams.derive(len(keys), light_buckets=case["n_light"])
    got = O.bucket_ids(keys, case["heavy"], P, case["depth"], case["identity"])
    assert np.array_equal(got, G[case["tag"]])


@pytest.mark.parametrize("case", M["distribute"], ids=lambda c: c["name"])
def test_counts_scan_distribute(case):
    p = f"dist_{case['name']}_"
    ids = G[p + "ids"]
    C = O.count_rows(ids, case["sub_len"], case["n_buckets"])
    assert np.array_equal(C, G[p + "counts"])
    X, off = O.col_scan(C)
    assert np.array_equal(X, G[p + "prefix"])
    assert np.array_equal(off, G[p + "offsets"])
    dest = O.scatter_positions(ids, X, case["sub_len"])
    out = np.empty(len(ids), dtype=np.uint64)
    out[dest] = np.arange(len(ids), dtype=np.uint64)
    assert np.array_equal(out, G[p + "out"])


@pytest.mark.parametrize("name", M["base"])
@pytest.mark.parametrize("ident", [0, 1])
def test_base_cases(name, ident):
    keys = G[f"base_{name}_keys"]
    assert np.array_equal(O.eq_leaf_order(keys, bool(ident)), G[f"base_{name}_eq_{ident}"])
    assert np.array_equal(O.lt_leaf_order(keys), G[f"base_{name}_lt_{ident}"])


def _tel_eq(tel, ref):
    assert tel.max_depth == ref["max_depth"]
    assert tel.nodes == ref["nodes"]
    assert tel.scratch_moves == ref["scratch_moves"]
    assert tel.bucket_assignments == ref["bucket_assignments"]
    assert {str(k): v for k, v in tel.matrix_cells_by_level.items()} == ref["matrix_cells_by_level"]


@pytest.mark.parametrize("case", M["semisort_small"], ids=lambda c: c["name"])
def test_semisort_small(case):
    keys = G[f"ss_{case['name']}_keys"]
    n = len(keys)
    vals = np.arange(n, dtype=keys.dtype)
    P = O.OracleParams.derive(n, **case["params"])
    ko, vo, tel = O.semisort(keys, vals, P, case["mode"], case["identity"])
    assert np.array_equal(vo, G[f"ss_{case['name']}_out"])
    assert np.array_equal(ko, keys[vo.astype(np.int64)])
    _tel_eq(tel, case["telemetry"])


def _gen(gen, hashed):
    fam, par, n, bits = gen
    keys, vals = gen_keys_values(fam, par, n, bits, seed=1)
    return keys, vals


@pytest.mark.parametrize("case", M["semisort_digest"], ids=lambda c: c["name"])
def test_semisort_digest(case):
    keys, vals = _gen(case["gen"], case["hash_ranks"])
    assert sha(keys, vals) == case["input_sha"]
    if case["hash_ranks"]:
        keys = O.mix64_np(keys - np.uint64(1))
    n = len(keys)
    P = O.OracleParams.derive(n, **case["params"])
    ko, vo, tel = O.semisort(keys, np.arange(n, dtype=keys.dtype), P, case["mode"], case["identity"])
    assert sha(ko, vo) == case["out_sha"]
    _tel_eq(tel, case["telemetry"])


@pytest.mark.parametrize("case", M["aggregate"], ids=lambda c: c["name"])
def test_aggregate_small(case):
    p = f"ag_{case['name']}_"
    keys, vals = G[p + "keys"], G[p + "vals"]
    P = O.OracleParams.derive(len(keys), **case["params"])
    hist, th = O.collect_reduce(keys, vals, P, "count", case["identity"])
    summ, ts = O.collect_reduce(keys, vals, P, "sum64", case["identity"])
    assert np.array_equal(np.array(hist, dtype=np.uint64).reshape(-1, 2), G[p + "hist"])
    assert np.array_equal(np.array(summ, dtype=np.uint64).reshape(-1, 2), G[p + "sum"])
    _tel_eq(th, case["tel_hist"])
    _tel_eq(ts, case["tel_sum"])


@pytest.mark.parametrize("case", M["aggregate_digest"], ids=lambda c: c["name"])
def test_aggregate_digest(case):
    fam, par, n, bits = case["gen"]
    keys, vals = gen_keys_values(fam, par, n, bits, seed=1)
    assert sha(keys, vals) == case["input_sha"]
    vals = vals >> (np.uint64(32) if bits == 64 else np.uint32(0))
    P = O.OracleParams.derive(n, **case["params"])
    pairs, tel = O.collect_reduce(keys, vals, P, case["kind"], False)
    arr = np.array(pairs, dtype=np.uint64).reshape(-1, 2)
    assert sha(arr) == case["pairs_sha"]
    _tel_eq(tel, case["telemetry"])


def test_checkers_agree_on_oracle_output():
    keys, _ = gen_keys_values("uniform", 1000, 50000, 64)
    n = len(keys)
    P = O.OracleParams.derive(n, base_case_cutoff=512)
    ko, vo, _ = O.semisort(keys, np.arange(n, dtype=np.uint64), P)
    assert O.semisort_valid(keys, np.arange(n, dtype=np.uint64), ko, vo) == (True, True, True)
    assert O.semisort_valid_indexed(keys, ko, vo)
    bad = vo.copy()
    bad[[10, 11]] = bad[[11, 10]]
    assert not O.semisort_valid_indexed(keys, keys[bad.astype(np.int64)], bad) or \
        ko[10] != ko[11]
