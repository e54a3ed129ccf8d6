"""128-bit keys (adapters.py:147-198, records.py:8-10).

CPU tier: the oracle's u128 restatement reproduces the reference's outputs
(tests/golden/golden_u128.npz, made by make_golden_u128.py from the
unmodified reference) and its heavy-key sampler.  GPU tier: semisort through
the public API reproduces the same fixtures byte for byte, and matches the
oracle at larger sizes in both modes.
"""

from __future__ import annotations

import os

import numpy as np
import pytest

import oracle as O

HERE = os.path.dirname(os.path.abspath(__file__))
G = np.load(os.path.join(HERE, "golden", "golden_u128.npz"))
TAGS = [str(t) for t in G["tags"]]
CASES = [str(c) for c in G["cases"]]
_PK = ("light_buckets", "subarray_len", "base_case_cutoff", "max_heavy")


def _kw(case):
    return {k: int(v) for k, v in zip(_PK, G[f"{case}_params"]) if v >= 0}


def _split(tag):
    case, mode, ident, with_v = tag.rsplit("_", 3)
    return case, mode, ident == "1", with_v == "1"


def _vals(n, with_v):
    return np.arange(n, dtype=np.uint64) * 3 + 1 if with_v else None


@pytest.mark.parametrize("tag", TAGS)
def test_oracle_matches_reference(tag):
    case, mode, ident, with_v = _split(tag)
    keys = G[f"{case}_keys"]
    n = len(keys)
    ko, vo, _ = O.semisort(keys, _vals(n, with_v), O.OracleParams.derive(n, **_kw(case)), mode, ident)
    assert np.array_equal(ko, G[f"{tag}_out_k"])
    if with_v:
        assert np.array_equal(vo, G[f"{tag}_out_v"])


@pytest.mark.parametrize("case", [c for c in CASES if f"{c}_heavy_0" in G.files])
@pytest.mark.parametrize("ident", [0, 1])
def test_oracle_sampler_matches_reference(case, ident):
    keys = G[f"{case}_keys"]
    P = O.OracleParams.derive(len(keys), **_kw(case))
    got = np.asarray(O.sample_heavy(keys, P, 1234), dtype=np.uint64).reshape(-1, 2)
    assert np.array_equal(got, G[f"{case}_heavy_{ident}"])


def test_oracle_hash_u128():
    k = np.array([[1, 2], [2**64 - 1, 0], [0, 2**64 - 1]], dtype=np.uint64)
    h = O.key_hash(k, False)
    for (lo, hi), hv in zip(k.tolist(), h.tolist()):
        assert hv == O.mix64_int(O.mix64_int(hi) ^ lo)           # adapters.py:157-159
    assert np.array_equal(O.key_hash(k, True), k[:, 0])


# ---- GPU ------------------------------------------------------------------

@pytest.fixture(scope="module")
def S():
    import paper_2304_10078_b200 as S
    return S


@pytest.mark.gpu
@pytest.mark.parametrize("tag", TAGS)
def test_semisort_u128_golden(S, tag):
    case, mode, ident, with_v = _split(tag)
    keys = G[f"{case}_keys"]
    n = len(keys)
    data = S.RecordArray(keys, _vals(n, with_v))
    S.semisort(data, S.UInt128KeyAdapter(identity=ident), mode, S.TuningParams.for_input(n, **_kw(case)))
    assert np.array_equal(data.keys_host(), G[f"{tag}_out_k"])
    if with_v:
        assert np.array_equal(data.values_host(), G[f"{tag}_out_v"])


def _u128_keys(rng, n, dist):
    k = np.empty((n, 2), dtype=np.uint64)
    if dist == "uniform":
        k[:] = rng.integers(0, 2**64 - 1, (n, 2), dtype=np.uint64, endpoint=True)
    elif dist == "zipf":
        z = np.minimum(rng.zipf(1.3, n), 10**7).astype(np.uint64)
        k[:, 0] = O.mix64_np(z)
        k[:, 1] = z & np.uint64(7)
    else:   # few distinct keys differing in hi only
        k[:, 0] = 12345
        k[:, 1] = rng.integers(0, 300, n).astype(np.uint64)
    return k


@pytest.mark.gpu
@pytest.mark.parametrize("dist", ["uniform", "zipf", "hionly"])
@pytest.mark.parametrize("mode", ["eq", "lt"])
def test_semisort_u128_vs_oracle_1m(S, dist, mode):
    rng = np.random.default_rng(17)
    n = 1 << 20
    keys = _u128_keys(rng, n, dist)
    vals = np.arange(n, dtype=np.uint64)
    ident = dist == "hionly" and mode == "eq"   # identity hash: every key collides on lo
    ko, vo, tel_o = O.semisort(keys, vals, O.OracleParams.derive(n), mode, ident)
    data = S.RecordArray(keys, vals)
    tel = S.Telemetry()
    S.semisort(data, S.UInt128KeyAdapter(identity=ident), mode, S.TuningParams.for_input(n), telemetry=tel)
    assert np.array_equal(data.values_host(), vo)
    assert np.array_equal(data.keys_host(), ko)
    assert tel.max_depth == tel_o.max_depth and tel.nodes == tel_o.nodes


@pytest.mark.gpu
def test_u128_value_layouts(S):
    rng = np.random.default_rng(3)
    n = 200000
    keys = _u128_keys(rng, n, "zipf")
    P = O.OracleParams.derive(n, base_case_cutoff=2048)
    _, vo, _ = O.semisort(keys, np.arange(n, dtype=np.uint64), P)
    for vals in (None, np.arange(n, dtype=np.uint32),
                 np.stack([np.arange(n), np.arange(n) * 7], axis=1).astype(np.uint64)):
        d = S.RecordArray(keys, vals)
        S.semisort(d, S.UInt128KeyAdapter(), "eq", S.TuningParams.for_input(n, base_case_cutoff=2048))
        assert np.array_equal(d.keys_host(), keys[vo.astype(np.int64)])
        if vals is not None:
            v = d.values_host()
            v0 = v[:, 0] if v.ndim == 2 else v
            assert np.array_equal(v0.astype(np.int64), vo.astype(np.int64))


@pytest.mark.gpu
def test_u128_errors(S):
    k = np.array([[1, 2], [3, 4]], dtype=np.uint64)
    with pytest.raises(S.ContractError):            # adapter / key kind mismatch
        S.semisort(S.RecordArray(k), S.UIntKeyAdapter(), "eq")
    with pytest.raises(S.ContractError):
        S.semisort(S.RecordArray(np.array([1, 2], np.uint64)), S.UInt128KeyAdapter(), "eq")
    with pytest.raises(S.ContractError):            # aggregation: adapter / key kind mismatch
        S.histogram(S.RecordArray(k), S.UIntKeyAdapter())
    with pytest.raises(S.ContractError):
        S.histogram(S.RecordArray(np.array([1, 2], np.uint64)), S.UInt128KeyAdapter())


# ---- collect_reduce / histogram over 128-bit keys (aggregate.py:267-299) -----

GA = np.load(os.path.join(HERE, "golden", "golden_u128_agg.npz"))
AGG_TAGS = [str(t) for t in GA["tags"]]
AGG_META = __import__("json").loads(str(GA["meta"]))


def _agg_split(tag):
    case, kind, ident = tag.rsplit("_", 2)
    return case, kind, ident == "1"


def _multiset(k, a):
    k = np.asarray(k, dtype=np.uint64).reshape(-1, 2)
    order = np.lexsort((k[:, 0], k[:, 1]))
    return k[order], np.asarray(a, dtype=np.uint64)[order]


@pytest.mark.parametrize("tag", AGG_TAGS)
def test_u128_aggregate_fixture_semantics(tag):
    """The reference's pairs are one (key, count | wrapping sum) per distinct
    128-bit key (numpy restatement: unique rows + bincount / add.at)."""
    case, kind, _ = _agg_split(tag)
    keys = G[f"{case}_keys"]
    uniq, inv = np.unique(keys, axis=0, return_inverse=True) if len(keys) else (np.zeros((0, 2), np.uint64), None)
    if kind == "count":
        agg = np.bincount(inv.ravel(), minlength=len(uniq)).astype(np.uint64) if len(keys) else np.zeros(0, np.uint64)
    else:
        agg = np.zeros(len(uniq), dtype=np.uint64)
        if len(keys):
            np.add.at(agg, inv.ravel(), GA[f"{case}_vals"])
    rk, ra = _multiset(GA[f"{tag}_k"], GA[f"{tag}_a"])
    ek, ea = _multiset(uniq, agg)
    assert np.array_equal(rk, ek) and np.array_equal(ra, ea)


@pytest.mark.gpu
@pytest.mark.parametrize("tag", AGG_TAGS)
def test_u128_aggregate_gpu_matches_reference(S, tag):
    case, kind, ident = _agg_split(tag)
    keys = G[f"{case}_keys"]
    n = len(keys)
    params = S.TuningParams.for_input(n, **_kw(case))
    adp = S.UInt128KeyAdapter(identity=ident)
    tel = S.Telemetry()
    if kind == "count":
        res = S.histogram(S.RecordArray(keys), adp, params, telemetry=tel)
    else:
        res = S.collect_reduce(S.RecordArray(keys, GA[f"{case}_vals"]), adp, S.ReduceSpec.summing64(), params,
                               telemetry=tel)
    k, a = res.to_numpy()
    rk, ra = _multiset(GA[f"{tag}_k"], GA[f"{tag}_a"])
    gk, ga = _multiset(k, a)
    assert np.array_equal(gk, rk) and np.array_equal(ga, ra)
    ref = AGG_META[tag]
    assert (tel.max_depth, tel.nodes, tel.scratch_moves, tel.bucket_assignments) == \
        (ref["max_depth"], ref["nodes"], ref["scratch_moves"], ref["bucket_assignments"])
    assert {str(k): v for k, v in tel.matrix_cells_by_level.items()} == ref["matrix_cells_by_level"]
    if n:
        assert res.pairs and isinstance(res.pairs[0][0], tuple)   # (lo, hi) like the reference


@pytest.mark.gpu
def test_u128_aggregate_1m_vs_numpy(S):
    rng = np.random.default_rng(29)
    n = 1 << 20
    keys = _u128_keys(rng, n, "zipf")
    vals = rng.integers(0, 2**63, n).astype(np.uint64)
    uniq, inv = np.unique(keys, axis=0, return_inverse=True)
    cnt = np.bincount(inv.ravel(), minlength=len(uniq)).astype(np.uint64)
    sm = np.zeros(len(uniq), dtype=np.uint64)
    np.add.at(sm, inv.ravel(), vals)
    for kind, want in (("count", cnt), ("sum64", sm)):
        if kind == "count":
            res = S.histogram(S.RecordArray(keys), S.UInt128KeyAdapter())
        else:
            res = S.collect_reduce(S.RecordArray(keys, vals), S.UInt128KeyAdapter(), S.ReduceSpec.summing64())
        gk, ga = _multiset(*res.to_numpy())
        ek, ea = _multiset(uniq, want)
        assert np.array_equal(gk, ek) and np.array_equal(ga, ea)
