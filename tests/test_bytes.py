"""Byte-view keys and n-grams (adapters.py:200-275,
hashing.py:56-106, ngrams.py).

Fixtures: tests/golden/make_golden_bytes.py ran the unmodified reference.
CPU tier: the oracle's hash and byte-view semisort reproduce them; the
package's host hash (BytesKeyAdapter.hash_scalar) too.  GPU tier: the device
hash, the device n-gram builder, semisort (eq / lt) and histogram /
collect_reduce reproduce the reference byte for byte (pairs as multisets,
every Telemetry counter equal); a forced hash collision raises instead of
merging groups.
"""

from __future__ import annotations

import json
import os

import numpy as np
import pytest
import torch

import oracle as O

HERE = os.path.dirname(os.path.abspath(__file__))
G = np.load(os.path.join(HERE, "golden", "golden_bytes.npz"))
META = json.loads(str(G["meta"]))
TEXTS = META["texts"]
SORTS = META["sorts"]
AGGS = META["aggs"]


def _kat_strings():
    blob = G["kat_blob"].tobytes()
    out, at = [], 0
    for n in G["kat_len"].tolist():
        out.append(blob[at:at + n])
        at += n
    return out


def _params(S_or_O, n, kw):
    return S_or_O.TuningParams.for_input(n, **kw) if hasattr(S_or_O, "TuningParams") else \
        O.OracleParams.derive(n, **kw)


def _tel_eq(tel, ref):
    assert (tel.max_depth, tel.nodes, tel.scratch_moves, tel.bucket_assignments) == \
        (ref["max_depth"], ref["nodes"], ref["scratch_moves"], ref["bucket_assignments"])
    assert {str(k): v for k, v in tel.matrix_cells_by_level.items()} == ref["matrix_cells_by_level"]


# ---- CPU tier ------------------------------------------------------------------

def test_oracle_hash_kats():
    assert [O.hash_bytes(s) for s in _kat_strings()] == G["kat_hash"].tolist()


def test_oracle_prefix_hasher_views():
    cs = O.bytes_oracle.contents(G["pre_arena"], np.stack([G["pre_off"], G["pre_len"]], axis=1))
    assert [O.hash_bytes(c) for c in cs] == G["pre_hash"].tolist()


def test_host_hash_scalar_matches_reference():
    from paper_2304_10078_b200.adapters import BytesKeyAdapter
    a = BytesKeyAdapter()
    assert [a.hash_scalar(s) for s in _kat_strings()] == G["kat_hash"].tolist()


@pytest.mark.parametrize("case", SORTS, ids=lambda c: f"{c['name']}-{c['mode']}")
def test_oracle_semisort_bytes_matches_reference(case):
    name, mode = case["name"], case["mode"]
    from_ref = _ngram_ref(name)
    keys, values, arena = from_ref
    n = len(keys)
    vo, vv, tel = O.semisort_bytes(arena, keys, values, O.OracleParams.derive(n, **case["params"]), mode)
    assert np.array_equal(vo, G[f"sort_{name}_{mode}_keys"])
    assert np.array_equal(vv, G[f"sort_{name}_{mode}_values"])
    _tel_eq(tel, case["telemetry"])


def _ngram_ref(name):
    """The corpus' n-gram records as the reference's build_ngrams made them."""
    return G[f"cng_{name}_keys"], G[f"cng_{name}_values"], G[f"cng_{name}_arena"]


def _np_build_ngrams(text: bytes, g: int):
    """numpy statement of ngrams.py:23-89 (test helper)."""
    raw = np.frombuffer(text, dtype=np.uint8).astype(np.int32)
    low = np.where((raw >= 65) & (raw <= 90), raw + 32, raw)
    alpha = (low >= 97) & (low <= 122)
    words, cur = [], []
    for c, a in zip(low.tolist(), alpha.tolist()):
        if a:
            cur.append(c)
        elif cur:
            words.append(bytes(cur))
            cur = []
    if cur:
        words.append(bytes(cur))
    arena = b" ".join(words)
    starts = np.cumsum([0] + [len(w) + 1 for w in words[:-1]]).astype(np.uint64) if words else np.zeros(0, np.uint64)
    lens = np.array([len(w) for w in words], dtype=np.uint64)
    count = max(0, len(words) - g + 1)
    keys = np.zeros((count, 2), np.uint64)
    values = np.zeros((count, 2), np.uint64)
    if count:
        h = g - 1
        keys[:, 0] = starts[:count]
        keys[:, 1] = starts[h - 1:h - 1 + count] + lens[h - 1:h - 1 + count] - starts[:count]
        values[:, 0] = starts[h:h + count]
        values[:, 1] = lens[h:h + count]
    return np.frombuffer(arena, dtype=np.uint8), keys, values


@pytest.mark.parametrize("t", TEXTS, ids=lambda t: t["name"])
def test_np_ngram_statement_matches_reference(t):
    name = t["name"]
    arena, keys, values = _np_build_ngrams(G[f"text_{name}"].tobytes(), t["gram"])
    assert np.array_equal(arena, G[f"ng_{name}_arena"])
    assert np.array_equal(keys, G[f"ng_{name}_keys"]) and np.array_equal(values, G[f"ng_{name}_values"])


# ---- GPU tier --------------------------------------------------------------------

@pytest.fixture(scope="module")
def S():
    import paper_2304_10078_b200 as S
    assert torch.cuda.is_available()
    return S


def _records(S, name):
    """The device n-gram builder on the corpus text (checked against the
    reference's arrays here too)."""
    from paper_2304_10078_b200.ngrams import build_ngrams
    g = next(c["gram"] for c in SORTS if c["name"] == name)
    rec = build_ngrams(G[f"corpus_{name}"].tobytes(), g)
    assert np.array_equal(rec.keys_host(), G[f"cng_{name}_keys"])
    assert np.array_equal(rec.values_host(), G[f"cng_{name}_values"])
    assert np.array_equal(rec.arena.cpu().numpy(), G[f"cng_{name}_arena"])
    return rec


@pytest.mark.gpu
def test_device_hash_kats(S):
    from paper_2304_10078_b200 import bytes_keys
    strings = _kat_strings()
    lens = np.array([len(s) for s in strings], dtype=np.uint64)
    offs = np.concatenate([[0], np.cumsum(lens)[:-1]]).astype(np.uint64)
    data = S.RecordArray(np.stack([offs, lens], axis=1), key_kind="bytes", arena=G["kat_blob"])
    assert bytes_keys.content_hashes(data).cpu().numpy().tolist() == G["kat_hash"].tolist()
    pre = S.RecordArray(np.stack([G["pre_off"], G["pre_len"]], axis=1), key_kind="bytes", arena=G["pre_arena"])
    assert np.array_equal(bytes_keys.content_hashes(pre).cpu().numpy(), G["pre_hash"])


@pytest.mark.gpu
@pytest.mark.parametrize("t", TEXTS, ids=lambda t: t["name"])
def test_device_build_ngrams_matches_reference(S, t):
    from paper_2304_10078_b200.ngrams import build_ngrams
    name = t["name"]
    rec = build_ngrams(G[f"text_{name}"].tobytes(), t["gram"])
    assert np.array_equal(rec.arena.cpu().numpy(), G[f"ng_{name}_arena"])
    assert np.array_equal(rec.keys_host().reshape(-1, 2), G[f"ng_{name}_keys"])
    assert np.array_equal(rec.values_host().reshape(-1, 2), G[f"ng_{name}_values"])


@pytest.mark.gpu
@pytest.mark.parametrize("case", SORTS, ids=lambda c: f"{c['name']}-{c['mode']}")
def test_gpu_semisort_bytes_matches_reference(S, case):
    from paper_2304_10078_b200.ngrams import ngram_adapter
    name, mode = case["name"], case["mode"]
    rec = _records(S, name)
    tel = S.Telemetry()
    S.semisort(rec, ngram_adapter(rec), mode, S.TuningParams.for_input(len(rec), **case["params"]), telemetry=tel)
    assert np.array_equal(rec.keys_host(), G[f"sort_{name}_{mode}_keys"])
    assert np.array_equal(rec.values_host(), G[f"sort_{name}_{mode}_values"])
    _tel_eq(tel, case["telemetry"])
    assert tel.scratch_allocations == 1


@pytest.mark.gpu
@pytest.mark.parametrize("case", AGGS, ids=lambda c: f"{c['name']}-{c['kind']}")
def test_gpu_aggregate_bytes_matches_reference(S, case):
    from paper_2304_10078_b200.ngrams import ngram_adapter
    rec = _records(S, case["name"])
    before = rec.copy()
    tel = S.Telemetry()
    params = S.TuningParams.for_input(len(rec), **case["params"])
    if case["kind"] == "count":
        res = S.histogram(rec, ngram_adapter(rec), params, telemetry=tel)
    else:
        res = S.collect_reduce(rec, ngram_adapter(rec), S.ReduceSpec.summing64(), params, telemetry=tel)
    got = sorted([k.decode("latin-1"), int(v)] for k, v in res.pairs)
    assert got == case["pairs"]
    _tel_eq(tel, case["telemetry"])
    assert rec.same_bytes(before)   # aggregation never modifies its input


@pytest.mark.gpu
def test_gpu_ngram_reference_example(S):
    """test_aggregate.py:191-198 of the reference."""
    from paper_2304_10078_b200.ngrams import build_ngrams, ngram_adapter
    rec = build_ngrams("a b a b a c a b", 2)
    res = S.histogram(rec, ngram_adapter(rec), S.TuningParams.for_input(len(rec), light_buckets=4,
                                                                        subarray_len=8, base_case_cutoff=8,
                                                                        max_heavy=2))
    assert dict(res.pairs) == {b"a": 4, b"b": 2, b"c": 1}


@pytest.mark.gpu
def test_gpu_bytes_validate_and_errors(S):
    from paper_2304_10078_b200 import bytes_keys
    from paper_2304_10078_b200.ngrams import ngram_adapter
    rec = _records(S, "small")
    before = rec.copy()
    S.semisort(rec, ngram_adapter(rec), "eq")
    assert S.validate_semisort(before, rec).valid
    bad = S.RecordArray(np.array([[0, 5], [3, 9]], np.uint64), key_kind="bytes", arena=np.zeros(8, np.uint8))
    with pytest.raises(S.InputFormatError):
        S.semisort(bad, S.BytesKeyAdapter(bad.arena), "eq")
    with pytest.raises(S.ContractError):
        S.semisort(rec, S.UIntKeyAdapter(), "eq")
    with pytest.raises(S.ContractError):
        S.semisort(S.RecordArray(np.arange(4, dtype=np.uint64)), S.BytesKeyAdapter(), "eq")
    assert bytes_keys.HashCollision


@pytest.mark.gpu
def test_gpu_bytes_hash_collision_is_detected(S, monkeypatch):
    """Equal (hash, length) with different bytes must not merge groups."""
    from paper_2304_10078_b200 import bytes_keys
    arena = np.frombuffer(b"abcdabceabcd", dtype=np.uint8)
    views = np.array([[0, 4], [4, 4], [8, 4]], np.uint64)
    monkeypatch.setattr(bytes_keys, "content_hashes",
                        lambda data: torch.zeros(len(data), dtype=torch.uint64, device=data.device))
    rec = S.RecordArray(views, key_kind="bytes", arena=arena)
    with pytest.raises(bytes_keys.HashCollision):
        S.semisort(rec, S.BytesKeyAdapter(rec.arena), "eq")
    with pytest.raises(bytes_keys.HashCollision):
        S.histogram(S.RecordArray(views, key_kind="bytes", arena=arena), S.BytesKeyAdapter(arena))
