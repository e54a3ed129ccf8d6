"""local_refine (core.py:533-563) and _distribute_ids on a window with
base > 0 (core.py:339-362) against outputs of the unmodified reference
(tests/golden/make_golden_refine.py -> golden_refine.npz).

CPU tier: the oracle restatement reproduces every fixture byte for byte.
GPU tier: the drop-in phase API (sample_and_bucket with the same Philox
stream -> assign_bucket_ids -> counts -> scan -> distribute_ids ->
local_refine) reproduces the refined buffer and the telemetry byte for
byte; distribute_ids on a middle window moves exactly that window."""
import json
import os

import numpy as np
import pytest

import oracle as O

G = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden_refine.npz"))
M = json.loads(bytes(G["meta"]).decode())


def _oracle_flow(case):
    p = f"rf_{case['name']}_"
    keys = G[p + "keys"]
    n = len(keys)
    vals = np.arange(n, dtype=np.uint64)
    P = O.OracleParams.derive(n, **case["params"])
    heavy = O.sample_heavy(keys, P, case["philox_key"])
    ids = O.bucket_ids(keys, heavy, P, 0, case["identity"])
    C = O.count_rows(ids, P.sub_len, P.n_light + len(heavy))
    X, off = O.col_scan(C)
    pos = O.scatter_positions(ids, X, P.sub_len)
    dk, dv = np.empty_like(keys), np.empty_like(vals)
    dk[pos], dv[pos] = keys, vals
    if case["live_in_primary"]:
        prim, scr = (dk, dv), (np.empty_like(keys), np.empty_like(vals))
    else:
        prim, scr = (keys, vals), (dk, dv)
    return heavy, O.local_refine(prim, scr, off, case["live_in_primary"], P, case["mode"], case["identity"])


@pytest.mark.parametrize("case", M["refine"], ids=lambda c: c["name"])
def test_oracle_local_refine_matches_reference(case):
    p = f"rf_{case['name']}_"
    heavy, (ko, vo, tel) = _oracle_flow(case)
    assert [int(h) for h in heavy] == G[p + "heavy"].tolist()
    assert np.array_equal(ko, G[p + "out_keys"]) and np.array_equal(vo, G[p + "out_vals"])
    t = case["telemetry"]
    assert (tel.max_depth, tel.nodes, tel.scratch_moves, tel.bucket_assignments) == \
        (t["max_depth"], t["nodes"], t["scratch_moves"], t["bucket_assignments"])
    assert {str(k): v for k, v in tel.matrix_cells_by_level.items()} == t["matrix_cells_by_level"]


@pytest.mark.parametrize("case", M["window"], ids=lambda c: c["name"])
def test_oracle_distribute_window_matches_reference(case):
    p = f"win_{case['name']}_"
    keys, vals, ids = G[p + "keys"], G[p + "vals"], G[p + "ids"]
    base, m = case["base"], case["m"]
    P = O.OracleParams.derive(m, **case["params"])
    C = O.count_rows(ids, P.sub_len, P.n_light)
    X, _ = O.col_scan(C)
    dk, dv = np.full(len(keys), 7, np.uint64), np.full(len(keys), 9, np.uint64)
    pos = base + O.scatter_positions(ids, X, P.sub_len)
    dk[pos], dv[pos] = keys[base:base + m], vals[base:base + m]
    assert np.array_equal(dk, G[p + "dst_keys"]) and np.array_equal(dv, G[p + "dst_vals"])


# ---- GPU tier -------------------------------------------------------------

@pytest.fixture(scope="module")
def S():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2304_10078_b200 as S
    return S


@pytest.mark.gpu
@pytest.mark.parametrize("case", M["refine"], ids=lambda c: c["name"])
def test_gpu_local_refine_matches_reference(S, case):
    p = f"rf_{case['name']}_"
    keys = G[p + "keys"]
    n = len(keys)
    adp = S.UIntKeyAdapter(identity=case["identity"])
    P = S.TuningParams.for_input(n, **case["params"])
    data = S.RecordArray(keys, np.arange(n, dtype=np.uint64))
    heavy = S.sample_and_bucket(data, adp, P, 0, np.random.Generator(np.random.Philox(key=case["philox_key"])))
    assert heavy.keys == G[p + "heavy"].tolist()
    ids = S.assign_bucket_ids(data, heavy, adp, P, 0)
    nb = P.light_buckets + len(heavy)
    counts = S.core.counts_from_ids(ids, P, nb)
    prefix, offsets = S.column_major_exclusive_scan(counts)
    other = data.empty_like()
    S.core.distribute_ids(data, other, 0, ids, prefix, P, nb)
    if case["live_in_primary"]:
        bufs = S.WorkBuffers(primary=other, scratch=data.empty_like(), live_in_primary=True)
    else:
        bufs = S.WorkBuffers(primary=data, scratch=other, live_in_primary=False)
    tel = S.Telemetry()
    S.local_refine(bufs, S.BucketPlan(heavy, counts, prefix, offsets), adp, case["mode"], P, depth=0, telemetry=tel)
    assert np.array_equal(bufs.primary.keys_host(), G[p + "out_keys"])
    assert np.array_equal(bufs.primary.values_host(), G[p + "out_vals"])
    t = case["telemetry"]
    assert (tel.max_depth, tel.nodes, tel.scratch_moves, tel.bucket_assignments) == \
        (t["max_depth"], t["nodes"], t["scratch_moves"], t["bucket_assignments"])
    assert {str(k): v for k, v in tel.matrix_cells_by_level.items()} == t["matrix_cells_by_level"]


@pytest.mark.gpu
@pytest.mark.parametrize("case", M["window"], ids=lambda c: c["name"])
def test_gpu_distribute_window_matches_reference(S, case):
    """distribute_ids moves exactly src[base:base+len(ids)]."""
    import torch
    p = f"win_{case['name']}_"
    keys, vals, ids = G[p + "keys"], G[p + "vals"], G[p + "ids"]
    base, m = case["base"], case["m"]
    P = S.TuningParams.for_input(m, **case["params"])
    counts = S.core.counts_from_ids(ids, P, P.light_buckets)
    prefix, _ = S.column_major_exclusive_scan(counts)
    src = S.RecordArray(keys, vals)
    dst = S.RecordArray(np.full(len(keys), 7, np.uint64), np.full(len(keys), 9, np.uint64))
    S.core.distribute_ids(src, dst, base, torch.from_numpy(ids).cuda(), prefix, P, P.light_buckets)
    assert np.array_equal(dst.keys_host(), G[p + "dst_keys"]) and np.array_equal(dst.values_host(), G[p + "dst_vals"])


@pytest.mark.gpu
def test_gpu_bucket_id_range_checked(S):
    """Out-of-range caller ids raise ConfigurationError (no device fault)."""
    import torch
    P = S.TuningParams.for_input(1000, light_buckets=8, subarray_len=64)
    bad = torch.full((1000,), 3, dtype=torch.int32, device="cuda")
    bad[500] = 8
    with pytest.raises(S.ConfigurationError):
        S.core.counts_from_ids(bad, P, 8)
    bad[500] = -1
    with pytest.raises(S.ConfigurationError):
        S.core.counts_from_ids(bad, P, 8)
    data = S.RecordArray(np.arange(1000, dtype=np.uint64), np.arange(1000, dtype=np.uint64))
    counts = torch.zeros((P.num_subarrays(1000), 8), dtype=torch.int64, device="cuda")
    prefix, _ = S.column_major_exclusive_scan(counts)
    with pytest.raises(S.ConfigurationError):
        S.core.distribute_ids(data, data.empty_like(), 0, bad, prefix, P, 8)
    # the context is still usable afterwards
    good = torch.full((1000,), 3, dtype=torch.int32, device="cuda")
    assert int(S.core.counts_from_ids(good, P, 8).sum().item()) == 1000
