"""The fallback kernels behind the fast paths, against the same fixtures
(GPU tier).

* SS_HW_RANK=0: the distribute and leaf kernels rank by shared atomicOr
  peer masks instead of relying on a shared atomicAdd returning old values
  in lane order (probe.cuh); output must not change (the reference's
  "no atomics decide order").
* SS_DIST_KERNEL=radix: the two-pass 7-bit LSD distribute (dist.cuh)
  instead of the single-pass one (dist1.cuh), which also turns the pair
  scratch layout off.
* Both at once.
Each mode reruns the reference's small semisorts (byte-equal outputs and
telemetry), the reference digests (c1 included), the 4M-record oracle
comparisons and the aggregates.  The environment is read on every call.
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
MODES = {"hw_rank_off": {"SS_HW_RANK": "0"}, "radix": {"SS_DIST_KERNEL": "radix"},
         "both": {"SS_HW_RANK": "0", "SS_DIST_KERNEL": "radix"}}


@pytest.fixture(scope="module")
def S():
    import paper_2304_10078_b200 as S
    assert torch.cuda.is_available()
    return S


@pytest.fixture(params=list(MODES))
def fallback(request, monkeypatch):
    for k, v in MODES[request.param].items():
        monkeypatch.setenv(k, v)
    return request.param


def _tel_eq(tel, ref):
    assert (tel.max_depth, tel.nodes, tel.scratch_moves, tel.bucket_assignments) == \
        (ref["max_depth"], ref["nodes"], ref["scratch_moves"], ref["bucket_assignments"])
    assert {str(k): v for k, v in tel.matrix_cells_by_level.items()} == ref["matrix_cells_by_level"]


def test_semisort_small_fallback(S, fallback):
    for case in M["semisort_small"]:
        keys = G[f"ss_{case['name']}_keys"]
        n = len(keys)
        data = S.RecordArray(keys, np.arange(n, dtype=keys.dtype))
        tel = S.Telemetry()
        S.semisort(data, S.UIntKeyAdapter(identity=case["identity"]), case["mode"],
                   S.TuningParams.for_input(n, **case["params"]), telemetry=tel)
        assert np.array_equal(data.values_host(), G[f"ss_{case['name']}_out"]), case["name"]
        _tel_eq(tel, case["telemetry"])


def test_semisort_digest_fallback(S, fallback):
    for case in M["semisort_digest"]:
        fam, par, n, bits = case["gen"]
        keys, vals = gen_keys_values(fam, par, n, bits, seed=1)
        if case["hash_ranks"]:
            keys = O.mix64_np(keys - np.uint64(1))
        data = S.RecordArray(keys, np.arange(n, dtype=keys.dtype))
        tel = S.Telemetry()
        S.semisort(data, S.UIntKeyAdapter(identity=case["identity"]), case["mode"],
                   S.TuningParams.for_input(n, **case["params"]), telemetry=tel)
        assert sha(data.keys_host(), data.values_host()) == case["out_sha"], case["name"]
        _tel_eq(tel, case["telemetry"])


@pytest.mark.parametrize("dist", ["uniform", "zipf", "few"])
def test_semisort_vs_oracle_4m_fallback(S, fallback, dist):
    rng = np.random.default_rng(42)
    n = 1 << 22
    if dist == "uniform":
        keys = rng.integers(0, 1 << 22, n).astype(np.uint64)
    elif dist == "zipf":
        keys = O.mix64_np(np.minimum(rng.zipf(1.3, n), 10**7).astype(np.uint64))
    else:
        keys = rng.integers(0, 300, n).astype(np.uint64)
    vals = np.arange(n, dtype=np.uint64)
    ko, vo, _ = O.semisort(keys, vals, O.OracleParams.derive(n))
    data = S.RecordArray(keys, vals)
    S.semisort(data, S.UIntKeyAdapter(), "eq", S.TuningParams.for_input(n))
    assert np.array_equal(data.values_host(), vo) and np.array_equal(data.keys_host(), ko)


def test_aggregates_fallback(S, fallback):
    for case in M["aggregate"]:
        p = f"ag_{case['name']}_"
        keys, vals = G[p + "keys"], G[p + "vals"]
        P = S.TuningParams.for_input(len(keys), **case["params"])
        adp = S.UIntKeyAdapter(identity=case["identity"])
        data = S.RecordArray(keys, vals)
        for spec, kind in ((S.ReduceSpec.counting(), "count"), (S.ReduceSpec.summing64(), "sum64")):
            k, v = S.collect_reduce(data, adp, spec, P).to_numpy()
            assert dict(zip(k.tolist(), v.tolist())) == O.reduce_by_key(keys, vals, kind), case["name"]
    rng = np.random.default_rng(8)
    n = 2_000_000
    keys = np.floor(rng.exponential(1e3, n)).astype(np.uint64)
    vals = rng.integers(0, 2**63, n).astype(np.uint64)
    k, v = S.collect_reduce(S.RecordArray(keys, vals), S.UIntKeyAdapter(), S.ReduceSpec.summing64()).to_numpy()
    assert dict(zip(k.tolist(), v.tolist())) == O.reduce_by_key(keys, vals, "sum64")
    k32 = rng.integers(0, 10**6, n).astype(np.uint32)
    k, v = S.histogram(S.RecordArray(k32), S.UIntKeyAdapter()).to_numpy()
    assert dict(zip(k.tolist(), v.tolist())) == O.reduce_by_key(k32, None, "count")
