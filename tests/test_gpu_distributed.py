"""The multi-GPU data path on one GPU (GPU tier): the device stable hash
partition (ss_partition) against its numpy statement, and the whole
partition -> source-ordered exchange -> local semisort / reduce pipeline
for G = 2, 4, 8 shards with the exchange done on the host (no cross-rank
waits on one device).  The NCCL orchestration itself is covered over gloo
(test_distributed_gloo.py)."""
import numpy as np
import pytest
import torch

import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def S():
    import paper_2304_10078_b200 as S
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    return S


def _np_partition(keys, parts):
    bits = parts.bit_length() - 1
    dest = (O.mix64_np(keys.astype(np.uint64)) >> np.uint64(64 - bits)).astype(np.int64) if bits else \
        np.zeros(len(keys), np.int64)
    return np.argsort(dest, kind="stable"), np.bincount(dest, minlength=parts)


@pytest.mark.parametrize("parts", [1, 2, 4, 8])
@pytest.mark.parametrize("kdt", [np.uint32, np.uint64])
def test_device_partition_matches_numpy(S, parts, kdt):
    from paper_2304_10078_b200.distributed import device_partition
    rng = np.random.default_rng(parts)
    n = 1_000_003
    keys = rng.integers(0, 2**63, n).astype(np.uint64)
    keys[: n // 3] = keys[: n // 3] % 1000   # repeated keys
    keys = keys.astype(kdt)
    vals = np.arange(n, dtype=np.uint64)
    out, counts = device_partition(S.RecordArray(keys, vals), parts)
    order, ref_counts = _np_partition(keys, parts)
    assert counts == ref_counts.tolist()
    assert np.array_equal(out.keys_host(), keys[order]) and np.array_equal(out.values_host(), vals[order])


@pytest.mark.parametrize("G", [2, 4, 8])
def test_sharded_semisort_pipeline(S, G):
    """Rank-ordered concatenation of the per-rank outputs is a valid stable
    global semisort, every key on the rank its hash names."""
    from paper_2304_10078_b200.distributed import device_partition
    rng = np.random.default_rng(G)
    n = 1 << 21
    # c5-style mix: half uniform 64-bit, half Zipf(0.8)-ish over a small universe
    keys = np.where(rng.random(n) < 0.5, rng.integers(0, 2**63, n).astype(np.uint64),
                    np.minimum(rng.zipf(1.3, n), 10**6).astype(np.uint64))
    vals = np.arange(n, dtype=np.uint64)
    shards = np.array_split(np.arange(n), G)
    sent = []
    for idx in shards:
        out, counts = device_partition(S.RecordArray(keys[idx], vals[idx]), G)
        k, v = out.keys_host(), out.values_host()
        bounds = np.concatenate([[0], np.cumsum(counts)])
        sent.append([(k[bounds[r]:bounds[r + 1]], v[bounds[r]:bounds[r + 1]]) for r in range(G)])
    outk, outv = [], []
    for r in range(G):   # receive in source-rank order, then the local semisort
        rk = np.concatenate([sent[s][r][0] for s in range(G)])
        rv = np.concatenate([sent[s][r][1] for s in range(G)])
        if len(rk) == 0:
            continue
        d = S.RecordArray(rk, rv)
        S.semisort(d, S.UIntKeyAdapter(), "eq", S.TuningParams.for_input(len(rk)))
        ok, ov = d.keys_host(), d.values_host()
        dest = (O.mix64_np(ok) >> np.uint64(64 - (G.bit_length() - 1))).astype(np.int64)
        assert (dest == r).all()
        outk.append(ok)
        outv.append(ov)
    gk, gv = np.concatenate(outk), np.concatenate(outv)
    rep = S.validate_semisort(S.RecordArray(keys, vals), S.RecordArray(gk, gv))
    assert rep.valid, rep


@pytest.mark.parametrize("G", [2, 4])
def test_sharded_histogram_pipeline(S, G):
    """Local reduce, partition of the partial pairs, source-ordered exchange,
    merge: per-key counts equal the global ones, each key on one rank."""
    from paper_2304_10078_b200.distributed import device_partition
    rng = np.random.default_rng(40 + G)
    n = 1 << 20
    keys = rng.integers(0, 50000, n).astype(np.uint64)
    shards = np.array_split(keys, G)
    sent = []
    for sk in shards:
        res = S.histogram(S.RecordArray(sk), S.UIntKeyAdapter())
        k, a = res.to_numpy()
        out, counts = device_partition(S.RecordArray(k.astype(np.uint64), a.astype(np.uint64)), G)
        kk, aa = out.keys_host(), out.values_host()
        b = np.concatenate([[0], np.cumsum(counts)])
        sent.append([(kk[b[r]:b[r + 1]], aa[b[r]:b[r + 1]]) for r in range(G)])
    total = {}
    for r in range(G):
        rk = np.concatenate([sent[s][r][0] for s in range(G)])
        ra = np.concatenate([sent[s][r][1] for s in range(G)])
        res = S.collect_reduce(S.RecordArray(rk, ra), S.UIntKeyAdapter(), S.ReduceSpec.summing64())
        k, a = res.to_numpy()
        for kk, aa in zip(k.tolist(), a.tolist()):
            assert kk not in total
            total[kk] = aa
    assert total == O.reduce_by_key(keys, None, "count")
