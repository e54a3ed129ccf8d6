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


# ---- packed exchange path (ss_partition_pairs / ss_semisort_pairs) --------

@pytest.mark.parametrize("parts", [1, 2, 8])
@pytest.mark.parametrize("kdt", [np.uint32, np.uint64])
def test_pack_partition_matches_numpy(S, parts, kdt):
    from paper_2304_10078_b200.distributed import device_pack_partition
    rng = np.random.default_rng(10 + parts)
    n = 700_001
    keys = (rng.integers(0, 2**63, n) % (1000 if parts == 2 else 2**62)).astype(kdt)
    vals = rng.integers(0, 2**31, n).astype(kdt)
    words, counts = device_pack_partition(S.RecordArray(keys, vals), parts)
    order, ref_counts = _np_partition(keys, parts)
    w = words.cpu().numpy()
    assert counts == ref_counts.tolist()
    assert np.array_equal(w[0::2], keys[order]) and np.array_equal(w[1::2], vals[order])


@pytest.mark.parametrize("n", [0, 1, 5000, 16383, 16384, 300_000, 1 << 21])
@pytest.mark.parametrize("kdt", [np.uint32, np.uint64])
@pytest.mark.parametrize("mode", ["eq", "lt"])
def test_semisort_packed_equals_semisort(S, n, kdt, mode):
    """Semisort from packed records leaves the SoA result in the same memory,
    byte-identical to semisort of the unpacked columns (and the oracle)."""
    from paper_2304_10078_b200.core import semisort_packed
    rng = np.random.default_rng(n)
    keys = np.where(rng.random(n) < 0.5, rng.integers(0, 2**31, n), rng.zipf(1.2, n) % 5000).astype(kdt)
    vals = np.arange(n, dtype=kdt)
    ref = S.RecordArray(keys, vals)
    t_ref, t_p = S.Telemetry(), S.Telemetry()
    S.semisort(ref, S.UIntKeyAdapter(), mode, telemetry=t_ref)
    words = np.empty(2 * n, dtype=kdt)
    words[0::2], words[1::2] = keys, vals
    dw = torch.from_numpy(words).cuda()
    for scratch in (None, torch.empty(2 * n + 8, dtype=dw.dtype, device="cuda")):
        dw.copy_(torch.from_numpy(words))
        out = semisort_packed(dw, n, S.UIntKeyAdapter(), mode, scratch=scratch, telemetry=t_p)
        assert np.array_equal(out.keys_host(), ref.keys_host()) and np.array_equal(out.values_host(), ref.values_host())
        assert out.keys.data_ptr() == dw.data_ptr()
    assert t_p.nodes == 2 * t_ref.nodes and t_p.bucket_assignments == 2 * t_ref.bucket_assignments
    if n and n < 1 << 20:
        ko, vo, _ = O.semisort(keys, vals, O.OracleParams.derive(n), mode)
        assert np.array_equal(ref.keys_host(), ko) and np.array_equal(ref.values_host(), vo)


def test_semisort_packed_errors(S):
    from paper_2304_10078_b200.core import semisort_packed
    w = torch.zeros(10, dtype=torch.uint64, device="cuda")
    with pytest.raises(S.ConfigurationError):
        semisort_packed(w, 6, S.UIntKeyAdapter())
    with pytest.raises(S.ConfigurationError):
        semisort_packed(w, 5, S.UIntKeyAdapter(), "zz")
    with pytest.raises(S.ContractError):
        semisort_packed(w.to(torch.int64), 5, S.UIntKeyAdapter())


def test_nccl_c_abi_pipeline_world_one(S):
    """ss_dist_semisort through a one-rank NCCL communicator (partition,
    count exchange and packed all-to-allv to self, semisort from the packed
    receive buffer) equals semisort; a too-small capacity fails before the
    payload exchange with the input intact."""
    import os
    import torch.distributed as dist
    from paper_2304_10078_b200.distributed import NcclSemisort
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29531")
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        ds = NcclSemisort()
        rng = np.random.default_rng(3)
        n = 1_000_000
        keys = np.where(rng.random(n) < 0.5, rng.integers(0, 2**63, n), rng.zipf(1.1, n) % 10**5).astype(np.uint64)
        vals = np.arange(n, dtype=np.uint64)
        ref = S.RecordArray(keys, vals)
        S.semisort(ref, S.UIntKeyAdapter())
        cap = n + 4096
        blk = torch.empty(2 * cap, dtype=torch.uint64, device="cuda")
        scr = torch.empty(2 * cap, dtype=torch.uint64, device="cuda")
        data = S.core._raw(blk[:n], blk[cap:cap + n], "u64")   # the input lives in the receive block
        data.keys.copy_(torch.from_numpy(keys))
        data.values.copy_(torch.from_numpy(vals))
        out = ds(data, recv_block=blk, scratch=scr, capacity=cap, params_template=S.TuningParams.for_input(n))
        assert len(out) == n
        assert np.array_equal(out.keys_host(), ref.keys_host()) and np.array_equal(out.values_host(), ref.values_host())
        # a shard larger than the buffers' capacity is refused before any work
        small = S.RecordArray(keys[:5000], vals[:5000])
        b2 = torch.empty(2 * 5000, dtype=torch.uint64, device="cuda")
        s2 = torch.empty(2 * 5000, dtype=torch.uint64, device="cuda")
        with pytest.raises(S.ConfigurationError):
            ds(small, recv_block=b2, scratch=s2, capacity=4000)
        assert np.array_equal(small.keys_host(), keys[:5000])
        ds.close()
    finally:
        dist.destroy_process_group()


def test_validate_shard_and_fingerprints(S):
    """ss_validate_shard on a semisorted generated c5 shard: records intact,
    stable, contiguous; fingerprints equal those of the index range; a
    corrupted record and a swapped pair are caught."""
    import ctypes as C
    from paper_2304_10078_b200 import _lib
    from paper_2304_10078_b200.core import _stream, _workspace
    from paper_2304_10078_b200.datagen import generate_device
    from paper_2304_10078_b200.validate import count_distinct
    n, first = 1 << 20, 12345
    d = generate_device("mix", 0.8, n, key_bits=64, seed=1, universe=10**8, values="index", first_index=first)
    S.semisort(d, S.UIntKeyAdapter())

    def check(out):
        res = (C.c_uint64 * 7)()
        ws = _workspace(4096, out.device)
        _lib.check(_lib.lib().ss_validate_shard(4, 0.8, 10**8, 1, 0, out.keys.data_ptr(), out.values.data_ptr(),
                                                len(out), 8, 1, 0, ws.data_ptr(), ws.numel(), res,
                                                _stream(out.device)))
        return [int(x) for x in res]

    r = check(d)
    fp = (C.c_uint64 * 3)()
    ws = _workspace(4096, d.device)
    _lib.check(_lib.lib().ss_index_fingerprint(first, first + n, ws.data_ptr(), ws.numel(), fp, _stream(d.device)))
    assert r[0] == 0 and r[2] == 0 and r[3] == 0 and r[1] == count_distinct(d.keys)
    assert r[4:7] == [int(x) for x in fp]
    bad = d.copy()
    kb = bad.keys.cpu().numpy()
    kb[7] ^= np.uint64(1)
    bad.keys.copy_(torch.from_numpy(kb))
    assert check(bad)[0] >= 1
    sw = d.copy()
    k = sw.keys.cpu().numpy()
    i = int(np.flatnonzero(k[1:] == k[:-1])[0])       # two records of one run: swap their values
    v = sw.values.cpu().numpy()
    v[i], v[i + 1] = v[i + 1], v[i]
    sw.values.copy_(torch.from_numpy(v))
    assert check(sw)[2] >= 1
