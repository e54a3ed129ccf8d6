"""Multi-rank orchestration of paper_2304_10078_b200.distributed over gloo
(world_size 2 and 4, CPU).  The device kernels are replaced by CPU stand-ins
(a stable numpy hash partition and the oracle) so the host logic — count
exchange, all_to_all_v in source-rank order, local sort / merge — is tested
here; the same code path drives NCCL on GPUs."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _ra(keys, vals, kind="u64"):
    from paper_2304_10078_b200.records import RecordArray
    r = RecordArray.__new__(RecordArray)
    r.keys, r.values, r.arena, r.key_kind = keys, vals, None, kind
    return r


def cpu_partition(data, parts):
    """Stable partition by dest = top bits of mix64(key) (ss_partition semantics)."""
    k = data.keys.numpy()
    bits = parts.bit_length() - 1
    dest = (O.mix64_np(k) >> np.uint64(64 - bits)).astype(np.int64) if bits else np.zeros(len(k), np.int64)
    order = np.argsort(dest, kind="stable")
    counts = np.bincount(dest, minlength=parts).tolist()
    vals = None if data.values is None else torch.from_numpy(data.values.numpy()[order].copy())
    return _ra(torch.from_numpy(k[order].copy()), vals, data.key_kind), counts


def cpu_sort(data, params):
    k, v = data.keys.numpy(), data.values.numpy()
    P = O.OracleParams.derive(len(k), base_case_cutoff=256)
    ko, vo, _ = O.semisort(k, v, P)
    data.keys.copy_(torch.from_numpy(ko))
    data.values.copy_(torch.from_numpy(vo))


def cpu_reduce(data, spec, params):
    from paper_2304_10078_b200.aggregate import KeyedResult
    kind = spec.vector_kind
    d = O.reduce_by_key(data.keys.numpy(), None if data.values is None else data.values.numpy(), kind)
    ks = np.array(list(d.keys()), dtype=np.uint64)
    vs = np.array(list(d.values()), dtype=np.uint64)
    return KeyedResult(key_tensor=torch.from_numpy(ks), agg_tensor=torch.from_numpy(vs))


def cpu_pack(data, parts, out=None):
    """ss_partition_pairs semantics: stable partition into packed (key, value) words."""
    grouped, counts = cpu_partition(data, parts)
    n = len(grouped.keys)
    words = torch.empty(2 * n, dtype=grouped.keys.dtype) if out is None else out
    w = words.numpy() if out is None else words.numpy()
    w[0:2 * n:2] = grouped.keys.numpy()
    w[1:2 * n:2] = grouped.values.numpy()
    return words, counts


def cpu_sort_packed(words, m, params, scratch):
    """ss_semisort_pairs semantics: semisort m packed records, leave SoA in place."""
    from paper_2304_10078_b200.core import _raw
    w = words.numpy()
    k, v = w[0:2 * m:2].copy(), w[1:2 * m:2].copy()
    P = O.OracleParams.derive(m, base_case_cutoff=256)
    ko, vo, _ = O.semisort(k, v, P)
    w[:m] = ko
    w[m:2 * m] = vo
    return _raw(words[:m], words[m:2 * m], "u64")


def _worker(rank, world, port, q, packed=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2304_10078_b200.distributed import dist_histogram, dist_semisort
        n_local = 3000 + 517 * rank            # uneven shards
        rng = np.random.default_rng(100 + rank)
        keys = np.where(rng.random(n_local) < 0.5, rng.integers(0, 2**63, n_local),
                        rng.zipf(1.3, n_local) % 500).astype(np.uint64)
        offset = sum(3000 + 517 * r for r in range(rank))
        vals = np.arange(offset, offset + n_local, dtype=np.uint64)
        data = _ra(torch.from_numpy(keys.copy()), torch.from_numpy(vals))
        if packed:   # one exchange of packed records, sort from the packed receive buffer
            out = dist_semisort(data, pack=cpu_pack, sort_packed=cpu_sort_packed)
            hist = dist_histogram(_ra(torch.from_numpy(keys.copy()), None), pack=cpu_pack, local_reduce=cpu_reduce)
        else:
            out = dist_semisort(data, partitioner=cpu_partition, local_sort=cpu_sort)
            hist = dist_histogram(_ra(torch.from_numpy(keys.copy()), None), partitioner=cpu_partition,
                                  local_reduce=cpu_reduce)
        gathered = [None] * world
        dist.all_gather_object(gathered, (keys, out.keys.numpy(), out.values.numpy(),
                                          hist.key_tensor.numpy(), hist.agg_tensor.numpy()))
        if rank == 0:
            q.put(gathered)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,packed", [(2, False), (4, False), (2, True), (4, True)])
def test_dist_semisort_and_histogram_gloo(world, packed):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, packed)) for r in range(world)]
    for p in procs:
        p.start()
    gathered = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    keys_in = np.concatenate([g[0] for g in gathered])
    ko = np.concatenate([g[1] for g in gathered])
    vo = np.concatenate([g[2] for g in gathered])
    # the concatenation of rank outputs is a stable global semisort
    assert O.semisort_valid_indexed(keys_in, ko, vo)
    bits = world.bit_length() - 1
    for r, g in enumerate(gathered):
        assert np.all((O.mix64_np(g[1]) >> np.uint64(64 - bits)) == r)   # dest(key) == rank
    # distributed histogram == global histogram
    hk = np.concatenate([g[3] for g in gathered])
    ha = np.concatenate([g[4] for g in gathered])
    assert len(np.unique(hk)) == len(hk)
    assert dict(zip(hk.tolist(), ha.tolist())) == O.reduce_by_key(keys_in, None, "count")
