"""Multi-GPU semisort / collect-reduce / histogram (one process per GPU).

SURVEY.md §8(e).  Each rank holds a shard of the input.  Semisort:
1. stable partition of the local records by dest = top log2(G) bits of
   mix64(key) (device kernel ``ss_partition``; always hashed, so identity
   keys spread too; bits 60-63 are never used by level-0 light ids);
2. exchange the per-destination counts (G x G all_to_all);
3. all_to_all_v of keys and values over NCCL (NVLink / NVSwitch), received
   in source-rank order;
4. local semisort of what arrived.
Every key lives on exactly one rank, sources are input-ordered and the
partition is stable, so the concatenation of rank outputs in rank order is
a valid stable global semisort.  Output size per rank differs from its
input size, hence a new shard is returned (not in place).

collect-reduce / histogram reduce locally first, then exchange only the
(key, partial) pairs and merge them with a wrapping-sum reduce.

The exchange is the one collective; there is no other data-path
communication.  ``partitioner`` / ``local_sort`` / ``local_reduce`` hooks
exist so the host orchestration can be exercised with CPU tensors over
gloo in tests; the product path uses the device kernels.
"""

from __future__ import annotations

import ctypes as C

import torch
import torch.distributed as dist

from . import _lib
from .adapters import KeyAdapter, UIntKeyAdapter
from .aggregate import KeyedResult, ReduceSpec, collect_reduce
from .core import Telemetry, _layout, _ptr, _stream, _workspace, semisort
from .params import TuningParams
from .records import RecordArray, signed_view


def device_partition(data: RecordArray, parts: int):
    """(grouped RecordArray, counts list) via the stable device partition."""
    kb, vb = _layout(data)
    n = len(data)
    dev = data.device
    out = data.empty_like()
    lib = _lib.lib()
    ws = _workspace(lib.ss_partition_workspace_bytes(n, parts), dev)
    counts = (C.c_uint64 * parts)()
    _lib.check(lib.ss_partition(data.keys.data_ptr(), _ptr(data.values), n, kb, vb, parts, out.keys.data_ptr(),
                                _ptr(out.values), counts, ws.data_ptr(), ws.numel(), _stream(dev)))
    return out, [int(c) for c in counts]


def _exchange(cols, send_counts, group, device):
    """all_to_all_v of each column; returns received columns and counts."""
    world = dist.get_world_size(group)
    sc = torch.tensor(send_counts, dtype=torch.int64, device=device)
    rc = torch.empty(world, dtype=torch.int64, device=device)
    dist.all_to_all_single(rc, sc, group=group)
    recv_counts = [int(x) for x in rc.cpu().tolist()]
    total = sum(recv_counts)
    out = []
    for col in cols:
        if col is None:
            out.append(None)
            continue
        src = signed_view(col)
        dst = torch.empty((total,) + tuple(col.shape[1:]), dtype=src.dtype, device=device)
        dist.all_to_all_single(dst, src, output_split_sizes=recv_counts, input_split_sizes=send_counts, group=group)
        out.append(dst.view(col.dtype))
    return out, recv_counts


def dist_semisort(data: RecordArray, adapter: KeyAdapter | None = None, mode: str = "eq",
                  params_factory=None, *, group=None, telemetry: Telemetry | None = None,
                  partitioner=None, local_sort=None) -> RecordArray:
    """Globally semisort the union of all ranks' shards; returns this rank's
    output shard (keys with dest == rank, in stable order)."""
    adapter = adapter or UIntKeyAdapter()
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    make = params_factory or TuningParams.for_input
    sort = local_sort or (lambda d, p: semisort(d, adapter, mode, p, telemetry=telemetry))
    if world == 1:
        sort(data, make(len(data)))
        return data
    part = partitioner or device_partition
    grouped, counts = part(data, world)
    (keys, vals), _ = _exchange([grouped.keys, grouped.values], counts, group, data.device)
    out = RecordArray.__new__(RecordArray)
    out.keys, out.values, out.arena, out.key_kind = keys, vals, None, data.key_kind
    sort(out, make(len(out)))
    return out


def dist_collect_reduce(data: RecordArray, adapter: KeyAdapter | None, spec: ReduceSpec, params_factory=None, *,
                        group=None, partitioner=None, local_reduce=None) -> KeyedResult:
    """Reduce locally, exchange partial pairs by key hash, merge by sum."""
    adapter = adapter or UIntKeyAdapter()
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    make = params_factory or TuningParams.for_input
    red = local_reduce or (lambda d, s, p: collect_reduce(d, adapter, s, p))
    local = red(data, spec, make(len(data)))
    if world == 1:
        return local
    partials = RecordArray.__new__(RecordArray)
    partials.keys, partials.values, partials.arena = local.key_tensor, local.agg_tensor, None
    partials.key_kind = data.key_kind
    part = partitioner or device_partition
    grouped, counts = part(partials, world)
    (keys, aggs), _ = _exchange([grouped.keys, grouped.values], counts, group, data.device)
    merged = RecordArray.__new__(RecordArray)
    merged.keys, merged.values, merged.arena, merged.key_kind = keys, aggs, None, data.key_kind
    # partial counts and partial sums both merge by wrapping uint64 addition
    return red(merged, ReduceSpec.summing64(), make(len(merged)))


def dist_histogram(data: RecordArray, adapter: KeyAdapter | None = None, params_factory=None, *, group=None,
                   partitioner=None, local_reduce=None) -> KeyedResult:
    return dist_collect_reduce(data, adapter, ReduceSpec.counting(), params_factory, group=group,
                               partitioner=partitioner, local_reduce=local_reduce)
