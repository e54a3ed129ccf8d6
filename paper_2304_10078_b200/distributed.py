"""Multi-GPU semisort / collect-reduce / histogram (one process per GPU).

SURVEY.md §8(e).  Each rank holds a shard of the input.  Semisort:
1. stable partition of the local records by dest = top log2(G) bits of
   mix64(key) (device kernel ``ss_partition_pairs``; always hashed, so
   identity keys spread too), written as packed (key, value) records;
2. exchange of the per-destination counts (G x G all_to_all);
3. ONE all_to_all_v of the packed records over NCCL (NVLink / NVSwitch),
   received in source-rank order;
4. local semisort of what arrived straight from the packed records
   (``ss_semisort_pairs``), finishing as SoA columns in the receive buffer,
   with the send buffer reused as its scratch.
Every key lives on exactly one rank, sources are input-ordered and the
partition is stable, so the concatenation of rank outputs in rank order is
a valid stable global semisort.  Output size per rank differs from its
input size, hence a new shard is returned (views of the receive buffer).

Buffer reuse (strong scaling): ``recv_block`` and ``scratch`` let the
caller provide both buffers; ``recv_block`` may be the memory of the input
columns themselves (the partition consumes them before anything arrives),
so a rank needs two record-sized buffers plus the workspace.

collect-reduce / histogram reduce locally first, then exchange only the
(key, partial) pairs (packed, one exchange) and merge them with a
wrapping-sum reduce.

``NcclSemisort`` drives the same pipeline through the C ABI
(``ss_dist_semisort`` over an NCCL communicator of the library's own): what
a non-Python caller of the library binds.

The ``pack`` / ``sort_packed`` / ``local_reduce`` hooks let the host
orchestration run with CPU tensors over gloo in tests; the product path
uses the device kernels.
"""

from __future__ import annotations

import ctypes as C

import torch
import torch.distributed as dist

from . import _lib
from .adapters import KeyAdapter, UIntKeyAdapter, device_identity_flag
from .aggregate import KeyedResult, ReduceSpec, collect_reduce
from .core import Telemetry, _layout, _ptr, _raw, _stream, _workspace, semisort, semisort_packed
from .errors import ConfigurationError
from .params import TuningParams
from .records import RecordArray, signed_view


def device_partition(data: RecordArray, parts: int):
    """(grouped RecordArray, counts list) via the stable device partition (SoA)."""
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


def packable(data: RecordArray) -> bool:
    """Records that travel as one packed (key, value) column."""
    return data.values is not None and data.key_kind in ("u32", "u64") and data.values.dim() == 1 and \
        data.values.dtype == data.keys.dtype


def device_pack_partition(data: RecordArray, parts: int, out: torch.Tensor | None = None):
    """(packed records [2n words], counts list): stable partition by dest."""
    n = len(data)
    dev = data.device
    if out is None or out.numel() < 2 * n:
        out = torch.empty(2 * n, dtype=data.keys.dtype, device=dev)
    lib = _lib.lib()
    ws = _workspace(lib.ss_partition_pairs_workspace_bytes(n, parts), dev)
    counts = (C.c_uint64 * parts)()
    _lib.check(lib.ss_partition_pairs(data.keys.data_ptr(), data.values.data_ptr(), n, data.keys.element_size(), parts,
                                      out.data_ptr(), counts, ws.data_ptr(), ws.numel(), _stream(dev)))
    return out, [int(c) for c in counts]


def _exchange_counts(send_counts, group, device):
    world = dist.get_world_size(group)
    sc = torch.tensor(send_counts, dtype=torch.int64, device=device)
    rc = torch.empty(world, dtype=torch.int64, device=device)
    dist.all_to_all_single(rc, sc, group=group)
    return [int(x) for x in rc.cpu().tolist()]


def _exchange(cols, send_counts, group, device):
    """all_to_all_v of each column; returns received columns and counts."""
    recv_counts = _exchange_counts(send_counts, group, device)
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


def _exchange_packed(send: torch.Tensor, send_counts, group, device, recv_block=None):
    """ONE all_to_all_v of packed (key, value) records: returns (recv words,
    received record count); the receive buffer is ``recv_block`` when it
    holds 2m words, else a new tensor."""
    recv_counts = _exchange_counts(send_counts, group, device)
    m, n = sum(recv_counts), sum(send_counts)
    if recv_block is not None and recv_block.numel() >= 2 * m and recv_block.dtype == send.dtype:
        recv = recv_block.reshape(-1)
    else:
        recv = torch.empty(2 * m, dtype=send.dtype, device=device)
    dist.all_to_all_single(signed_view(recv[:2 * m]).view(m, 2), signed_view(send[:2 * n]).view(n, 2),
                           output_split_sizes=recv_counts, input_split_sizes=send_counts, group=group)
    return recv, m


def dist_semisort(data: RecordArray, adapter: KeyAdapter | None = None, mode: str = "eq",
                  params_factory=None, *, group=None, telemetry: Telemetry | None = None,
                  recv_block: torch.Tensor | None = None, scratch: torch.Tensor | None = None,
                  pack=None, sort_packed=None, partitioner=None, local_sort=None) -> RecordArray:
    """Globally semisort the union of all ranks' shards; returns this rank's
    output shard (keys with dest == rank, in stable order).

    Records whose value column has the key's width travel packed (one
    exchange); others (no values, 128-bit values) take one exchange per
    column through ``device_partition``.  recv_block / scratch: optional
    caller buffers (>= 2 x the records this rank will receive / send, in
    words of the key dtype); recv_block may alias the input's memory."""
    adapter = adapter or UIntKeyAdapter()
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    make = params_factory or TuningParams.for_input
    if world == 1:
        sort = local_sort or (lambda d, p: semisort(d, adapter, mode, p, telemetry=telemetry))
        sort(data, make(len(data)))
        return data
    if partitioner is None and local_sort is None and (pack is not None or packable(data)):
        pk = pack or device_pack_partition
        srt = sort_packed or (lambda words, m, p, scr: semisort_packed(words, m, adapter, mode, p, scratch=scr,
                                                                       telemetry=telemetry))
        send, counts = pk(data, world) if scratch is None else pk(data, world, scratch)
        recv, m = _exchange_packed(send, counts, group, data.device, recv_block)
        scr = send if send.numel() >= 2 * m else None
        return srt(recv, m, make(m), scr)
    part = partitioner or device_partition
    sort = local_sort or (lambda d, p: semisort(d, adapter, mode, p, telemetry=telemetry))
    grouped, counts = part(data, world)
    (keys, vals), _ = _exchange([grouped.keys, grouped.values], counts, group, data.device)
    out = _raw(keys, vals, data.key_kind)
    sort(out, make(len(out)))
    return out


def dist_collect_reduce(data: RecordArray, adapter: KeyAdapter | None, spec: ReduceSpec, params_factory=None, *,
                        group=None, pack=None, partitioner=None, local_reduce=None) -> KeyedResult:
    """Reduce locally, exchange packed (key, partial) pairs by key hash in
    one all_to_all_v, merge by wrapping sum."""
    adapter = adapter or UIntKeyAdapter()
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    make = params_factory or TuningParams.for_input
    red = local_reduce or (lambda d, s, p: collect_reduce(d, adapter, s, p))
    local = red(data, spec, make(len(data)))
    if world == 1:
        return local
    kind = data.key_kind
    keys = local.key_tensor
    aggs = local.agg_tensor
    if keys.dtype != aggs.dtype:   # u32 keys: partial pairs travel as u64 words
        keys = (signed_view(keys).to(torch.int64) & 0xFFFFFFFF).view(torch.uint64)
    partials = _raw(keys, aggs, "u64")
    if partitioner is None:
        pk = pack or device_pack_partition
        send, counts = pk(partials, world)
        recv, m = _exchange_packed(send, counts, group, data.device)
        pairs = signed_view(recv[:2 * m]).view(m, 2)
        mk = pairs[:, 0].contiguous().view(torch.uint64)
        ma = pairs[:, 1].contiguous().view(torch.uint64)
    else:
        grouped, counts = partitioner(partials, world)
        (mk, ma), _ = _exchange([grouped.keys, grouped.values], counts, group, data.device)
    if kind == "u32":
        mk = signed_view(mk).to(torch.int32).view(torch.uint32)
    merged = _raw(mk, ma, kind)
    # partial counts and partial sums both merge by wrapping uint64 addition
    return red(merged, ReduceSpec.summing64(), make(len(merged)))


def dist_histogram(data: RecordArray, adapter: KeyAdapter | None = None, params_factory=None, *, group=None,
                   pack=None, partitioner=None, local_reduce=None) -> KeyedResult:
    return dist_collect_reduce(data, adapter, ReduceSpec.counting(), params_factory, group=group, pack=pack,
                               partitioner=partitioner, local_reduce=local_reduce)


class NcclSemisort:
    """The sharded semisort through the C ABI (``ss_dist_semisort``) over an
    NCCL communicator owned by the library (bootstrapped once through
    torch.distributed's object broadcast).  ``__call__`` returns this
    rank's output shard as views of ``recv_block``."""

    def __init__(self, group=None):
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        lib = _lib.lib()
        uid = C.create_string_buffer(128)
        if self.rank == 0:
            _lib.check(lib.ss_nccl_unique_id(uid))
        obj = [bytes(uid.raw) if self.rank == 0 else None]
        dist.broadcast_object_list(obj, src=0, group=group)
        self.comm = C.c_void_p()
        _lib.check(lib.ss_nccl_comm_init(C.create_string_buffer(obj[0], 128), self.world, self.rank,
                                         C.byref(self.comm)))

    def close(self):
        if self.comm:
            _lib.check(_lib.lib().ss_nccl_comm_destroy(self.comm))
            self.comm = C.c_void_p()

    def __call__(self, data: RecordArray, adapter: KeyAdapter | None = None, mode: str = "eq", *,
                 recv_block: torch.Tensor, scratch: torch.Tensor, capacity: int,
                 params_template: TuningParams | None = None, telemetry: Telemetry | None = None) -> RecordArray:
        adapter = adapter or UIntKeyAdapter()
        if not packable(data):
            raise ConfigurationError("ss_dist_semisort needs values of the key width")
        ident = device_identity_flag(adapter)
        n = len(data)
        kb = data.keys.element_size()
        if recv_block.numel() < 2 * capacity or scratch.numel() < 2 * capacity:
            raise ConfigurationError("recv_block and scratch must hold 2 x capacity words")
        tmpl = (params_template or TuningParams.for_input(capacity)).as_c()
        lib = _lib.lib()
        dev = data.device
        ws = _workspace(lib.ss_dist_semisort_workspace_bytes(capacity, kb, self.world, C.byref(tmpl)), dev)
        tel = telemetry if telemetry is not None else Telemetry()
        ct = tel._c()
        out_n = C.c_uint64(0)
        _lib.check(lib.ss_dist_semisort(self.comm, self.world, self.rank, data.keys.data_ptr(), data.values.data_ptr(),
                                        n, kb, _lib.SS_MODE_LT if mode == "lt" else _lib.SS_MODE_EQ, ident,
                                        C.byref(tmpl), recv_block.data_ptr(), scratch.data_ptr(), capacity,
                                        ws.data_ptr(), ws.numel(), C.byref(out_n), C.byref(ct), _stream(dev)))
        tel._absorb(ct)
        m = out_n.value
        flat = recv_block.reshape(-1)
        return _raw(flat[:m], flat[m:2 * m], data.key_kind)
