"""Drop-in collect-reduce / histogram (the reference's aggregate.py) on the GPU.

The two vectorised monoids of the reference run on the device:
``ReduceSpec.counting()`` (histogram) and ``ReduceSpec.summing64()``
(wrapping uint64 sum of the first value word), aggregate.py:62-79.  A spec
with an arbitrary Python map/combine cannot execute on the device and
raises ContractError (the reference's generic branch, aggregate.py:219-237
and :256-264, is outside the GPU hot path).  The input is never modified.
Results come back as a ``KeyedResult`` holding device tensors; ``pairs``
materialises the Python list on demand.
"""

from __future__ import annotations

import csv
import ctypes as C
from dataclasses import dataclass
from typing import Callable

import numpy as np
import torch

from . import _lib
from .adapters import BytesKeyAdapter, KeyAdapter, UInt128KeyAdapter, device_identity_flag
from .core import Telemetry, _check_params, _layout, _ptr, _stream, _workspace
from .errors import ConfigurationError, ContractError
from .params import TuningParams
from .records import RecordArray, signed_view

U64_MASK = (1 << 64) - 1
_VECTOR_KINDS = (None, "count", "sum64")


@dataclass(frozen=True)
class ReduceSpec:
    """Map function + associative monoid (aggregate.py:42-79)."""

    map_record: Callable
    combine: Callable
    identity: object
    vector_kind: str | None = None

    def __post_init__(self):
        if self.vector_kind not in _VECTOR_KINDS:
            raise ConfigurationError(f"unknown vector_kind {self.vector_kind!r}")

    @staticmethod
    def counting() -> "ReduceSpec":
        return ReduceSpec(lambda key, value: 1, lambda a, b: a + b, 0, "count")

    @staticmethod
    def summing64() -> "ReduceSpec":
        def map_record(key, value):
            if value is None:
                raise ConfigurationError("summing64 needs a value column")
            scalar = value[0] if isinstance(value, tuple) else value
            return scalar & U64_MASK

        return ReduceSpec(map_record, lambda a, b: (a + b) & U64_MASK, 0, "sum64")


def format_key(key) -> str:
    if isinstance(key, tuple):
        lo, hi = key
        return str((hi << 64) | lo)
    if isinstance(key, bytes):
        return key.decode("latin-1")
    return str(key)


class KeyedResult:
    """Distinct (key, aggregate) pairs (aggregate.py:82-110).

    Built either from a Python list (reference-compatible) or from device
    tensors ``key_tensor`` / ``agg_tensor`` (the GPU result); ``pairs`` is
    materialised lazily from the tensors.
    """

    __slots__ = ("_pairs", "key_tensor", "agg_tensor", "arena")

    def __init__(self, pairs: list | None = None, *, key_tensor=None, agg_tensor=None, arena=None):
        self._pairs = pairs
        self.key_tensor = key_tensor
        self.agg_tensor = agg_tensor
        self.arena = arena   # byte-view keys: key_tensor holds (offset, length) views into it

    @property
    def pairs(self) -> list:
        if self._pairs is None:
            if self.key_tensor is None:
                self._pairs = []
            else:
                ks = self.key_tensor.cpu().numpy().tolist()
                if self.arena is not None:   # byte-view keys: the content bytes (adapters.py:216-218)
                    buf = self.arena.cpu().numpy().tobytes()
                    ks = [buf[o:o + n] for o, n in ks]
                elif self.key_tensor.dim() == 2:   # 128-bit keys: (lo, hi) tuples like the reference's canonical
                    ks = [tuple(k) for k in ks]
                ag = self.agg_tensor.cpu().numpy().tolist()
                self._pairs = list(zip(ks, ag))
        return self._pairs

    def __len__(self) -> int:
        if self._pairs is None and self.key_tensor is not None:
            return int(self.key_tensor.shape[0])
        return len(self.pairs)

    def __iter__(self):
        return iter(self.pairs)

    def __eq__(self, other) -> bool:
        if not isinstance(other, KeyedResult):
            return False
        if self.key_tensor is not None and other.key_tensor is not None and self._pairs is None \
                and other._pairs is None and self.arena is None and other.arena is None:
            return self.key_tensor.shape == other.key_tensor.shape and \
                self.key_tensor.dtype == other.key_tensor.dtype and \
                torch.equal(signed_view(self.key_tensor), signed_view(other.key_tensor.to(self.key_tensor.device))) \
                and torch.equal(signed_view(self.agg_tensor), signed_view(other.agg_tensor.to(self.agg_tensor.device)))
        return self.pairs == other.pairs

    def keys(self) -> list:
        return [k for k, _ in self.pairs]

    def aggregates(self) -> list:
        return [v for _, v in self.pairs]

    def to_numpy(self):
        """(keys, aggregates) as host arrays without building Python tuples."""
        if self.key_tensor is None:
            arr = np.array(self.pairs, dtype=np.uint64).reshape(-1, 2)
            return arr[:, 0], arr[:, 1]
        return self.key_tensor.cpu().numpy(), self.agg_tensor.cpu().numpy()

    def write_csv(self, fh, key_formatter=None) -> None:
        writer = csv.writer(fh)
        writer.writerow(["key", "aggregate"])
        fmt = key_formatter or format_key
        for key, value in self.pairs:
            writer.writerow([fmt(key), format_key(value)])


def _device_kind(spec: ReduceSpec) -> int:
    if spec.vector_kind == "count":
        return _lib.SS_AGG_COUNT
    if spec.vector_kind == "sum64":
        return _lib.SS_AGG_SUM64
    raise ContractError("only ReduceSpec.counting() and ReduceSpec.summing64() run on the GPU path")


def collect_reduce(data: RecordArray, adapter: KeyAdapter, spec: ReduceSpec, params: TuningParams | None = None,
                   *, workers: int | None = None, telemetry: Telemetry | None = None) -> KeyedResult:
    """Per-key count / wrapping-sum of ``data`` (aggregate.py:267-290)."""
    if getattr(data, "key_kind", None) == "bytes" or isinstance(adapter, BytesKeyAdapter):
        return _collect_reduce_bytes(data, adapter, spec, params, telemetry)
    ident = device_identity_flag(adapter, allow_u128=True)
    kind = _device_kind(spec)
    kb, vb = _layout(data, allow_u128=True)
    if (kb == 16) != (data.key_kind == "u128") or (kb == 16) != (adapter.key_kind == "u128"):
        raise ContractError(f"{type(adapter).__name__} does not match {data.key_kind} keys")
    n = len(data)
    params = _check_params(params, n)
    if kind == _lib.SS_AGG_SUM64 and data.values is None and n:
        raise ConfigurationError("summing64 needs a value column")
    tel = telemetry if telemetry is not None else Telemetry()
    dev = data.device
    vals = data.values if kind == _lib.SS_AGG_SUM64 else None
    vbytes = vb if kind == _lib.SS_AGG_SUM64 else 0
    pc = params.as_c()
    lib = _lib.lib()
    wsb = lib.ss_aggregate_workspace_bytes(n, kb, vbytes, C.byref(pc))
    if wsb == 0:
        _lib.check(_lib.SS_ERR_CONFIG)
    ws = _workspace(wsb, dev)
    count = C.c_uint64(0)
    ct = tel._c()
    _lib.check(lib.ss_collect_reduce(data.keys.data_ptr(), _ptr(vals), n, kb, vbytes, kind, ident, C.byref(pc),
                                     ws.data_ptr(), ws.numel(), C.byref(count), C.byref(ct), _stream(dev)))
    tel._absorb(ct)
    m = count.value
    keys = torch.empty((m, 2) if kb == 16 else (m,), dtype=data.keys.dtype, device=dev)
    aggs = torch.empty(m, dtype=torch.uint64, device=dev)
    if m:
        _lib.check(lib.ss_result_copy(ws.data_ptr(), n, kb, vbytes, C.byref(pc), keys.data_ptr(), aggs.data_ptr(),
                                      m, _stream(dev)))
    return KeyedResult(key_tensor=keys, agg_tensor=aggs)


def _collect_reduce_bytes(data, adapter, spec, params, telemetry) -> KeyedResult:
    """Byte-view keys (adapters.py:200-275): aggregation of 128-bit identity
    keys (content hash, length), then one representative view per distinct
    content, byte-checked against every record of its group (bytes_keys.py).
    Result keys are the content bytes, as the reference's canonical()."""
    from . import bytes_keys
    if not isinstance(adapter, BytesKeyAdapter) or getattr(data, "key_kind", None) != "bytes":
        raise ContractError(f"{type(adapter).__name__} does not match {getattr(data, 'key_kind', None)} keys")
    syn = bytes_keys.synthetic_keys(data, "eq")
    res = collect_reduce(RecordArray(syn, data.values, "u128"), UInt128KeyAdapter(identity=True), spec, params,
                         telemetry=telemetry)
    views = bytes_keys.representatives(data, syn, res.key_tensor)
    return KeyedResult(key_tensor=views, agg_tensor=res.agg_tensor, arena=data.arena)


def histogram(data: RecordArray, adapter: KeyAdapter, params: TuningParams | None = None, *,
              workers: int | None = None, telemetry: Telemetry | None = None) -> KeyedResult:
    """One (key, multiplicity) pair per distinct key (aggregate.py:293-299)."""
    return collect_reduce(data, adapter, ReduceSpec.counting(), params, workers=workers, telemetry=telemetry)
