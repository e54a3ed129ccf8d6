"""RecordArray on device memory (the reference's records.py:34-132).

Same SoA layout as the reference: a 1-D ``keys`` column (uint32 or uint64)
and an optional ``values`` column (uint32 / uint64, or (n, 2) uint64 for
128-bit payloads).  Columns are torch CUDA tensors; numpy arrays (or any
array-like) are copied to the device on construction, which is how host
data enters the drop-in path.  Views never copy.
"""

from __future__ import annotations

import os
import struct

import numpy as np
import torch

from .errors import InputFormatError

KEY_KINDS = ("u32", "u64", "u128", "bytes")
_KEY_WIDTH = {"u32": 32, "u64": 64, "u128": 128, "bytes": 128}

_NP2T = {np.dtype(np.uint32): torch.uint32, np.dtype(np.uint64): torch.uint64,
         np.dtype(np.int64): torch.uint64}


def signed_view(t: torch.Tensor) -> torch.Tensor:
    """Same bits as a signed tensor (torch implements few ops on uint32/uint64)."""
    if t.dtype == torch.uint64:
        return t.view(torch.int64)
    if t.dtype == torch.uint32:
        return t.view(torch.int32)
    return t


def default_device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2304_10078_b200 needs a CUDA device (B200); there is no CPU path")
    return torch.device("cuda", torch.cuda.current_device())


def as_device_column(a, dtype: torch.dtype | None = None, device=None) -> torch.Tensor:
    """A contiguous CUDA tensor for one column (copies host data in)."""
    if isinstance(a, torch.Tensor):
        t = a
        if dtype is not None and t.dtype != dtype:
            t = t.to(dtype)
        if not t.is_cuda:
            t = t.to(device or default_device())
        return t if t.is_contiguous() else t.contiguous()
    arr = np.asarray(a)
    if dtype is None:
        if arr.dtype == np.uint32:
            dtype = torch.uint32
        else:
            dtype = torch.uint64
    np_dt = {torch.uint32: np.uint32, torch.uint64: np.uint64}[dtype]
    arr = np.ascontiguousarray(arr.astype(np_dt, copy=False))
    return torch.from_numpy(arr).to(device or default_device())


def as_byte_arena(a, device) -> torch.Tensor:
    """A contiguous uint8 CUDA tensor for a byte arena (bytes / numpy / tensor)."""
    if isinstance(a, torch.Tensor):
        t = a if a.dtype == torch.uint8 else a.view(torch.uint8)
        return t.to(device).contiguous()
    if isinstance(a, (bytes, bytearray, memoryview)):
        a = np.frombuffer(bytes(a), dtype=np.uint8)
    arr = np.ascontiguousarray(np.asarray(a, dtype=np.uint8))
    return torch.from_numpy(arr.copy()).to(device)


class RecordArray:
    """Records (key, value) as device columns; mirrors records.py:34-132."""

    __slots__ = ("keys", "values", "arena", "key_kind")

    def __init__(self, keys, values=None, key_kind=None, arena=None):
        if key_kind == "bytes" or arena is not None:
            if key_kind not in (None, "bytes"):
                raise ValueError(f"an arena goes with byte-view keys, not {key_kind!r}")
            if arena is None:
                raise ValueError("bytes keys require an arena")
            key_kind = "bytes"
        if isinstance(keys, torch.Tensor):
            kt = keys
        else:
            arr = np.asarray(keys)
            if key_kind is None:
                key_kind = "u128" if arr.ndim == 2 else ("u32" if arr.dtype == np.uint32 else "u64")
            kt = as_device_column(arr, torch.uint32 if key_kind == "u32" else torch.uint64)
        if key_kind is None:
            key_kind = "u128" if kt.dim() == 2 else ("u32" if kt.dtype == torch.uint32 else "u64")
        if key_kind not in KEY_KINDS:
            raise ValueError(f"unknown key kind {key_kind!r}")
        if key_kind == "u32":
            kt = as_device_column(kt, torch.uint32)
        elif key_kind == "u64":
            kt = as_device_column(kt, torch.uint64)
        else:
            kt = as_device_column(kt, torch.uint64)
            if kt.dim() != 2 or kt.shape[1] != 2:
                raise ValueError(f"{key_kind} keys must have shape (n, 2)")
        vt = None
        if values is not None:
            if isinstance(values, torch.Tensor):
                vt = as_device_column(values, values.dtype if values.dtype in (torch.uint32, torch.uint64)
                                      else torch.uint64, kt.device)
            else:
                va = np.asarray(values)
                vt = as_device_column(va, torch.uint32 if va.dtype == np.uint32 else torch.uint64, kt.device)
            if vt.shape[0] != kt.shape[0]:
                raise ValueError("values length must match keys length")
        self.keys = kt
        self.values = vt
        # byte-view keys: (offset, length) rows into a shared, caller-owned
        # uint8 arena (records.py:11-13), kept on the device next to them
        self.arena = None if arena is None else as_byte_arena(arena, kt.device)
        self.key_kind = key_kind

    # -- shape & views --------------------------------------------------------
    def __len__(self) -> int:
        return int(self.keys.shape[0])

    @property
    def key_width(self) -> int:
        return _KEY_WIDTH[self.key_kind]

    @property
    def key_bytes(self) -> int:
        return self.keys.element_size() * (2 if self.key_kind in ("u128", "bytes") else 1)

    @property
    def value_bytes(self) -> int:
        if self.values is None:
            return 0
        return self.values.element_size() * (self.values.shape[1] if self.values.dim() == 2 else 1)

    @property
    def device(self) -> torch.device:
        return self.keys.device

    def view(self, lo: int, hi: int) -> "RecordArray":
        out = RecordArray.__new__(RecordArray)
        out.keys = self.keys[lo:hi]
        out.values = None if self.values is None else self.values[lo:hi]
        out.arena = self.arena
        out.key_kind = self.key_kind
        return out

    def _wrap(self, keys, values) -> "RecordArray":
        out = RecordArray.__new__(RecordArray)
        out.keys, out.values, out.arena, out.key_kind = keys, values, self.arena, self.key_kind
        return out

    def copy(self) -> "RecordArray":
        return self._wrap(self.keys.clone(), None if self.values is None else self.values.clone())

    def empty_like(self, n: int | None = None) -> "RecordArray":
        n = len(self) if n is None else n
        keys = torch.empty((n,) + tuple(self.keys.shape[1:]), dtype=self.keys.dtype, device=self.device)
        values = None
        if self.values is not None:
            values = torch.empty((n,) + tuple(self.values.shape[1:]), dtype=self.values.dtype, device=self.device)
        return self._wrap(keys, values)

    def gather(self, idx) -> "RecordArray":
        idx = torch.as_tensor(np.asarray(idx) if not isinstance(idx, torch.Tensor) else idx,
                              device=self.device).to(torch.int64)
        keys = signed_view(self.keys)[idx].view(self.keys.dtype)
        values = None if self.values is None else signed_view(self.values)[idx].view(self.values.dtype)
        return self._wrap(keys, values)

    def value_at(self, i: int):
        if self.values is None:
            return None
        row = self.values[i].cpu().numpy()
        return tuple(int(x) for x in row) if row.ndim else int(row)

    # -- host views (for checking; copies device -> host) ----------------------
    def keys_host(self) -> np.ndarray:
        return self.keys.cpu().numpy()

    def values_host(self):
        return None if self.values is None else self.values.cpu().numpy()

    def row_bytes(self) -> np.ndarray:
        n = len(self)
        parts = [np.ascontiguousarray(self.keys_host()).view(np.uint8).reshape(n, -1)]
        if self.values is not None:
            parts.append(np.ascontiguousarray(self.values_host()).view(np.uint8).reshape(n, -1))
        return parts[0] if len(parts) == 1 else np.hstack(parts)

    def same_bytes(self, other: "RecordArray") -> bool:
        if len(self) != len(other) or self.key_kind != other.key_kind:
            return False
        if self.keys.dtype != other.keys.dtype:
            return False
        if not torch.equal(signed_view(self.keys), signed_view(other.keys.to(self.device))):
            return False
        if (self.values is None) != (other.values is None):
            return False
        if self.values is None:
            return True
        return self.values.dtype == other.values.dtype and torch.equal(
            signed_view(self.values), signed_view(other.values.to(self.device)))


# -- binary record dump (records.py:149-202) ----------------------------------
# 16-byte header: magic "SSR1", key_width u16, value_width u16, n u64 (little
# endian); then n packed rows, key bytes first.  The payload moves between the
# file and HBM untouched (one pinned staging buffer, one copy each way); the
# row <-> column split runs on the device (ss_records_unpack / _pack).

DUMP_MAGIC = b"SSR1"
_HEADER = struct.Struct("<HHQ")


def _payload_stage(nbytes: int) -> torch.Tensor:
    t = torch.empty(max(nbytes, 1), dtype=torch.uint8)
    return t.pin_memory() if torch.cuda.is_available() else t


def write_records(path, data: "RecordArray") -> None:
    """records.py:152-169: same header and row bytes as the reference."""
    from . import _lib
    if data.key_kind == "bytes":
        raise InputFormatError("byte-view records cannot be dumped (arena-backed)")
    n = len(data)
    kb = data.key_bytes
    vb = data.value_bytes
    header = DUMP_MAGIC + _HEADER.pack(data.key_width, vb * 8, n)
    row = kb + vb
    dev = data.device
    stage = _payload_stage(n * row)
    if n:
        rows = torch.empty(n * row, dtype=torch.uint8, device=dev)
        st = torch.cuda.current_stream(dev).cuda_stream
        _lib.check(_lib.lib().ss_records_pack(data.keys.data_ptr(),
                                              None if data.values is None else data.values.data_ptr(),
                                              n, kb, vb, rows.data_ptr(), st))
        stage[: n * row].copy_(rows)
    with open(path, "wb") as fh:
        fh.write(header)
        if n:
            fh.write(memoryview(stage[: n * row].numpy()))


def read_records(path, device=None) -> "RecordArray":
    """records.py:172-202: same checks and errors; columns land on the GPU."""
    from . import _lib
    with open(path, "rb") as fh:
        header = fh.read(16)
        if len(header) != 16 or header[:4] != DUMP_MAGIC:
            raise InputFormatError(f"{path}: not a record dump")
        key_width, value_width, n = _HEADER.unpack(header[4:])
        row = (key_width + value_width) // 8
        size = os.fstat(fh.fileno()).st_size - 16
        if key_width not in (32, 64, 128) or size != n * row:
            raise InputFormatError(f"{path}: corrupt record dump header")
        if value_width not in (0, 32) and value_width % 64:
            raise InputFormatError(f"{path}: value width {value_width} is not 32 or a multiple of 64")
        stage = _payload_stage(n * row)
        if n and fh.readinto(memoryview(stage[: n * row].numpy())) != n * row:
            raise InputFormatError(f"{path}: truncated record dump")
    dev = device or default_device()
    kind = {32: "u32", 64: "u64", 128: "u128"}[key_width]
    kshape = (n, 2) if key_width == 128 else (n,)
    keys = torch.empty(kshape, dtype=torch.uint32 if key_width == 32 else torch.uint64, device=dev)
    values = None
    if value_width == 32:
        values = torch.empty(n, dtype=torch.uint32, device=dev)
    elif value_width == 64:
        values = torch.empty(n, dtype=torch.uint64, device=dev)
    elif value_width:
        values = torch.empty((n, value_width // 64), dtype=torch.uint64, device=dev)
    if n:
        rows = stage[: n * row].to(dev, non_blocking=True)
        st = torch.cuda.current_stream(dev).cuda_stream
        _lib.check(_lib.lib().ss_records_unpack(rows.data_ptr(), n, key_width // 8, value_width // 8,
                                                keys.data_ptr(), None if values is None else values.data_ptr(),
                                                st))
        torch.cuda.current_stream(dev).synchronize()   # the staging buffer is reused by the caller's GC
    return RecordArray(keys, values, kind)
