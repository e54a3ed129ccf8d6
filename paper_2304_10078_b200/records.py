"""RecordArray on device memory (the reference's records.py:34-132).

Same SoA layout as the reference: a 1-D ``keys`` column (uint32 or uint64)
and an optional ``values`` column (uint32 / uint64, or (n, 2) uint64 for
128-bit payloads).  Columns are torch CUDA tensors; numpy arrays (or any
array-like) are copied to the device on construction, which is how host
data enters the drop-in path.  Views never copy.
"""

from __future__ import annotations

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


class RecordArray:
    """Records (key, value) as device columns; mirrors records.py:34-132."""

    __slots__ = ("keys", "values", "arena", "key_kind")

    def __init__(self, keys, values=None, key_kind=None, arena=None):
        if key_kind == "bytes" or arena is not None:
            raise InputFormatError("byte-view keys are not supported by the GPU path")
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
        self.arena = None
        self.key_kind = key_kind

    # -- shape & views --------------------------------------------------------
    def __len__(self) -> int:
        return int(self.keys.shape[0])

    @property
    def key_width(self) -> int:
        return _KEY_WIDTH[self.key_kind]

    @property
    def key_bytes(self) -> int:
        return self.keys.element_size() * (2 if self.key_kind == "u128" else 1)

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
        out.arena = None
        out.key_kind = self.key_kind
        return out

    def _wrap(self, keys, values) -> "RecordArray":
        out = RecordArray.__new__(RecordArray)
        out.keys, out.values, out.arena, out.key_kind = keys, values, None, self.key_kind
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
