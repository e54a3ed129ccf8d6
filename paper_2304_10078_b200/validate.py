"""Validators on the device (the reference's oracle.py:22-160 surface).

``validate_semisort`` checks permutation, contiguity and stability.  For
inputs whose values are the record indices (every benchmark input) it runs
the O(n) device check of SURVEY.md §8(c): a permutation bitmap over the
values, keys_out[i] == keys_in[values_out[i]], run count == distinct key
count (GPU hash set), strictly increasing values inside a run.  Other
inputs are checked on the host by the definition (a checker, not a
compute path).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .core import _stream, _workspace
from .records import RecordArray, signed_view


@dataclass
class ValidationReport:
    is_permutation: bool
    is_contiguous: bool
    is_stable: bool
    first_violation: tuple | None = None

    @property
    def valid(self) -> bool:
        return self.is_permutation and self.is_contiguous and self.is_stable

    def __bool__(self) -> bool:
        return self.valid


def count_distinct(keys: torch.Tensor) -> int:
    """Distinct keys of a device key column (GPU hash set)."""
    n = int(keys.shape[0])
    if n == 0:
        return 0
    lib = _lib.lib()
    ws = _workspace(lib.ss_count_distinct_workspace_bytes(n), keys.device)
    out = C.c_uint64(0)
    _lib.check(lib.ss_count_distinct(keys.data_ptr(), n, keys.element_size(), ws.data_ptr(), ws.numel(),
                                     C.byref(out), _stream(keys.device)))
    return int(out.value)


def validate_indexed(keys_in: torch.Tensor, keys_out: torch.Tensor, values_out: torch.Tensor,
                     distinct: int | None = None) -> ValidationReport:
    """O(n) device validation for inputs with values == record index."""
    n = int(keys_in.shape[0])
    if int(keys_out.shape[0]) != n or int(values_out.shape[0]) != n:
        return ValidationReport(False, False, False, (0, "length mismatch"))
    if distinct is None:
        distinct = count_distinct(keys_in)
    lib = _lib.lib()
    ws = _workspace(lib.ss_validate_workspace_bytes(n), keys_in.device)
    flags = (C.c_int32 * 4)()
    _lib.check(lib.ss_validate_indexed(keys_in.data_ptr(), keys_out.data_ptr(), values_out.data_ptr(), n,
                                       keys_in.element_size(), values_out.element_size(), distinct,
                                       ws.data_ptr(), ws.numel(), flags, _stream(keys_in.device)))
    perm = bool(flags[0]) and bool(flags[1])
    return ValidationReport(perm, bool(flags[2]), bool(flags[3]))


def _is_index_column(values: torch.Tensor | None) -> bool:
    if values is None or values.dim() != 1:
        return False
    n = int(values.shape[0])
    ar = torch.arange(n, device=values.device, dtype=torch.int64)
    return bool(torch.equal(signed_view(values).to(torch.int64), ar))


def _flat_keys(k: np.ndarray) -> np.ndarray:
    """128-bit (n, 2) rows as one comparable void16 column."""
    return k if k.ndim == 1 else np.ascontiguousarray(k).view(np.dtype((np.void, 16))).ravel()


def _content_ids(a: RecordArray, b: RecordArray):
    """Dense ids of the views' contents (equal bytes -> equal id), both arrays."""
    seen: dict[bytes, int] = {}

    def ids(d):
        buf = d.arena.cpu().numpy().tobytes()
        return np.array([seen.setdefault(buf[o:o + n], len(seen)) for o, n in d.keys_host().tolist()],
                        dtype=np.int64)
    return ids(a), ids(b)


def validate_semisort(input_data: RecordArray, output_data: RecordArray, adapter=None) -> ValidationReport:
    n = len(input_data)
    if len(output_data) != n:
        return ValidationReport(False, False, False, (0, "length mismatch"))
    if n == 0:
        return ValidationReport(True, True, True)
    if input_data.key_kind in ("u32", "u64") and _is_index_column(input_data.values):
        return validate_indexed(input_data.keys, output_data.keys, output_data.values)
    # definition-level host check (checker only)
    if input_data.key_kind == "bytes":   # byte-view keys compare by content (adapters.py:200-275)
        ki, ko = _content_ids(input_data, output_data)
    else:
        ki, ko = _flat_keys(input_data.keys_host()), _flat_keys(output_data.keys_host())
    brk = np.ones(n, dtype=bool)
    brk[1:] = ko[1:] != ko[:-1]
    contiguous = len(np.unique(ko[brk])) == int(brk.sum())
    oi, oo = np.argsort(ki, kind="stable"), np.argsort(ko, kind="stable")
    stable = np.array_equal(ki[oi], ko[oo])
    if stable and input_data.values is not None:
        stable = np.array_equal(input_data.values_host()[oi], output_data.values_host()[oo])
    if stable:
        return ValidationReport(True, contiguous, True)
    ri = np.sort(input_data.row_bytes().view(np.void), axis=0)
    ro = np.sort(output_data.row_bytes().view(np.void), axis=0)
    return ValidationReport(bool(np.array_equal(ri, ro)), contiguous, False)


def multiset_equal(a, b, adapter=None) -> bool:
    """Order-insensitive equality of two KeyedResults (oracle.py:150-160)."""
    ka, va = a.to_numpy()
    kb, vb = b.to_numpy()
    if len(ka) != len(kb):
        return False
    oa, ob = np.argsort(ka, kind="stable"), np.argsort(kb, kind="stable")
    ka, va, kb, vb = ka[oa], va[oa], kb[ob], vb[ob]
    if len(ka) > 1 and np.any(ka[1:] == ka[:-1]):
        return False
    return bool(np.array_equal(ka.astype(np.uint64), kb.astype(np.uint64)) and
                np.array_equal(va.astype(np.uint64), vb.astype(np.uint64)))
