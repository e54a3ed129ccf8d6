"""Byte-view keys on the device (adapters.py:200-275, hashing.py:56-106).

A byte-view key is an (offset, length) row into a shared uint8 arena; the
reference hashes, compares and orders the referenced bytes.  The GPU path
turns every view into a 128-bit identity key and runs the fixed-width engine
on it:

* lo = the content hash, computed on the device exactly like
  ``BytePrefixHasher.hash_views`` (``ss_bytes_hash``) -- so the light buckets,
  the sampled heavy keys and the chained leaf order (all functions of the
  hash and of key equality) are the reference's;
* hi = the length for ``semisort(eq)`` / aggregation (equal (hash, length)
  stands for equal content, and that is CHECKED: records the engine grouped
  together are compared byte for byte, and a 64-bit hash collision between
  different contents raises instead of merging them), or the exact rank of
  the content in lexicographic byte order for ``semisort(lt)`` -- the
  128-bit key order (hi, lo) then sorts leaves by content, as the reference's
  ``sort_block`` does.

The engine permutes (key, record index) pairs; the caller's views and values
are then gathered by that permutation (semisort mutates in place, like the
reference).  Aggregation returns one representative view per distinct
content (the first record that has it).
"""

from __future__ import annotations

import ctypes as C

import torch

from . import _lib
from .errors import ContractError, InputFormatError


def _stream(dev) -> int:
    return torch.cuda.current_stream(dev).cuda_stream


def _views(data) -> torch.Tensor:
    if data.key_kind != "bytes" or data.arena is None:
        raise ContractError("byte-view keys need a RecordArray of kind 'bytes' with an arena")
    return data.keys


def content_hashes(data) -> torch.Tensor:
    """uint64[n]: the reference's content hash of every view (ss_bytes_hash)."""
    views = _views(data)
    n = len(data)
    out = torch.empty(n, dtype=torch.uint64, device=views.device)
    ctr = torch.empty(1, dtype=torch.uint64, device=views.device)
    rc = _lib.lib().ss_bytes_hash(data.arena.data_ptr(), data.arena.numel(), views.data_ptr(), n, out.data_ptr(),
                                  ctr.data_ptr(), _stream(views.device))
    if rc == _lib.SS_ERR_CONFIG:
        raise InputFormatError(_lib.lib().ss_last_error().decode("utf-8", "replace"))
    _lib.check(rc)
    return out


def content_ranks(data) -> torch.Tensor:
    """int64[n]: dense rank of every view's bytes in lexicographic order (a
    proper prefix first), refined 7 bytes at a time: rank <- dense rank of
    (rank, next chunk) rows until every view is exhausted."""
    views = _views(data)
    n = len(data)
    rank = torch.zeros(n, dtype=torch.int64, device=views.device)
    if n == 0:
        return rank
    max_len = int(views.view(torch.int64)[:, 1].max().item())
    chunk = torch.empty(n, dtype=torch.int64, device=views.device)
    for c in range(max(1, (max_len + 6) // 7)):
        _lib.check(_lib.lib().ss_bytes_chunk(data.arena.data_ptr(), views.data_ptr(), n, c, chunk.data_ptr(),
                                             _stream(views.device)))
        _, rank = torch.unique(torch.stack([rank, chunk], dim=1), dim=0, return_inverse=True)
    return rank


def synthetic_keys(data, mode: str = "eq") -> torch.Tensor:
    """uint64[n, 2] identity keys (lo = content hash, hi = length | rank)."""
    h = content_hashes(data)
    hi = content_ranks(data).view(torch.uint64) if mode == "lt" else data.keys[:, 1].contiguous()
    return torch.stack([h, hi], dim=1).contiguous()


def mismatches(data, a: torch.Tensor, b: torch.Tensor) -> int:
    """Number of i where the bytes of views a[i] and b[i] differ."""
    n = int(a.shape[0])
    if n == 0:
        return 0
    a, b = a.contiguous(), b.contiguous()
    ctr = torch.empty(1, dtype=torch.uint64, device=a.device)
    out = C.c_uint64(0)
    _lib.check(_lib.lib().ss_bytes_equal(data.arena.data_ptr(), a.data_ptr(), b.data_ptr(), n, ctr.data_ptr(),
                                         C.byref(out), _stream(a.device)))
    return int(out.value)


class HashCollision(RuntimeError):
    """Two different byte contents share a 64-bit content hash and length."""


def check_grouped(data, sorted_keys: torch.Tensor, perm: torch.Tensor) -> None:
    """After a semisort(eq) on synthetic keys: records with equal (hash,
    length) are contiguous; every such neighbour pair must hold equal bytes."""
    if sorted_keys.shape[0] < 2:
        return
    s = sorted_keys.view(torch.int64)
    same = (s[1:] == s[:-1]).all(dim=1)
    idx = torch.nonzero(same).flatten()
    if idx.numel() == 0:
        return
    v = data.keys.view(torch.int64)
    if mismatches(data, v[perm[idx + 1]], v[perm[idx]]):
        raise HashCollision("64-bit content-hash collision between different byte keys")


def representatives(data, syn: torch.Tensor, result_keys: torch.Tensor):
    """Views of one record per distinct synthetic key, in result order, and a
    byte-level check that every record equals its group's representative."""
    n = int(syn.shape[0])
    s = syn.view(torch.int64)
    uniq, inv = torch.unique(s, dim=0, return_inverse=True)
    first = torch.full((uniq.shape[0],), n, dtype=torch.int64, device=s.device)
    first.scatter_reduce_(0, inv, torch.arange(n, device=s.device), reduce="amin")
    v = data.keys.view(torch.int64)
    if mismatches(data, v, v[first[inv]]):
        raise HashCollision("64-bit content-hash collision between different byte keys")
    r = result_keys.view(torch.int64)
    both, inv2 = torch.unique(torch.cat([uniq, r]), dim=0, return_inverse=True)
    if both.shape[0] != uniq.shape[0]:
        raise RuntimeError("aggregate keys are not the input's distinct keys")
    return v[first[inv2[uniq.shape[0]:]]].contiguous().view(torch.uint64)
