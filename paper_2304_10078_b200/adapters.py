"""Key adapters of the drop-in surface (adapters.py:25-284 of the reference).

The GPU path implements the fixed-width integer adapters: hash =
mix64(u64(key)) or the identity (adapters.py:112-119), equality on the key
bits, stable order by key value; the 128-bit adapter (hash mix64(mix64(hi) ^
lo) or lo, order (hi, lo); adapters.py:147-198); and byte-view keys
(content hash, content equality and order; adapters.py:200-275).  Any
adapter whose hash or equality is arbitrary Python (a subclass overriding
them) cannot run on the device and is rejected with ContractError instead of
being silently executed on the CPU.
"""

from __future__ import annotations

from .errors import ContractError

U64_MASK = (1 << 64) - 1
_GAMMA, _M1, _M2 = 0x9E3779B97F4A7C15, 0xBF58476D1CE4E5B9, 0x94D049BB133111EB


def _mix64(x: int) -> int:
    z = (x + _GAMMA) & U64_MASK
    z = ((z ^ (z >> 30)) * _M1) & U64_MASK
    z = ((z ^ (z >> 27)) * _M2) & U64_MASK
    return z ^ (z >> 31)


class KeyAdapter:
    """Base adapter (adapters.py:25-78)."""

    key_kind: str = "abstract"
    identity_mode: bool = False
    has_lt: bool = True

    def hash_scalar(self, key) -> int:
        raise NotImplementedError


class UIntKeyAdapter(KeyAdapter):
    """Plain 32/64-bit unsigned integer keys (adapters.py:103-144)."""

    key_kind = "uint"

    def __init__(self, identity: bool = False, with_lt: bool = True):
        self.identity_mode = identity
        self.has_lt = with_lt

    def hash_scalar(self, key) -> int:
        """Host scalar form of the device hash (for host-side bookkeeping)."""
        k = int(key) & U64_MASK
        return k if self.identity_mode else _mix64(k)


class UInt128KeyAdapter(KeyAdapter):
    """128-bit keys as (lo, hi) word pairs (adapters.py:147-198).

    semisort, collect_reduce and histogram run them on the device; the
    phase-level entry points stay 32/64-bit and reject them with ContractError.
    """

    key_kind = "u128"

    def __init__(self, identity: bool = False, with_lt: bool = True):
        self.identity_mode = identity
        self.has_lt = with_lt

    def hash_scalar(self, key) -> int:
        lo, hi = key
        lo &= U64_MASK
        return lo if self.identity_mode else _mix64(_mix64(hi & U64_MASK) ^ lo)


_POLY_MULT = 0x100000001B3   # hashing.py:19 (the FNV-1a prime)


def hash_bytes(data: bytes) -> int:
    """Host scalar form of the content hash (hashing.py:56-66): mix64 of the
    wrapping polynomial over the bytes xor mix64(len).  The device computes
    the same (ss_bytes_hash)."""
    acc = 0
    for b in bytes(data):
        acc = (acc * _POLY_MULT + b) & U64_MASK
    return _mix64(acc ^ _mix64(len(data)))


class BytesKeyAdapter(KeyAdapter):
    """Byte-view keys over a shared arena (adapters.py:200-275): equality and
    order compare the referenced bytes, the hash is the content polynomial
    (offsets never matter).  On the GPU (bytes_keys.py) the views become
    128-bit identity keys (content hash, length or exact content rank)."""

    key_kind = "bytes"
    identity_mode = False
    has_lt = True

    def __init__(self, arena=None):
        self.arena = arena

    def hash_scalar(self, key) -> int:
        return hash_bytes(key)


def adapter_for(data, *, identity: bool = False) -> KeyAdapter:
    if data.key_kind in ("u32", "u64"):
        return UIntKeyAdapter(identity=identity)
    if data.key_kind == "u128":
        return UInt128KeyAdapter(identity=identity)
    return BytesKeyAdapter(getattr(data, "arena", None))


def device_identity_flag(adapter: KeyAdapter, allow_u128: bool = False) -> int:
    """1/0 identity mode for a device-executable adapter, else ContractError."""
    base = UIntKeyAdapter
    if allow_u128 and isinstance(adapter, UInt128KeyAdapter):
        base = UInt128KeyAdapter
    elif not isinstance(adapter, UIntKeyAdapter):
        raise ContractError(
            f"{type(adapter).__name__} keys are not supported by this GPU entry point "
            "(fixed-width integer keys only)")
    custom = ("hash_scalar", "hash_block", "group_block", "sort_block", "match_packed", "match_rows")
    for cls in type(adapter).__mro__:
        if cls is base:
            break
        for name in custom:
            if name in cls.__dict__:
                raise ContractError(
                    f"{type(adapter).__name__}.{name} is custom Python; the GPU path only runs the "
                    "built-in mix64 / identity integer hash")
    return 1 if adapter.identity_mode else 0
