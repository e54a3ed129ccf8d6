"""Seeded synthetic workloads generated on the device (benchmark inputs).

The reference generators (datagen.py:66-158) draw from numpy Philox on the
host at ~40-300 Mrec/s, far too slow for 10^9-record inputs on each GPU box.
``generate_device`` reproduces the same families and parameters — uniform,
floor(exponential), bounded Zipf by the same rejection-inversion sampler,
uniform 64-bit and the config-5 mix — from a counter-based Philox stream on
the device, so any shard of a global input can be regenerated
independently (value = global index for the semisort configs).
"""

from __future__ import annotations

import torch

from . import _lib
from .core import _stream
from .records import RecordArray, default_device

FAMILIES = {"uniform": 0, "exponential": 1, "zipfian": 2, "uniform64": 3, "mix": 4}


def generate_device(family: str, param: float, n: int, *, key_bits: int = 64, seed: int = 1,
                    universe: int | None = None, hash_ranks: bool = False, values: str = "index",
                    first_index: int = 0, value_shift: int = 0, device=None) -> RecordArray:
    """values: "index" (value = global index), "random" (uniform bits >>
    value_shift) or "none"."""
    dev = device or default_device()
    kdt = torch.uint32 if key_bits == 32 else torch.uint64
    keys = torch.empty(n, dtype=kdt, device=dev)
    vals = None if values == "none" else torch.empty(n, dtype=kdt, device=dev)
    vmode = {"none": 0, "index": 1, "random": 2}[values]
    uni = universe if universe is not None else n
    _lib.check(_lib.lib().ss_generate(FAMILIES[family], float(param), int(uni), n, first_index, key_bits // 8,
                                      seed, 1 if hash_ranks else 0, keys.data_ptr(),
                                      None if vals is None else vals.data_ptr(),
                                      0 if vals is None else key_bits // 8, vmode, value_shift, _stream(dev)))
    return RecordArray(keys, vals)


# -- the reference's generator surface (datagen.py:34-61, 121-195) ------------

import math  # noqa: E402
from dataclasses import dataclass  # noqa: E402

from .errors import ConfigurationError  # noqa: E402

SPEC_FAMILIES = ("uniform", "exponential", "zipfian")
HEAVY_STAT_FACTOR = 500


@dataclass(frozen=True)
class DistributionSpec:
    """datagen.py:34-55: same fields and validation (ConfigurationError)."""

    family: str
    parameter: float
    n: int
    key_width: int = 64
    seed: int = 1

    def __post_init__(self):
        if self.family not in SPEC_FAMILIES:
            raise ConfigurationError(f"unknown family {self.family!r}")
        if self.n < 0:
            raise ConfigurationError("n must be >= 0")
        if self.key_width not in (32, 64, 128):
            raise ConfigurationError("key_width must be 32, 64 or 128")
        if self.family == "uniform":
            if self.parameter < 1 or self.parameter != int(self.parameter):
                raise ConfigurationError("uniform mu must be a positive integer")
            if self.key_width == 32 and self.parameter > 2**32:
                raise ConfigurationError("uniform mu exceeds 32-bit keys")
        elif self.parameter <= 0:
            raise ConfigurationError(f"{self.family} parameter must be > 0")


def generate(spec: DistributionSpec, *, workers: int | None = None, device=None) -> RecordArray:
    """datagen.py:121-158 on the device: the same families, parameters and
    layouts (keys of the spec's width, random value words of the key width;
    128-bit keys carry the draw in the low word).  The draws come from the
    device Philox stream, so the bytes differ from the reference's numpy
    streams; feed a reference dump through ``read_records`` for byte-level
    comparisons."""
    dev = device or default_device()
    n = spec.n
    if n == 0:
        kdt = torch.uint32 if spec.key_width == 32 else torch.uint64
        shape = (0, 2) if spec.key_width == 128 else (0,)
        return RecordArray(torch.empty(shape, dtype=kdt, device=dev), torch.empty(shape, dtype=kdt, device=dev),
                           {32: "u32", 64: "u64", 128: "u128"}[spec.key_width])
    bits = 32 if spec.key_width == 32 else 64
    base = generate_device(spec.family, float(spec.parameter), n, key_bits=bits, seed=spec.seed,
                           universe=n if spec.family == "zipfian" else None, values="random", device=dev)
    if spec.key_width != 128:
        return base
    hi = generate_device("uniform", 1.0, n, key_bits=64, seed=spec.seed ^ 0x5EED, values="random", device=dev)
    keys = torch.zeros((n, 2), dtype=torch.uint64, device=dev)
    keys[:, 0] = base.keys
    values = torch.stack([base.values, hi.values], dim=1).contiguous()
    return RecordArray(keys, values, "u128")


@dataclass(frozen=True)
class InputStats:
    """datagen.py:58-62."""

    distinct_keys: int
    max_frequency: int
    heavy_freq_ratio: float


def heavy_stat_threshold(n: int) -> float:
    return HEAVY_STAT_FACTOR * math.log2(max(n, 2))


def compute_stats(data: RecordArray, adapter=None) -> InputStats:
    """datagen.py:165-195 on the device: per-key counts from the GPU
    histogram (32/64-bit keys) or from the runs of a GPU semisort (128-bit)."""
    from .adapters import UInt128KeyAdapter, UIntKeyAdapter
    from .aggregate import histogram
    from .core import semisort
    n = len(data)
    if n == 0:
        return InputStats(0, 0, 0.0)
    if data.key_kind == "u128":
        work = data.copy()
        semisort(work, UInt128KeyAdapter(), "eq")
        k = work.keys.view(torch.int64)
        change = torch.ones(n, dtype=torch.bool, device=k.device)
        change[1:] = (k[1:] != k[:-1]).any(dim=1)
        starts = torch.nonzero(change).flatten()
        counts = torch.diff(torch.cat([starts, torch.tensor([n], device=k.device)]))
    else:
        counts = histogram(data, UIntKeyAdapter()).agg_tensor.view(torch.int64)
    threshold = heavy_stat_threshold(n)
    heavy = int(counts[counts.to(torch.float64) > threshold].sum())
    return InputStats(distinct_keys=int(counts.numel()), max_frequency=int(counts.max()),
                      heavy_freq_ratio=heavy / n)
