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
