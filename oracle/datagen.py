"""Host restatement of the reference workload generators (datagen.py).

TEST INFRASTRUCTURE ONLY.  Regenerates the golden inputs byte for byte on
the GPU box (where /root/reference is absent) from the same numpy Philox
streams: per 2^18-record block, key = mix64_pair(mix64_pair(seed, family),
block) (datagen.py:66-69), keys then values drawn from that stream
(datagen.py:111-158).  ``tests/golden`` stores digests of the reference's
own outputs so a drift here is caught.
"""

from __future__ import annotations

import numpy as np

from .semisort_oracle import mix64_pair_int

__all__ = ["gen_keys_values", "GEN_BLOCK"]

GEN_BLOCK = 1 << 18                            # datagen.py:28
_FAMILY = {"uniform": 1, "exponential": 2, "zipfian": 3}   # datagen.py:22 order


def _zipf(rng, count, s, n):
    """Bounded Zipf by rejection-inversion (datagen.py:72-108)."""
    if s == 1.0:
        H, Hinv = np.log, np.exp
    else:
        a = 1.0 - s
        H = lambda x: np.expm1(a * np.log(x)) / a          # noqa: E731
        Hinv = lambda x: np.exp(np.log1p(x * a) / a)       # noqa: E731
    h = lambda x: np.exp(-s * np.log(x))                   # noqa: E731
    lo, hi = H(1.5) - 1.0, H(n + 0.5)
    cut = 2.0 - float(Hinv(H(2.5) - h(2.0)))
    out = np.empty(count, dtype=np.float64)
    todo = np.arange(count)
    while len(todo):
        u = lo + rng.random(len(todo)) * (hi - lo)
        x = Hinv(u)
        k = np.clip(np.floor(x + 0.5), 1.0, float(n))
        ok = (k - x <= cut) | (u >= H(k + 0.5) - h(k))
        out[todo[ok]] = k[ok]
        todo = todo[~ok]
    return out.astype(np.uint64)


def gen_keys_values(family: str, param, n: int, key_width: int = 64, seed: int = 1, universe=None):
    """(keys, values) exactly as the reference ``generate`` for 32/64-bit keys.

    ``universe`` overrides the Zipf rank range (the reference uses n,
    datagen.py:118); bench.py uses it to draw a bounded sample of the
    10^9-rank c2 workload."""
    kdt = np.uint32 if key_width == 32 else np.uint64
    keys = np.empty(n, dtype=kdt)
    vals = np.empty(n, dtype=kdt)
    for blk in range(-(-n // GEN_BLOCK)):
        lo, hi = blk * GEN_BLOCK, min((blk + 1) * GEN_BLOCK, n)
        rng = np.random.Generator(np.random.Philox(
            key=mix64_pair_int(mix64_pair_int(seed, _FAMILY[family]), blk)))
        cnt = hi - lo
        if family == "uniform":
            d = rng.integers(0, int(param), size=cnt, dtype=np.uint64)
        elif family == "exponential":
            d = np.floor(rng.exponential(scale=1.0 / param, size=cnt)).astype(np.uint64)
        else:
            d = _zipf(rng, cnt, float(param), n if universe is None else int(universe))
        keys[lo:hi] = d.astype(kdt)
        top = 2**32 - 1 if key_width == 32 else 2**64 - 1
        vals[lo:hi] = rng.integers(0, top, size=cnt, dtype=kdt, endpoint=True)
    return keys, vals
