"""CPU tier: the C-ABI library loads and exports every declared symbol, and
the host-side logic (params, adapters, error mapping) matches the reference."""
import ctypes
import math
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "semisort_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ss_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2304_10078_b200 import _build, _lib
    _build.build()
    lib = ctypes.CDLL(_lib.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 20
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    assert set(syms) == set(_lib.EXPORTS), set(syms) ^ set(_lib.EXPORTS)


def test_library_reports_version_and_errors_without_gpu():
    from paper_2304_10078_b200 import _lib
    L = _lib.lib()
    assert L.ss_version() == 1
    P = _lib.SSParams()
    P.light_buckets, P.light_bits, P.subarray_len, P.base_case_cutoff = 3, 1, 4, 1
    # size query validates params on the host: bad light_buckets -> 0 and a message
    assert L.ss_semisort_workspace_bytes(8, 8, 8, ctypes.byref(P)) == 0
    assert b"power of two" in L.ss_last_error()
    with pytest.raises(Exception) as ei:
        _lib.check(_lib.SS_ERR_CONFIG)
    from paper_2304_10078_b200.errors import ConfigurationError
    assert isinstance(ei.value, ConfigurationError) and isinstance(ei.value, ValueError)


def test_workspace_sizes_scale():
    from paper_2304_10078_b200 import TuningParams, _lib
    L = _lib.lib()
    for n in (0, 1, 1000, 2**20, 10**9):
        P = TuningParams.for_input(n).as_c()
        ws = L.ss_semisort_workspace_bytes(n, 8, 8, ctypes.byref(P))
        assert ws >= 16 * n
        if n == 10**9:
            assert ws < 26 * n       # scratch + u16 ids + bounded level structures
        wa = L.ss_aggregate_workspace_bytes(n, 8, 8, ctypes.byref(P))
        assert wa >= 32 * n


@pytest.mark.parametrize("n", [0, 1, 2, 7, 1000, 2**20, 10**9, 8 * 10**9])
def test_params_match_reference_derivation(n):
    from paper_2304_10078_b200 import TuningParams
    import oracle as O
    p, o = TuningParams.for_input(n), O.OracleParams.derive(n)
    assert (p.light_buckets, p.light_bits, p.subarray_len, p.base_case_cutoff, p.max_heavy,
            p.sample_factor, p.seed, p.sample_count) == \
        (o.n_light, o.bits, o.sub_len, o.alpha, o.max_heavy, o.sample_factor, o.seed, o.samples)
    assert p.heavy_threshold == o.threshold
    assert p.as_c().heavy_threshold_int == max(1, math.ceil(o.threshold))
    assert p.rounds_per_hash == o.rounds


def test_params_validation_and_env():
    from paper_2304_10078_b200 import ConfigurationError, TuningParams
    with pytest.raises(ConfigurationError):
        TuningParams.for_input(10, light_buckets=3)
    with pytest.raises(ConfigurationError):
        TuningParams.for_input(10, subarray_len=4, light_buckets=8)
    with pytest.raises(ConfigurationError):
        TuningParams.for_input(-1)
    p = TuningParams.from_env(1000, env={"SEMISORT_LIGHT_BUCKETS": "16", "SEMISORT_SEED": "9"})
    assert p.light_buckets == 16 and p.seed == 9
    with pytest.raises(ConfigurationError):
        TuningParams.from_env(1000, env={"SEMISORT_SEED": "x"})


def test_adapter_contracts():
    from paper_2304_10078_b200 import ContractError, UInt128KeyAdapter, UIntKeyAdapter
    from paper_2304_10078_b200.adapters import device_identity_flag
    import oracle as O
    assert device_identity_flag(UIntKeyAdapter()) == 0
    assert device_identity_flag(UIntKeyAdapter(identity=True)) == 1

    class FixedHash(UIntKeyAdapter):
        def hash_scalar(self, key):
            return int(key)

    class Plain(UIntKeyAdapter):
        pass

    assert device_identity_flag(Plain()) == 0
    with pytest.raises(ContractError):
        device_identity_flag(FixedHash())
    with pytest.raises(ContractError):
        device_identity_flag(UInt128KeyAdapter())
    a = UIntKeyAdapter()
    assert a.hash_scalar(0) == O.mix64_int(0) == 0xE220A8397B1DCDAF
    assert UIntKeyAdapter(identity=True).hash_scalar(13) == 13


def test_reduce_spec_and_keyed_result_host():
    import io
    from paper_2304_10078_b200 import ConfigurationError, KeyedResult, ReduceSpec
    with pytest.raises(ConfigurationError):
        ReduceSpec(lambda k, v: 1, lambda a, b: a + b, 0, "bogus")
    s = ReduceSpec.summing64()
    assert s.combine(2**64 - 1, 3) == 2
    with pytest.raises(ConfigurationError):
        s.map_record(1, None)
    r = KeyedResult([(3, 2), (1, 1), ((5, 1), 7)])
    buf = io.StringIO()
    r.write_csv(buf)
    lines = buf.getvalue().splitlines()
    assert lines[0] == "key,aggregate" and lines[1] == "3,2" and lines[3] == f"{(1 << 64) | 5},7"
    assert r == KeyedResult([(3, 2), (1, 1), ((5, 1), 7)]) and len(r) == 3


def test_philox_key_extraction():
    from paper_2304_10078_b200 import ContractError
    from paper_2304_10078_b200.core import _philox_key
    assert _philox_key(np.random.Generator(np.random.Philox(key=12345))) == 12345
    g = np.random.Generator(np.random.Philox(key=3))
    g.integers(0, 10)
    with pytest.raises(ContractError):
        _philox_key(g)
    with pytest.raises(ContractError):
        _philox_key(np.random.default_rng(1))
