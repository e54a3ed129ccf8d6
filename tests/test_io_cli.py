"""Record-dump I/O and the CLI backend.

Fixtures (tests/golden/io/, made by make_golden_io.py with the unmodified
reference): dumps for every key/value layout written by the reference's
``write_records``, and the reference CLI's ``sort`` / ``histogram`` /
``reduce`` / ``stats`` / ``transpose`` outputs on them.

CPU tier: the oracle's dump restatement round-trips every reference dump
byte for byte, and oracle semisort of each dump reproduces the reference
CLI's ``sort`` output (pinning the CLI's params: from_env, seed 1).  GPU
tier: ``read_records`` / ``write_records`` and ``python -m
paper_2304_10078_b200.cli`` reproduce the reference's files byte for byte
(aggregate CSVs as row multisets: the pair order is implementation-defined,
SPEC.md:256), ``bench`` keeps the reference CSV row schema.
"""

from __future__ import annotations

import csv
import io
import json
import os

import numpy as np
import pytest

import oracle as O

HERE = os.path.dirname(os.path.abspath(__file__))
IO = os.path.join(HERE, "golden", "io")
MAN = json.load(open(os.path.join(IO, "manifest.json")))


def _p(name):
    return os.path.join(IO, name)


def _blob(name):
    with open(_p(name), "rb") as fh:
        return fh.read()


# ---- CPU: the oracle restatement against the reference's files --------------

@pytest.mark.parametrize("name", MAN["dumps"])
def test_oracle_dump_roundtrip(name):
    blob = _blob(f"{name}.ssr")
    keys, values, kind = O.parse_dump(blob)
    kw = {"u32": 32, "u64": 64, "u128": 128}[kind]
    assert O.dump_bytes(keys, values, kw) == blob


@pytest.mark.parametrize("case", MAN["sort"], ids=lambda c: c["out"])
def test_oracle_reproduces_reference_cli_sort(case):
    keys, values, kind = O.parse_dump(_blob(case["in"]))
    n = len(keys)
    algo = case["algo"]
    ko, vo, _ = O.semisort(keys, values, O.OracleParams.derive(n, seed=1), "lt" if algo.endswith("lt") else "eq",
                           algo.startswith("int-"))
    kw = {"u32": 32, "u64": 64, "u128": 128}[kind]
    assert O.dump_bytes(ko, vo, kw) == _blob(case["out"])


def test_oracle_rejects_bad_dumps():
    blob = _blob("u64_v64.ssr")
    with pytest.raises(ValueError):
        O.parse_dump(b"XXXX" + blob[4:])
    with pytest.raises(ValueError):
        O.parse_dump(blob[:-3])


def test_cli_schema_matches_reference():
    from paper_2304_10078_b200 import cli
    assert cli.BENCH_COLUMNS == MAN["bench_columns"]
    p = cli.build_parser()
    a = p.parse_args(["bench", "--algo", "int-lt", "--dist", "zipfian", "--param", "1.2", "--n", "100",
                      "--key-bits", "128", "--reps", "2", "--verify"])
    assert (a.algo, a.dist, a.param, a.n, a.key_bits, a.reps, a.verify) == ("int-lt", "zipfian", 1.2, 100, 128, 2,
                                                                              True)
    a = p.parse_args(["reduce", "--in", "x.ssr", "--op", "count", "--identity"])
    assert (a.infile, a.op, a.identity, a.seed) == ("x.ssr", "count", True, 1)


# ---- GPU ----------------------------------------------------------------------

@pytest.fixture(scope="module")
def S():
    import paper_2304_10078_b200 as S
    return S


def _cli(argv):
    import contextlib

    from paper_2304_10078_b200 import cli
    out, err = io.StringIO(), io.StringIO()
    with contextlib.redirect_stdout(out), contextlib.redirect_stderr(err):
        rc = cli.main(argv)
    return rc, out.getvalue(), err.getvalue()


@pytest.mark.gpu
@pytest.mark.parametrize("name", MAN["dumps"])
def test_read_write_records_golden(S, name, tmp_path):
    from paper_2304_10078_b200.records import read_records, write_records
    keys, values, kind = O.parse_dump(_blob(f"{name}.ssr"))
    d = read_records(_p(f"{name}.ssr"))
    assert d.key_kind == kind and len(d) == len(keys)
    assert np.array_equal(d.keys_host(), keys)
    if values is None:
        assert d.values is None
    else:
        assert np.array_equal(d.values_host(), values)
    out = tmp_path / "rt.ssr"
    write_records(str(out), d)
    assert out.read_bytes() == _blob(f"{name}.ssr")


@pytest.mark.gpu
def test_records_errors(S, tmp_path):
    from paper_2304_10078_b200.records import read_records
    blob = _blob("u64_v64.ssr")
    bad = tmp_path / "bad.ssr"
    bad.write_bytes(b"XXXX" + blob[4:])
    with pytest.raises(S.InputFormatError, match="not a record dump"):
        read_records(str(bad))
    bad.write_bytes(blob[:-8])
    with pytest.raises(S.InputFormatError, match="corrupt record dump header"):
        read_records(str(bad))
    bad.write_bytes(blob[:10])
    with pytest.raises(S.InputFormatError):
        read_records(str(bad))


@pytest.mark.gpu
def test_records_large_roundtrip(S, tmp_path):
    """Device pack / unpack at a size that spans many CTAs and a ragged tail."""
    import torch

    from paper_2304_10078_b200.records import read_records, write_records
    n = 3_000_001
    g = torch.Generator(device="cuda").manual_seed(5)
    for kshape, vshape in (((n,), (n, 3)), ((n, 2), (n,)), ((n,), None)):
        k = torch.randint(0, 2**62, kshape, generator=g, device="cuda").view(torch.uint64)
        v = None if vshape is None else torch.randint(0, 2**62, vshape, generator=g, device="cuda").view(
            torch.uint64)
        d = S.RecordArray(k, v, "u128" if len(kshape) == 2 else "u64")
        path = tmp_path / "big.ssr"
        write_records(str(path), d)
        kk, vv, _ = O.parse_dump(path.read_bytes())
        assert np.array_equal(kk, k.cpu().numpy())
        assert (v is None and vv is None) or np.array_equal(vv, v.cpu().numpy())
        back = read_records(str(path))
        assert torch.equal(back.keys, d.keys)
        assert (v is None and back.values is None) or torch.equal(back.values, d.values)


@pytest.mark.gpu
@pytest.mark.parametrize("case", MAN["sort"], ids=lambda c: c["out"])
def test_cli_sort_golden(S, case, tmp_path):
    out = tmp_path / "o.ssr"
    rc, _, err = _cli(["sort", "--algo", case["algo"], "--in", _p(case["in"]), "--out", str(out), "--verify"])
    assert rc == 0 and "verified=true" in err
    assert out.read_bytes() == _blob(case["out"])


def _rows(text):
    return sorted(tuple(r) for r in csv.reader(io.StringIO(text)))


@pytest.mark.gpu
@pytest.mark.parametrize("case", MAN["aggregate"], ids=lambda c: c["out"])
def test_cli_aggregate_golden(S, case, tmp_path):
    out = tmp_path / "o.csv"
    rc, _, err = _cli(case["argv"] + ["--in", _p(case["in"]), "--out", str(out), "--verify"])
    assert rc == 0 and "verified=true" in err
    got, ref = out.read_text(), _blob(case["out"]).decode()
    assert got.splitlines()[0] == ref.splitlines()[0] == "key,aggregate"
    assert _rows(got) == _rows(ref)


@pytest.mark.gpu
@pytest.mark.parametrize("case", MAN["transpose"], ids=lambda c: c["out"])
def test_cli_transpose_golden(S, case, tmp_path):
    out = tmp_path / "t.csr"
    rc, _, err = _cli(["transpose", "--in", _p(case["in"]), "--out", str(out), "--verify"])
    assert rc == 0 and "verified=true" in err
    assert out.read_bytes() == _blob(case["out"])


@pytest.mark.gpu
def test_cli_errors(S, tmp_path):
    rc, _, err = _cli(["transpose", "--in", _p("bad_edges.txt")])
    assert rc == 2 and "expected 'u v'" in err
    rc, _, err = _cli(["sort", "--in", str(tmp_path / "missing.ssr")])
    assert rc == 2
    rc, _, err = _cli(["sort"])
    assert rc == 2 and "provide --in FILE" in err


@pytest.mark.gpu
@pytest.mark.parametrize("algo", ["eq", "lt", "int-eq", "int-lt", "histogram", "collect-reduce"])
@pytest.mark.parametrize("bits", [32, 64, 128])
def test_cli_bench_rows(S, algo, bits):
    dist, param = ("zipfian", "1.2") if bits != 32 else ("uniform", "5000")
    rc, out, err = _cli(["bench", "--algo", algo, "--dist", dist, "--param", param, "--n", "200000",
                         "--key-bits", str(bits), "--reps", "2", "--verify"])
    assert rc == 0, err
    rows = list(csv.DictReader(io.StringIO(out)))
    assert list(rows[0]) == MAN["bench_columns"] and len(rows) == 1
    r = rows[0]
    assert r["verified"] == "true" and r["n"] == "200000" and r["key_bits"] == str(bits)
    assert float(r["median_seconds"]) > 0 and int(r["depth_max"]) >= 1


@pytest.mark.gpu
def test_cli_bench_from_file(S, tmp_path):
    rc, out, _ = _cli(["bench", "--algo", "eq", "--in", _p("u64_v64.ssr"), "--reps", "1", "--verify"])
    assert rc == 0
    r = next(csv.DictReader(io.StringIO(out)))
    assert r["dist"] == "file" and r["verified"] == "true" and r["n"] == "3000"
