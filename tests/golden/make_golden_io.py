"""Golden fixtures for record-dump I/O and the CLI, made by the UNMODIFIED
reference (records.py:149-202, cli.py:83-485,
graphs.py:108-161).

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden_io.py

Writes tests/golden/io/: record dumps written by the reference's
``write_records`` for every key/value layout, the outputs of the reference
CLI (``sort`` dumps for the four algos, ``histogram`` / ``reduce`` CSVs,
``stats`` CSVs, ``transpose`` binary CSRs) and ``manifest.json`` (the
commands, plus the reference's CSV column lists).  Nothing at test time
reads /root/reference.
"""

from __future__ import annotations

import contextlib
import io
import json
import os
import shutil
import sys

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "io")

import semisort as S  # noqa: E402
from semisort import cli  # noqa: E402


def dumps(r):
    n = 3000
    u128 = np.empty((n, 2), np.uint64)
    u128[:, 0] = r.integers(0, 60, n)
    u128[:, 1] = r.integers(0, 3, n)
    z = np.minimum(r.zipf(1.3, n), 500).astype(np.uint64)
    return {
        "u32": S.RecordArray(r.integers(0, 400, n).astype(np.uint32)),
        "u32_v32": S.RecordArray(r.integers(0, 2**32, n, dtype=np.uint64).astype(np.uint32),
                                 np.arange(n, dtype=np.uint32)),
        "u64_v64": S.RecordArray(z * np.uint64(0x9E3779B97F4A7C15), np.arange(n, dtype=np.uint64)),
        "u64_v32": S.RecordArray(z, np.arange(n, dtype=np.uint32)),
        "u64_v128": S.RecordArray(z, np.stack([np.arange(n), np.arange(n) * 5], 1).astype(np.uint64)),
        "u64_v192": S.RecordArray(z, np.stack([np.arange(n)] * 3, 1).astype(np.uint64)),
        "u128_v64": S.RecordArray(u128, np.arange(n, dtype=np.uint64), "u128"),
        "u128_v128": S.RecordArray(u128, np.stack([np.arange(n), np.arange(n) + 7], 1).astype(np.uint64),
                                   "u128"),
        "u64_empty": S.RecordArray(np.zeros(0, np.uint64), np.zeros(0, np.uint64)),
        "u64_one": S.RecordArray(np.array([42], np.uint64)),
    }


def run_cli(argv):
    err = io.StringIO()
    with contextlib.redirect_stderr(err):
        rc = cli.main(argv)
    return rc, err.getvalue()


def main():
    if os.path.isdir(OUT):
        shutil.rmtree(OUT)
    os.makedirs(OUT)
    r = np.random.default_rng(2024)
    manifest = {"bench_columns": cli.BENCH_COLUMNS, "grid_columns": cli.GRID_COLUMNS,
                "dumps": [], "sort": [], "aggregate": [], "stats": [], "transpose": []}
    for name, data in dumps(r).items():
        S.write_records(os.path.join(OUT, f"{name}.ssr"), data)
        manifest["dumps"].append(name)

    p = lambda f: os.path.join(OUT, f)  # noqa: E731
    for src in ("u64_v64", "u128_v64", "u32_v32"):
        for algo in ("eq", "lt", "int-eq", "int-lt"):
            out = f"sort_{src}_{algo}.ssr"
            rc, _ = run_cli(["sort", "--algo", algo, "--in", p(f"{src}.ssr"), "--out", p(out)])
            assert rc == 0
            manifest["sort"].append({"in": f"{src}.ssr", "algo": algo, "out": out})
    for src in ("u64_v64", "u32", "u64_v32"):
        for cmd in (["histogram"], ["histogram", "--identity"], ["reduce", "--op", "count"],
                    ["reduce", "--op", "sum"]):
            if cmd[-1] == "sum" and src == "u32":
                continue
            out = f"agg_{src}_{'_'.join(c.strip('-') for c in cmd)}.csv"
            rc, _ = run_cli(cmd + ["--in", p(f"{src}.ssr"), "--out", p(out)])
            assert rc == 0
            manifest["aggregate"].append({"in": f"{src}.ssr", "argv": cmd, "out": out})
    for src in ("u64_v64", "u32", "u128_v64", "u64_one"):
        out = f"stats_{src}.csv"
        rc, _ = run_cli(["stats", "--in", p(f"{src}.ssr"), "--out", p(out)])
        assert rc == 0
        manifest["stats"].append({"in": f"{src}.ssr", "out": out})

    # graphs: a text edge list (comments, blank lines) and a binary CSR input
    m, n = 4000, 300
    src = np.minimum(r.zipf(1.4, m) - 1, n - 1)
    dst = r.integers(0, n, m)
    with open(p("edges.txt"), "w") as fh:
        fh.write("# synthetic edge list\n\n")
        for u, v in zip(src.tolist(), dst.tolist()):
            fh.write(f"{u} {v}\n")
    S.graphs.write_csr(p("graph.csr"), S.graphs.from_edges(n, src.astype(np.uint32), dst.astype(np.uint32)))
    for gin in ("edges.txt", "graph.csr"):
        out = f"transpose_{gin.replace('.', '_')}.csr"
        rc, _ = run_cli(["transpose", "--in", p(gin), "--out", p(out)])
        assert rc == 0
        manifest["transpose"].append({"in": gin, "out": out})
    with open(p("bad_edges.txt"), "w") as fh:
        fh.write("0 1\n1 2 3\n")
    with open(p("manifest.json"), "w") as fh:
        json.dump(manifest, fh, indent=1)
    print("wrote", len(os.listdir(OUT)), "files")


if __name__ == "__main__":
    main()
