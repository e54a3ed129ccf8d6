"""The ctypes mirrors of the C-ABI structs match include/semisort_b200.h
field for field (names, order, offsets) -- checked by compiling the header
with gcc (CPU tier; no GPU)."""

import os
import re
import shutil
import subprocess
import tempfile

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "semisort_b200.h")


def _c_fields(struct):
    src = open(HEADER).read()
    body = re.search(r"typedef struct %s \{(.*?)\} %s;" % (struct, struct), src, re.S).group(1)
    body = re.sub(r"/\*.*?\*/", "", body, flags=re.S)
    return [re.match(r"\s*\w+\s+(\w+)", ln).group(1) for ln in body.split(";") if ln.strip()]


@pytest.mark.parametrize("struct,cls", [("ss_telemetry", "SSTelemetry"), ("ss_params", "SSParams")])
def test_ctypes_struct_matches_header(struct, cls):
    import ctypes as C

    from paper_2304_10078_b200 import _lib
    py = getattr(_lib, cls)
    names = [f[0] for f in py._fields_]
    assert names == _c_fields(struct)
    if not shutil.which("gcc"):
        pytest.skip("gcc not available")
    with tempfile.TemporaryDirectory() as d:
        prog = os.path.join(d, "off.c")
        lines = ["#include <stdio.h>", "#include <stddef.h>", '#include "semisort_b200.h"', "int main(void) {",
                 f'  printf("%zu\\n", sizeof({struct}));']
        lines += [f'  printf("%zu\\n", offsetof({struct}, {n}));' for n in names]
        lines += ["  return 0;", "}"]
        open(prog, "w").write("\n".join(lines))
        exe = os.path.join(d, "off")
        subprocess.run(["gcc", f"-I{os.path.dirname(HEADER)}", prog, "-o", exe], check=True)
        got = [int(x) for x in subprocess.run([exe], capture_output=True, text=True, check=True).stdout.split()]
    assert got[0] == C.sizeof(py)
    assert got[1:] == [getattr(py, n).offset for n in names]
