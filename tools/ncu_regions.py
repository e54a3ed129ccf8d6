"""Summarise an ncu report's SASS page by barrier-delimited regions (measurement helper).

    python tools/ncu_regions.py report.ncu-rep
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
data = rows[2:]
i_s = h.index("Warp Stall Sampling (All Samples)")
i_e = h.index("Instructions Executed")
num = lambda x: int(x) if x.isdigit() else 0  # noqa: E731
tot = sum(num(r[i_s]) for r in data)
print("instructions", len(data), "samples", tot, "warp-instr", sum(num(r[i_e]) for r in data))
cuts = [k for k, r in enumerate(data) if "BAR" in r[1] or "EXIT" in r[1]]
prev = 0
for b in cuts + [len(data) - 1]:
    s = sum(num(r[i_s]) for r in data[prev:b + 1])
    e = sum(num(r[i_e]) for r in data[prev:b + 1])
    if s > 0.005 * tot:
        print(f"{prev:5d}-{b:5d} samples {s:8d} ({100 * s / tot:5.1f}%) warp-instr {e:12d}  last: {data[b][1].strip()[:40]}")
    prev = b + 1
top = sorted(range(len(data)), key=lambda k: -num(data[k][i_s]))[:int(sys.argv[2]) if len(sys.argv) > 2 else 12]
for k in top:
    print(k, data[k][1].strip()[:64], data[k][i_s], data[k][i_e])
