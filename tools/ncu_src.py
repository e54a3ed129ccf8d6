"""Summarise an ncu SASS source page (CSV, optionally .gz) by barrier-delimited
regions, with stall samples, shared-memory wavefronts (actual / ideal) and the
top instructions (measurement helper).

    python tools/ncu_src.py gpurun_out/r2_c4_src2.csv.gz [top]
"""
import csv
import gzip
import io
import sys

f = sys.argv[1]
raw = gzip.open(f).read().decode() if f.endswith(".gz") else open(f).read()
rows = list(csv.reader(io.StringIO(raw)))
print(rows[0][1][:150])
h = rows[1]
data = [r for r in rows[2:] if len(r) == len(h)]
col = {name: h.index(name) for name in h}
num = lambda x: float(x) if x.replace(".", "", 1).isdigit() else 0.0  # noqa: E731
S, E = col["Warp Stall Sampling (All Samples)"], col["Instructions Executed"]
WS, WI = col["L1 Wavefronts Shared"], col["L1 Wavefronts Shared Ideal"]
L2S, L2I = col["L2 Theoretical Sectors Global"], col["L2 Theoretical Sectors Global Ideal"]
tot = sum(num(r[S]) for r in data)
print(f"instructions {len(data)} samples {tot:.0f} warp-instr {sum(num(r[E]) for r in data):.3e} "
      f"smem wavefronts {sum(num(r[WS]) for r in data):.3e} (ideal {sum(num(r[WI]) for r in data):.3e}) "
      f"L2 sectors {sum(num(r[L2S]) for r in data):.3e} (ideal {sum(num(r[L2I]) for r in data):.3e})")
cuts = [k for k, r in enumerate(data) if "BAR" in r[1] or "EXIT" in r[1]]
prev = 0
stalls = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
for b in cuts + [len(data) - 1]:
    seg = data[prev:b + 1]
    s = sum(num(r[S]) for r in seg)
    if s > 0.01 * tot:
        st = sorted(((sum(num(r[col[c]]) for r in seg), c) for c in stalls), reverse=True)[:3]
        print(f"{prev:5d}-{b:5d} samples {100 * s / tot:5.1f}% instr {sum(num(r[E]) for r in seg):.3e} "
              f"smem wf {sum(num(r[WS]) for r in seg):.3e}/{sum(num(r[WI]) for r in seg):.3e} "
              f"L2 sec {sum(num(r[L2S]) for r in seg):.3e}/{sum(num(r[L2I]) for r in seg):.3e} | "
              + " ".join(f"{c[6:]}={100 * v / max(s, 1):.0f}%" for v, c in st) + f" | {data[b][1].strip()[:30]}")
    prev = b + 1
top = int(sys.argv[2]) if len(sys.argv) > 2 else 15
print("top by samples:")
for k in sorted(range(len(data)), key=lambda k: -num(data[k][S]))[:top]:
    r = data[k]
    print(f"{k:5d} {r[1].strip()[:58]:58s} s={num(r[S]):7.0f} e={num(r[E]):.2e} wf={num(r[WS]):.2e}/{num(r[WI]):.2e}")
