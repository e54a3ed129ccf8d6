"""Time collect_reduce / histogram on the c3 / c4 workloads (measurement helper).

    python tools/time_agg.py c4 [n] [reps]
"""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2304_10078_b200 as S  # noqa: E402
from paper_2304_10078_b200.datagen import generate_device  # noqa: E402

w = sys.argv[1] if len(sys.argv) > 1 else "c4"
n = int(float(sys.argv[2])) if len(sys.argv) > 2 else 10**9
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
if w == "c4":
    src = generate_device("uniform", 1e7, n, key_bits=32, seed=1, values="none")
    spec = S.ReduceSpec.counting()
else:
    src = generate_device("exponential", 1e-4, n, key_bits=64, seed=1, values="random", value_shift=32)
    spec = S.ReduceSpec.summing64()
P = S.TuningParams.for_input(n)
for it in range(reps):
    tel = S.Telemetry(timing=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = S.collect_reduce(src, S.UIntKeyAdapter(), spec, P, telemetry=tel)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(w, n, f"{dt*1e3:.1f} ms", f"{n/dt/1e9:.2f} Grec/s", {k: round(v, 2) for k, v in tel.phase_ms.items()},
          "folded", tel.nodes_folded, "pairs", len(res), flush=True)
