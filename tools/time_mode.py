"""Time semisort on the c2 workload in a given mode (measurement helper)."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2304_10078_b200 as S  # noqa: E402
from paper_2304_10078_b200.datagen import generate_device  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "lt"
n = int(float(sys.argv[2])) if len(sys.argv) > 2 else 10**9
src = generate_device("zipfian", 1.2, n, key_bits=64, seed=1, universe=10**9, hash_ranks=True, values="index")
work = src.copy()
P = S.TuningParams.for_input(n)
for it in range(3):
    work.keys.copy_(src.keys)
    work.values.copy_(src.values)
    tel = S.Telemetry(timing=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    S.semisort(work, S.UIntKeyAdapter(), mode, P, telemetry=tel)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(mode, n, f"{dt*1e3:.1f} ms", f"{n/dt/1e9:.2f} Grec/s", {k: round(v, 2) for k, v in tel.phase_ms.items()},
          "leaves_global", tel.leaves_global)
