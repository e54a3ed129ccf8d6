# distribute with the stores skipped (1) / written tile-contiguous (2): outputs are wrong, times only
O=gpurun_out
for w in c3 c2; do
for d in 0 1 2; do
  SS_DIST_DEBUG=$d timeout 300 python bench.py --workload $w --steps 2 --warmup 1 --no-e2e --no-cpu --no-validate > $O/d_${w}_$d.json 2> $O/d_${w}_$d.err
  python - "$O/d_${w}_$d.json" $w $d <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    ph = {k: round(v, 2) for k, v in d["phase_ms_per_step"].items()}
    print(sys.argv[2], "dbg", sys.argv[3], "ms", round(d["ms_per_step"], 3), ph)
except Exception as e:
    print(sys.argv[2], "failed", e)
PY
done; done
