# A/B of the distribute launch shapes (SS_DIST_SHAPE) on c2 / c3 / c4
O=gpurun_out
for w in c2 c3 c4; do
  for s in 0 1 2; do
    SS_DIST_SHAPE=$s python bench.py --workload $w --steps 4 --warmup 3 --no-e2e --no-cpu > $O/shape_${w}_$s.json 2> $O/shape_${w}_$s.err
    python - "$O/shape_${w}_$s.json" $w $s <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(sys.argv[2], "shape", sys.argv[3], "ms", round(d["ms_per_step"], 3), "dist", round(d["phase_ms_per_step"]["distribute"], 3), "valid", d.get("validated"))
except Exception as e:
    print(sys.argv[2], sys.argv[3], "failed", e)
PY
  done
done
