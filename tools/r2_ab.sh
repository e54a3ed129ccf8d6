# correctness of the default path + A/B of SS_DIST_KERNEL (default dist2 vs v1) on c2/c3/c4/c5
O=gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > $O/pytest_ab.log 2>&1; tail -3 $O/pytest_ab.log
for w in c2 c3 c4 c5; do
  for k in default v1; do
    if [ $k = default ]; then unset SS_DIST_KERNEL; else export SS_DIST_KERNEL=$k; fi
    python bench.py --workload $w --steps 4 --warmup 3 --no-e2e --no-cpu > $O/ab_${w}_$k.json 2> $O/ab_${w}_$k.err
    python - "$O/ab_${w}_$k.json" $w $k <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(sys.argv[2], sys.argv[3], "ms", round(d["ms_per_step"], 3), "dist", round(d["phase_ms_per_step"]["distribute"], 3), "valid", d.get("validated"))
except Exception as e:
    print(sys.argv[2], sys.argv[3], "failed", e)
PY
  done
done
unset SS_DIST_KERNEL
