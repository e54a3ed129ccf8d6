# GPU tests + c2/c5/c3/c4 bench lines (no e2e / cpu legs)
O=gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > $O/pytest_q.log 2>&1; tail -2 $O/pytest_q.log
for w in ${WL:-c2 c5 c3 c4}; do
  python bench.py --workload $w --steps 4 --warmup 3 --no-e2e --no-cpu > $O/q_$w.json 2> $O/q_$w.err
  python - "$O/q_$w.json" $w <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    ph = {k: round(v, 2) for k, v in d["phase_ms_per_step"].items()}
    print(sys.argv[2], "ms", round(d["ms_per_step"], 3), "Grec/s", round(d["value"], 1), "valid", d.get("validated"), ph)
except Exception as e:
    print(sys.argv[2], "failed", e)
PY
done
