# A/B of environment switches on the bench lines: AB="VAR=val[,VAR=val] ..." (space-separated variants) WL="c2 c3 c4"
O=gpurun_out
for w in ${WL:-c2 c3 c4}; do
 for v in base $AB; do
  e=$(echo $v | tr ',' ' '); [ "$v" = base ] && e=""
  env $e python bench.py --workload $w --steps 4 --warmup 3 --no-e2e --no-cpu > $O/ab_$w.json 2> $O/ab_$w.err
  python - "$O/ab_$w.json" $w "$v" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    ph = {k: round(v, 2) for k, v in d["phase_ms_per_step"].items()}
    print(sys.argv[2], sys.argv[3], "ms", round(d["ms_per_step"], 3), "Grec/s", round(d["value"], 1), "valid", d.get("validated"), ph)
except Exception as e:
    print(sys.argv[2], "failed", e)
PY
 done
done
