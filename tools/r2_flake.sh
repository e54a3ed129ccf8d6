O=gpurun_out
for r in 1 2 3; do for w in c3 c4 c2; do
python bench.py --workload $w --steps 5 --warmup 3 --no-e2e --no-cpu --no-validate 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$w', round(d['ms_per_step'],2), d.get('ms_steps') or d.get('ms_steps_rank0'), round(sum(d['phase_ms_per_step'].values()),2))"
done; done
