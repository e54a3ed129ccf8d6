# phase profile of the distribute (SS_DIST_DEBUG=4: per-phase cycles of thread 0 of each CTA)
O=gpurun_out
for w in ${WL:-c2 c3 c4}; do
  SS_DIST_DEBUG=4 python bench.py --workload $w --steps 1 --warmup 1 --no-e2e --no-cpu --no-validate > $O/p_$w.json 2> $O/p_$w.err
  grep dist_prof $O/p_$w.err | tail -${TAILN:-2}
done
