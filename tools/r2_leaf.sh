O=gpurun_out
for w in c5 c2; do
SS_LEAF_STATS=1 python bench.py --workload $w --steps 1 --warmup 1 --no-e2e --no-cpu --no-validate > $O/l_$w.json 2> $O/l_$w.err
grep leaf_stats $O/l_$w.err | tail -4
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_leaf --csv --log-file $O/leafk_$w.csv python bench.py --workload $w --steps 1 --warmup 0 --no-e2e --no-cpu --no-validate > /dev/null 2>&1
python - $O/leafk_$w.csv <<'PY'
import csv, sys, collections
rows = list(csv.reader(l for l in open(sys.argv[1]) if l.startswith('"')))
hdr = rows[0]; ki = hdr.index("Kernel Name"); vi = hdr.index("Metric Value"); ui = hdr.index("Metric Unit")
agg = collections.OrderedDict()
for r in rows[1:]:
    v = float(r[vi].replace(",", "")); u = r[ui]
    ms = v / 1e6 if u in ("ns", "nsecond") else v / 1e3 if u in ("us", "usecond") else v
    agg.setdefault(r[ki][:60], []).append(ms)
for k, v in agg.items(): print(k, ["%.2f" % x for x in v])
PY
done
