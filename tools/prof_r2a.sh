# ncu captures of the hot kernels for c4 / c2 / c3 (one step each); the
# reports are summarised on the box (raw metrics CSV, details page, SASS
# source page of each kernel) and only the summaries come back.
set -x
B="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu"
O=gpurun_out
prof() {   # name, regex, count, extra bench args
  $B $4 > $O/p_$1.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"$2" -c $3 -o /tmp/$1 $B $4 > $O/ncu_$1.log 2>&1
  ncu -i /tmp/$1.ncu-rep --page raw --csv > $O/$1_raw.csv 2>/dev/null
  ncu -i /tmp/$1.ncu-rep --page details > $O/$1_details.txt 2>/dev/null
  for k in $(seq 0 $(($3 - 1))); do
    ncu -i /tmp/$1.ncu-rep --page source --csv --print-source sass --launch-skip $k --launch-count 1 2>/dev/null | gzip > $O/$1_src$k.csv.gz
  done
}
prof r2_c4 "k_distribute1|k_fold_nodes|k_count|k_sample" 8 "--workload c4"
prof r2_c2 "k_count|k_copy_heavy|k_leaf_eq|k_sample|k_distribute1" 14 ""
prof r2_c3 "k_distribute1|k_fold_nodes|k_count" 6 "--workload c3"
du -sh $O
