# ncu --set full of kernels matching $2 (count $3) in one bench step of workload $1; summaries into gpurun_out/$4*
set -x
B="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --no-validate --workload $1"
O=gpurun_out
$B > $O/p_$4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"$2" -c $3 -o /tmp/$4 $B > $O/ncu_$4.log 2>&1
ncu -i /tmp/$4.ncu-rep --page raw --csv > $O/$4_raw.csv 2>/dev/null
ncu -i /tmp/$4.ncu-rep --page details > $O/$4_details.txt 2>/dev/null
for k in $(seq 0 $(($3 - 1))); do
  ncu -i /tmp/$4.ncu-rep --page source --csv --print-source sass --launch-skip $k --launch-count 1 2>/dev/null | gzip > $O/$4_src$k.csv.gz
done
