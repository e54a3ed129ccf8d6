# Round-2 evidence: GPU tests, every bench line (c2 default with e2e + reference CPU baseline, lt, c5, c3, c4, c1,
# graph), the reference arm, and the ncu launch list of the default command.
O=gpurun_out/final
mkdir -p $O
nproc > $O/nproc.txt; lscpu > $O/lscpu.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
python bench.py > $O/b_c2.json 2> $O/b_c2.err
python bench.py --mode lt --no-cpu > $O/b_c2_lt.json 2> $O/b_c2_lt.err
python bench.py --workload c5 --no-cpu > $O/b_c5.json 2> $O/b_c5.err
python bench.py --workload c3 > $O/b_c3.json 2> $O/b_c3.err
python bench.py --workload c4 > $O/b_c4.json 2> $O/b_c4.err
python bench.py --workload c1 > $O/b_c1.json 2> $O/b_c1.err
python bench.py --workload graph --no-cpu > $O/b_graph.json 2> $O/b_graph.err
python bench.py --impl reference --steps 3 --warmup 1 > $O/b_ref.json 2> $O/b_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c2.csv \
  python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > $O/ncu_launch.log 2>&1
tail -2 $O/pytest_gpu.log
