# GPU tests + bench lines (c2 default with validation and the reference CPU
# baseline, c5, c3, c4) + the reference arm
O=gpurun_out
nproc > $O/nproc.txt
timeout 1500 python -m pytest tests -x -q -m gpu > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
python bench.py > $O/b_c2.json 2> $O/b_c2.err
python bench.py --workload c5 --no-cpu > $O/b_c5.json 2> $O/b_c5.err
python bench.py --workload c4 --no-cpu > $O/b_c4.json 2> $O/b_c4.err
python bench.py --workload c3 --no-cpu > $O/b_c3.json 2> $O/b_c3.err
python bench.py --impl reference --steps 3 --warmup 1 > $O/b_ref.json 2> $O/b_ref.err
tail -3 $O/pytest_gpu.log
