set -x
OUT=gpurun_out/${TAG:-b1}; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_batch1.py -x -q > $OUT/pytest_b1.log 2>&1; echo "rc=$?" >> $OUT/pytest_b1.log
timeout 600 python tools/b1_time.py > $OUT/b1time.jsonl 2> $OUT/b1time.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_nq1.csv python tools/prof_search.py --iters 3 --nq 1 --k 2 > /dev/null 2>&1
if [ -n "$FULL" ]; then timeout 600 ncu --set full --clock-control none --import-source on -k regex:search1 -s 2 -c 1 -o $OUT/k0 -f python tools/prof_search.py --iters 3 --nq 1 --k 2 > $OUT/ncu_k0.log 2>&1; python tools/ncu_summary.py $OUT/k0.ncu-rep 0.01 > $OUT/k0.txt 2>&1; fi
