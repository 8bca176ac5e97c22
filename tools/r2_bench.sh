# bench.py on one GPU: config B (default), config C unsharded, both reference arms, and the N>1 functional check.
set -x
OUT=gpurun_out/${TAG:-rb}; mkdir -p $OUT
timeout 1500 python bench.py $BENCH_ARGS > $OUT/bench.json 2> $OUT/bench.err; echo "rc=$?" >> $OUT/bench.err
PRAG_BENCH_CONFIG=C timeout 1500 python bench.py $BENCH_ARGS > $OUT/bench_C.json 2> $OUT/bench_C.err; echo "rc=$?" >> $OUT/bench_C.err
if [ -n "$REF" ]; then
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > $OUT/bench_ref.json 2> $OUT/bench_ref.err; echo "rc=$?" >> $OUT/bench_ref.err
PRAG_BENCH_CONFIG=C PRAG_BENCH_MODE=shard-lists timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > $OUT/bench_ref_C.json 2> $OUT/bench_ref_C.err; echo "rc=$?" >> $OUT/bench_ref_C.err
fi
if [ -n "$MR" ]; then TAG=${TAG:-rb} bash tools/multirank_check.sh; fi
ls -la $OUT
if [ -n "$NCU_B" ]; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:scan_skew -s 2 -c 1 -o $OUT/k3_B -f \
    python tools/prof_search.py --iters 3 > $OUT/ncu_B.log 2>&1
  python tools/ncu_summary.py $OUT/k3_B.ncu-rep 0.004 > $OUT/k3_B.txt 2>&1
  python tools/write_traffic.py $OUT/k3_B.ncu-rep > $OUT/traffic.json 2>&1
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_nq64.csv python tools/prof_search.py --iters 2 > /dev/null 2>&1
fi
