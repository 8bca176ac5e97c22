# GPU session: parity suite, latency breakdown (nq 64 and nq 1 launch lists), bench line.
set -x
OUT=gpurun_out/${TAG:-s}; mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1; nproc > $OUT/nproc.txt; lscpu > $OUT/lscpu.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 600 python tools/diag_latency.py > $OUT/diag.jsonl 2> $OUT/diag.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_nq64.csv python tools/prof_search.py --iters 2 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_nq1.csv python tools/prof_search.py --iters 2 --nq 1 > /dev/null 2>&1
if [ -n "$BENCH" ]; then timeout 1500 python bench.py $BENCH_ARGS > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err; fi
if [ -n "$FULL" ]; then timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$FULL" -s ${SKIP:-1} -c 1 -o $OUT/full -f python tools/prof_search.py --iters 3 $PROF_ARGS > $OUT/ncu_full.log 2>&1; fi
ls -la $OUT
