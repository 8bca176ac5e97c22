# K1b tail (one-batch rescoring when the window fits both buffers, warp-parallel ranking): GPU suite, traces, latency, bench.
OUT=gpurun_out/${TAG:-r4i}; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
tail -2 $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
for s in "--nq 64 --nprobe 16 --k 10" "--nq 1 --nprobe 16 --k 2" "--nq 8 --nprobe 64 --k 10"; do
  PRAG_GPU_LIB=$PWD/variants/lib_trace.so timeout 600 python tools/chain_trace.py $s >> $OUT/chain_trace.jsonl 2>> $OUT/chain.err
done
PRAG_GPU_LIB=$PWD/variants/lib_trace.so timeout 600 python tools/chain_trace.py --n 100000000 --nlist 16384 --m 64 --seed 3 --nq 1 --nprobe 16 --k 2 >> $OUT/chain_C.jsonl 2>> $OUT/chain.err
timeout 600 python tools/diag_latency.py --reps 20 > $OUT/diag_B.jsonl 2>> $OUT/diag.err
timeout 600 python tools/diag_latency.py --n 100000000 --nlist 16384 --m 64 --seed 3 --reps 20 > $OUT/diag_C.jsonl 2>> $OUT/diag.err
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_nq64.csv python tools/prof_search.py --iters 2 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_nq1.csv python tools/prof_search.py --iters 2 --nq 1 > /dev/null 2>&1
timeout 600 python tools/b1_time.py > $OUT/b1time.jsonl 2> $OUT/b1time.err
timeout 600 python tools/batch1_latency.py > $OUT/b1lat.jsonl 2> $OUT/b1lat.err
cut -c1-200 $OUT/bench.json
