# K1 with fp32 centroids split in SMEM: GPU suite, chain traces and latency at configs B and C.
OUT=gpurun_out/${TAG:-r4g}; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
tail -2 $OUT/pytest_gpu.log
timeout 600 python tools/diag_latency.py --reps 20 > $OUT/diag_B.jsonl 2>> $OUT/diag.err
timeout 600 python tools/diag_latency.py --n 100000000 --nlist 16384 --m 64 --seed 3 --reps 20 > $OUT/diag_C.jsonl 2>> $OUT/diag.err
for s in "--nq 1 --nprobe 16 --k 2" "--nq 64 --nprobe 16 --k 10"; do
  PRAG_GPU_LIB=$PWD/variants/lib_trace.so timeout 600 python tools/chain_trace.py --n 100000000 --nlist 16384 --m 64 --seed 3 $s >> $OUT/chain_C.jsonl 2>> $OUT/chain.err
  PRAG_GPU_LIB=$PWD/variants/lib_trace.so timeout 600 python tools/chain_trace.py $s >> $OUT/chain_B.jsonl 2>> $OUT/chain.err
done
timeout 900 python bench.py --no-sweep > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
cut -c1-300 $OUT/bench.json
