# K1b block size A/B (PRAG_GPU_K1B_THREADS 512 vs 1024): GPU suite, chain latency at configs B and C, chain traces.
OUT=gpurun_out/${TAG:-r4f}; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
tail -2 $OUT/pytest_gpu.log
for t in 512 1024 512 1024; do
  PRAG_GPU_K1B_THREADS=$t timeout 600 python tools/diag_latency.py --reps 20 >> $OUT/diag_B_t$t.jsonl 2>> $OUT/diag.err
  PRAG_GPU_K1B_THREADS=$t timeout 600 python tools/diag_latency.py --n 100000000 --nlist 16384 --m 64 --seed 3 --reps 20 >> $OUT/diag_C_t$t.jsonl 2>> $OUT/diag.err
done
for t in 512 1024; do
  for s in "--nq 1 --nprobe 16 --k 2" "--nq 64 --nprobe 16 --k 10"; do
    PRAG_GPU_K1B_THREADS=$t PRAG_GPU_LIB=$PWD/variants/lib_trace.so timeout 600 python tools/chain_trace.py --n 100000000 --nlist 16384 --m 64 --seed 3 $s >> $OUT/chain_C_t$t.jsonl 2>> $OUT/chain.err
    PRAG_GPU_K1B_THREADS=$t PRAG_GPU_LIB=$PWD/variants/lib_trace.so timeout 600 python tools/chain_trace.py $s >> $OUT/chain_B_t$t.jsonl 2>> $OUT/chain.err
  done
done
