# K1b U bound for 32 < nprobe <= 128: GPU suite, chain traces, batch-1 latency, then the full final session.
OUT=gpurun_out/${TAG:-r4k}; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
tail -2 $OUT/pytest_gpu.log
for s in "--nq 8 --nprobe 64 --k 10" "--nq 1 --nprobe 64 --k 2" "--nq 64 --nprobe 128 --k 10"; do
  PRAG_GPU_LIB=$PWD/variants/lib_trace.so timeout 600 python tools/chain_trace.py $s >> $OUT/chain_ub.jsonl 2>> $OUT/chain.err
done
