OUT=gpurun_out/${TAG:-r3p2}; mkdir -p $OUT
for mb in 0 16; do
  PRAG_GPU_L2_PERSIST=$mb PRAG_GPU_LIB=$PWD/variants/lib_trace.so timeout 600 python tools/chain_trace.py --nq 64 --nprobe 16 --k 10 >> $OUT/chain.jsonl 2>> $OUT/chain.err
  PRAG_GPU_L2_PERSIST=$mb timeout 900 python bench.py > $OUT/bench_$mb.json 2> $OUT/bench_$mb.err
done
