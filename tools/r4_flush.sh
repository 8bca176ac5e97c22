# K1b phases at config C batch 1 with and without the L2 flush (instruction-cache hypothesis).
OUT=gpurun_out/${TAG:-r4e}; mkdir -p $OUT
for fl in none read write; do
  PRAG_GPU_LIB=$PWD/variants/lib_trace.so timeout 600 python tools/chain_trace.py --n 100000000 --nlist 16384 --m 64 --seed 3 --nq 1 --nprobe 16 --k 2 --flush $fl >> $OUT/chain_C_flush.jsonl 2>> $OUT/chain_C_flush.err
done
