# Config C batch-1 chain traces (PRAG_CHAIN_TRACE build) and the N>1 functional check with striped shards.
OUT=gpurun_out/${TAG:-r4d}; mkdir -p $OUT
for s in "--nq 1 --nprobe 1 --k 2" "--nq 1 --nprobe 16 --k 2" "--nq 1 --nprobe 64 --k 10" "--nq 64 --nprobe 16 --k 10"; do
  PRAG_GPU_LIB=$PWD/variants/lib_trace.so timeout 600 python tools/chain_trace.py --n 100000000 --nlist 16384 --m 64 --seed 3 $s >> $OUT/chain_C.jsonl 2>> $OUT/chain_C.err
done
TAG=${TAG:-r4d} bash tools/multirank_check.sh > $OUT/multirank.log 2>&1
ls $OUT
