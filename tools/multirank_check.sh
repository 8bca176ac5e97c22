# Functional run of bench.py's N>1 paths on one GPU: 2 ranks over gloo sharing
# cuda:0 -- list sharding of config C (--small: 10M entries; the exchange goes
# through torch.distributed because NCCL needs one GPU per rank) and
# query-parallel replicas of config B, max-over-ranks timing. Its numbers are
# not bench values (the ranks share one device).
set -x
OUT=gpurun_out/${TAG:-mr}; mkdir -p $OUT
for MODE in shard-lists replicas; do
PRAG_BENCH_MODE=$MODE PRAG_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --small --no-sweep --steps 5 --warmup 3 \
  > $OUT/bench_n2_${MODE}.json 2> $OUT/bench_n2_${MODE}.err; echo "rc=$?" >> $OUT/bench_n2_${MODE}.err
done
ls -la $OUT
