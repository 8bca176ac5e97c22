# Functional run of bench.py's N>1 path on one GPU: 2 ranks over gloo sharing
# cuda:0 (sharded load, packed all-gather, exact merge, max-over-ranks timing).
# Its numbers are not bench values (ranks share one device).
set -x
OUT=gpurun_out/${TAG:-mr}; mkdir -p $OUT
PRAG_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --small --no-sweep --steps 5 --warmup 3 \
  > $OUT/bench_n2_gloo.json 2> $OUT/bench_n2_gloo.err; echo "rc=$?" >> $OUT/bench_n2_gloo.err
ls -la $OUT
