# Shard balance (tools/shard_balance.py) on the final code.
OUT=gpurun_out/${TAG:-r4m}; mkdir -p $OUT
timeout 1800 python tools/shard_balance.py > $OUT/shard_balance.json 2> $OUT/shard_balance.err; echo "rc=$?" >> $OUT/shard_balance.err
tail -1 $OUT/shard_balance.err
