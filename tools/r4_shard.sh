# Striped list sharding on one B200: sharded parity tests, then the per-shard balance tool.
OUT=gpurun_out/${TAG:-r4b}; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_parity.py -m gpu -q -x > $OUT/pytest_sharded.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_sharded.log
tail -3 $OUT/pytest_sharded.log
timeout 1800 python tools/shard_balance.py > $OUT/shard_balance.json 2> $OUT/shard_balance.err; echo "rc=$?" >> $OUT/shard_balance.err
tail -3 $OUT/shard_balance.err
