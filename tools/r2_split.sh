set -x
OUT=gpurun_out/${TAG:-split}; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale_parity.py tests/test_gpu_synthetic.py tests/test_gpu_sharded.py -q -x > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
timeout 900 python tools/item_sweep.py --rows 1:64,1:128,1:256,8:64 --env PRAG_GPU_SPLIT_ITEMS --per 0,148,296,592 > $OUT/splitC.jsonl 2> $OUT/splitC.err
timeout 600 python tools/item_sweep.py --n 10000000 --nlist 4096 --m 32 --seed 1 --rows 64:16,16:16,1:16,64:64 --env PRAG_GPU_SPLIT_ITEMS --per 0,148,296,592 > $OUT/splitB.jsonl 2> $OUT/splitB.err
