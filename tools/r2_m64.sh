set -x
OUT=gpurun_out/${TAG:-m64}; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_synthetic.py tests/test_gpu_scale_parity.py -q -x -k "64 or synthetic or config_c" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
timeout 900 python tools/item_sweep.py --rows 1:64,1:128,1:256,8:64,64:16 --per 1 > $OUT/sweepC.jsonl 2> $OUT/sweepC.err
