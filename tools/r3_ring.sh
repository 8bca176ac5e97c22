# quick K3 check: parity on the fast paths, config B bench, HBM rows subset.
set -x
OUT=gpurun_out/${TAG:-r3j}; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_synthetic.py tests/test_gpu_plan.py tests/test_gpu_batch1.py -x -q -m gpu > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "rc=$?" >> $OUT/bench.err
if [ -n "$HBM" ]; then timeout 1200 python tools/hbm_roofline.py $HBM > $OUT/hbm.json 2> $OUT/hbm.err; fi
