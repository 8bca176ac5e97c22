# K1b one-batch rescoring boundary: the coarse parity tests with window sizes around 128.
OUT=gpurun_out/${TAG:-r4o}; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "tc_coarse" > $OUT/pytest_tc_coarse.log 2>&1; echo "rc=$?" >> $OUT/pytest_tc_coarse.log
tail -3 $OUT/pytest_tc_coarse.log
