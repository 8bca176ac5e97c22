# Config D 1B sampled parity on the final code (gated test), plus the sharded/striped parity suite.
OUT=gpurun_out/${TAG:-r4n}; mkdir -p $OUT
PRAG_CONFIG_D=1 timeout 1500 python -m pytest tests/test_gpu_synthetic.py -m gpu -q -s -k config_d_1b > $OUT/config_d_1B_sampled_parity.log 2>&1; echo "rc=$?" >> $OUT/config_d_1B_sampled_parity.log
tail -3 $OUT/config_d_1B_sampled_parity.log
