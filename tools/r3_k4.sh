set -x
OUT=gpurun_out/${TAG:-r3m}; mkdir -p $OUT
PRAG_GPU_LIB=$PWD/variants/lib_trace.so timeout 600 python tools/chain_trace.py --nq 64 --nprobe 16 --k 10 > $OUT/chain.jsonl 2> $OUT/chain.err
PRAG_GPU_LIB=$PWD/variants/lib_trace.so timeout 600 python tools/chain_trace.py --nq 8 --nprobe 64 --k 10 >> $OUT/chain.jsonl 2>> $OUT/chain.err
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_synthetic.py tests/test_gpu_plan.py tests/test_gpu_pool_paths.py -x -q -m gpu > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "rc=$?" >> $OUT/bench.err
