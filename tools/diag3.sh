# GPU session: parity suite, latency breakdown, config-E loop, ncu launch list.
set -x
OUT=gpurun_out/${TAG:-diag}; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 600 python tools/diag_latency.py > $OUT/diag.jsonl 2> $OUT/diag.err
timeout 900 python tools/piperag_loop.py > $OUT/piperag.json 2> $OUT/piperag.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv python tools/prof_search.py --iters 2 > /dev/null 2>&1
ls -la $OUT
