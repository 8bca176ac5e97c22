# GPU session: parity suite, latency breakdown, ncu capture of the scan kernel.
set -x
OUT=gpurun_out/${TAG:-diag2}; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 600 python tools/diag_latency.py > $OUT/diag.jsonl 2> $OUT/diag.err
if [ -z "$NO_NCU" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:scan_skew -s 1 -c 1 -o $OUT/scan_full -f python tools/prof_search.py --iters 3 > $OUT/ncu_full.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv python tools/prof_search.py --iters 3 > $OUT/ncu_launch.log 2>&1
fi
ls -la $OUT
