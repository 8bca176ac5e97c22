# Round-2 GPU session: parity suite, synthetic HBM rows, ncu of K3 on them, bench.
# env: TAG (output dir), SKIP_TESTS, ROWS (synth rows), NCU_ROWS (one ncu --set full per row), BENCH=1
set -x
OUT=gpurun_out/${TAG:-r2}; mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
if [ -z "$SKIP_TESTS" ]; then
  timeout 1200 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
fi
if [ -n "$ROWS" ]; then
  timeout 600 python tools/synth_rows.py --rows "$ROWS" $SYNTH_ARGS > $OUT/synth_rows.json 2> $OUT/synth_rows.err
fi
for r in $NCU_ROWS; do
  n=$(echo $r | tr ':' '_')
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:scan_skew -s 2 -c 1 -o $OUT/k3_$n -f \
    python tools/synth_rows.py --ncu --rows $r $SYNTH_ARGS > $OUT/ncu_$n.log 2>&1
  python tools/ncu_summary.py $OUT/k3_$n.ncu-rep 0.004 > $OUT/k3_$n.txt 2>&1
done
if [ -n "$NCU_B" ]; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:scan_skew -s 2 -c 1 -o $OUT/k3_B -f \
    python tools/prof_search.py --iters 3 > $OUT/ncu_B.log 2>&1
  python tools/ncu_summary.py $OUT/k3_B.ncu-rep 0.004 > $OUT/k3_B.txt 2>&1
fi
if [ -n "$BENCH" ]; then timeout 1500 python bench.py $BENCH_ARGS > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err; fi
ls -la $OUT
