#!/bin/bash
# One GPU box session: parity tests, bench line, ncu launch list + full capture
# of the scan kernel. Outputs under gpurun_out/ (scratch; summaries go to profiles/).
set -x
OUT=gpurun_out/${TAG:-run}
mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
nproc > $OUT/nproc.txt; lscpu > $OUT/lscpu.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 1500 python bench.py ${BENCH_ARGS} > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
if [ -z "$NO_NCU" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
   -k regex:'coarse|select|plan|lut|scan|merge' python tools/prof_search.py --iters 3 > $OUT/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:scan_skew -s 1 -c 1 \
   -o $OUT/scan_full -f python tools/prof_search.py --iters 3 > $OUT/ncu_full.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'coarse|lut_kernel|select_probe|select_pool' -s 4 -c 4 \
   -o $OUT/aux_full -f python tools/prof_search.py --iters 3 > $OUT/ncu_aux.log 2>&1
fi
ls -la $OUT
