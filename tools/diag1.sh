set -x
OUT=gpurun_out/diag1; mkdir -p $OUT
nvidia-smi > $OUT/smi.txt 2>&1; nproc > $OUT/nproc.txt
timeout 600 python tools/diag_latency.py > $OUT/diag.jsonl 2> $OUT/diag.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:scan_skew -s 1 -c 1 -o $OUT/scan_full -f python tools/prof_search.py --iters 3 > $OUT/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:scan_skew -s 1 -c 1 -o $OUT/scan_full_nq1 -f python tools/prof_search.py --iters 3 --nq 1 > $OUT/ncu_full_nq1.log 2>&1
ls -la $OUT
