# Round-2 evidence session (final code) (one B200): parity suite, smoke, bench lines (config B,
# config C, reference arms), ncu captures (K3 config B + traffic stamp, K1 tensor
# pipe, config C nq1 rows), launch lists, HBM rows (config C trained, config D 1B),
# config E loop, batch-1 timings, N>1 functional check.
set -x
OUT=gpurun_out/${TAG:-fin}; mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1; nproc > $OUT/nproc.txt; lscpu > $OUT/lscpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:scan_skew -s 2 -c 1 -o $OUT/k3_B -f python tools/prof_search.py --iters 3 > $OUT/ncu_B.log 2>&1
python tools/ncu_summary.py $OUT/k3_B.ncu-rep 0.004 > $OUT/k3_B.txt 2>&1
python tools/write_traffic.py $OUT/k3_B.ncu-rep > $OUT/traffic.json 2>&1
timeout 600 ncu --set full --clock-control none -k regex:coarse_tc -s 2 -c 1 -o $OUT/k1_B -f python tools/prof_search.py --iters 3 > $OUT/ncu_k1.log 2>&1
python tools/ncu_summary.py $OUT/k1_B.ncu-rep > $OUT/k1_B.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_nq64.csv python tools/prof_search.py --iters 2 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_nq1.csv python tools/prof_search.py --iters 2 --nq 1 > /dev/null 2>&1
timeout 1500 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
timeout 900 python bench.py --impl reference > $OUT/bench_reference_arm.json 2> $OUT/bench_ref.err; echo "rc=$?" >> $OUT/bench_ref.err
PRAG_BENCH_CONFIG=C timeout 1500 python bench.py > $OUT/bench_configC.json 2> $OUT/bench_C.err; echo "rc=$?" >> $OUT/bench_C.err
PRAG_BENCH_CONFIG=C PRAG_BENCH_MODE=single timeout 900 python bench.py --impl reference > $OUT/bench_configC_reference_arm.json 2> $OUT/bench_refC.err; echo "rc=$?" >> $OUT/bench_refC.err
timeout 900 python tools/hbm_roofline.py > $OUT/hbm_roofline.json 2> $OUT/hbm_roofline.err
for r in 1:128 1:64; do
  nq=${r%%:*}; np=${r##*:}
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:scan_skew -s 2 -c 1 -o $OUT/k3C_$nq\_$np -f \
    python tools/prof_search.py --n 100000000 --nlist 16384 --m 64 --seed 3 --nq $nq --nprobe $np --iters 3 > $OUT/ncuC_$nq\_$np.log 2>&1
  python tools/ncu_summary.py $OUT/k3C_$nq\_$np.ncu-rep 0.004 > $OUT/k3C_$nq\_$np.txt 2>&1
done
timeout 900 python tools/piperag_loop.py --rsms 0,8,16 > $OUT/piperag.json 2> $OUT/piperag.err
timeout 600 python tools/b1_time.py > $OUT/b1time.jsonl 2> $OUT/b1time.err
timeout 600 python tools/batch1_latency.py > $OUT/b1lat.jsonl 2> $OUT/b1lat.err
TAG=$TAG bash tools/multirank_check.sh > /dev/null 2>&1
timeout 1500 python tools/config_d.py > $OUT/config_d.json 2> $OUT/config_d.err
ls -la $OUT
if [ -f variants/lib_trace.so ]; then
  for s in "--nq 64 --nprobe 16 --k 10" "--nq 1 --nprobe 16 --k 2" "--nq 8 --nprobe 64 --k 10"; do
    PRAG_GPU_LIB=$PWD/variants/lib_trace.so timeout 600 python tools/chain_trace.py $s >> $OUT/chain_trace.jsonl 2>> $OUT/chain_trace.err
  done
fi
