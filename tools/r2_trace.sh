set -x
OUT=gpurun_out/${TAG:-tr}; mkdir -p $OUT
touch paper_2403_05676_b200/csrc/scan_skew.cu
make -C paper_2403_05676_b200/csrc -j8 EXTRA=-DPRAG_K3_TRACE > $OUT/build.log 2>&1
timeout 600 python tools/k3_trace.py --nq 1 --nprobe 128 > $OUT/trC_1_128.json 2> $OUT/trC.err
timeout 600 python tools/k3_trace.py --nq 1 --nprobe 64 > $OUT/trC_1_64.json 2>> $OUT/trC.err
timeout 600 python tools/k3_trace.py --nq 64 --nprobe 16 > $OUT/trC_64_16.json 2>> $OUT/trC.err
timeout 600 python tools/k3_trace.py --n 10000000 --nlist 4096 --m 32 --seed 1 --nq 64 --nprobe 16 > $OUT/trB_64_16.json 2> $OUT/trB.err
