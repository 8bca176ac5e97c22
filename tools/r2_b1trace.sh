set -x
OUT=gpurun_out/${TAG:-b1t}; mkdir -p $OUT
touch paper_2403_05676_b200/csrc/batch1.cu
make -C paper_2403_05676_b200/csrc -j8 EXTRA=-DPRAG_B1_TRACE > $OUT/build.log 2>&1
for np in 1 16 64; do timeout 300 python tools/b1_trace.py --nprobe $np > $OUT/b1trace_$np.json 2>> $OUT/b1trace.err; done
