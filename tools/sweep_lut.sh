# K2 (LUT + planner) CTA-shape sweep: launch-list durations at nq 64 / nq 1 (nprobe 16).
OUT=gpurun_out/${TAG:-lut}; mkdir -p $OUT
for cfg in "4,4" "2,1" "2,2" "2,4" "4,1" "4,2" "8,1"; do
  for nq in 64 1; do
    PRAG_GPU_LUT_CFG=$cfg timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:lut_image --csv \
      --log-file $OUT/lut_${cfg/,/_}_nq$nq.csv python tools/prof_search.py --iters 3 --nq $nq > /dev/null 2>&1
  done
done
