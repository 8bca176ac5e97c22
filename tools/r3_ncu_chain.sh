set -x
OUT=gpurun_out/${TAG:-chain}; mkdir -p $OUT
for kn in lut_image select_window select_pool; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$kn -s 2 -c 1 -o $OUT/$kn -f python tools/prof_search.py --iters 3 > $OUT/ncu_$kn.log 2>&1
  python tools/ncu_summary.py $OUT/$kn.ncu-rep 0.01 > $OUT/$kn.txt 2>&1
done
