# Config C (trained 100M x 384, nlist 16384, m 64) HBM rows + ncu of K3 on the nq 1 rows.
set -x
OUT=gpurun_out/${TAG:-r2c}; mkdir -p $OUT
timeout 900 python tools/hbm_roofline.py > $OUT/hbm_roofline.json 2> $OUT/hbm_roofline.err
for r in ${NCU_ROWS:-1:128 1:64}; do
  nq=${r%%:*}; np=${r##*:}
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:scan_skew -s 2 -c 1 -o $OUT/k3C_$nq\_$np -f \
    python tools/prof_search.py --n 100000000 --nlist 16384 --m 64 --seed 3 --nq $nq --nprobe $np --iters 3 > $OUT/ncuC_$nq\_$np.log 2>&1
  python tools/ncu_summary.py $OUT/k3C_$nq\_$np.ncu-rep 0.004 > $OUT/k3C_$nq\_$np.txt 2>&1
done
ls -la $OUT
