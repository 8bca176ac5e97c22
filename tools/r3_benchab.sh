OUT=gpurun_out/${TAG:-r3ab}; mkdir -p $OUT
for v in default ${VARIANTS:-}; do
  for rep in 1 2; do
    if [ "$v" = default ]; then unset PRAG_GPU_LIB; else export PRAG_GPU_LIB=$PWD/variants/$v.so; fi
    timeout 900 python bench.py --steps 50 --warmup 5 > $OUT/bench_${v}_$rep.json 2> $OUT/bench_${v}_$rep.err
  done
done
