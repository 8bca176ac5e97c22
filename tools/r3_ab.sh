# A/B of library builds (variants/*.so via PRAG_GPU_LIB) on K3 rows of config B and config C.
OUT=gpurun_out/${TAG:-r3l}; mkdir -p $OUT
for v in default ${VARIANTS:-}; do
  if [ "$v" = default ]; then unset PRAG_GPU_LIB; else export PRAG_GPU_LIB=$PWD/variants/$v.so; fi
  timeout 600 python tools/item_sweep.py --n 10000000 --nlist 4096 --m 32 --seed 1 --rows ${ROWS_B:-64:16,1:16,8:64,64:128} --env PRAG_AB_DUMMY --per 0 --reps 9 2>>$OUT/ab.err | sed "s/^/{\"lib\": \"$v\", \"cfg\": \"B\", \"r\": /; s/$/}/" >> $OUT/ab.jsonl
  if [ -z "$NO_C" ]; then
  timeout 900 python tools/item_sweep.py --rows ${ROWS_C:-1:64,1:128,8:64,64:16} --env PRAG_AB_DUMMY --per 0 --reps 7 2>>$OUT/ab.err | sed "s/^/{\"lib\": \"$v\", \"cfg\": \"C\", \"r\": /; s/$/}/" >> $OUT/ab.jsonl
  fi
done
