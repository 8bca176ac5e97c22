OUT=gpurun_out/${TAG:-r3q2}; mkdir -p $OUT
timeout 900 python tools/item_sweep.py --rows 1:64,1:128,8:64 --env PRAG_GPU_L2_PREFETCH --per 0,2,4,8,16 --reps 7 > $OUT/C_pf.jsonl 2>>$OUT/err
