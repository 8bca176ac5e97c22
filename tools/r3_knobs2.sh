OUT=gpurun_out/${TAG:-r3x}; mkdir -p $OUT
timeout 600 python tools/item_sweep.py --n 10000000 --nlist 4096 --m 32 --seed 1 --rows 64:16,8:64,64:128 --env PRAG_GPU_TAIL_ONDEMAND --per 0,592,1184,1000000 --reps 11 > $OUT/B_tail.jsonl 2>>$OUT/err
timeout 900 python tools/item_sweep.py --rows 1:64,1:128,8:64,64:16 --env PRAG_GPU_TAIL_ONDEMAND --per 0,592,1000000 --reps 7 > $OUT/C_tail.jsonl 2>>$OUT/err
