# K3 knob sweeps (tail on-demand reservation, L2 prefetch distance) on config B and C rows.
OUT=gpurun_out/${TAG:-r3w}; mkdir -p $OUT
timeout 600 python tools/item_sweep.py --n 10000000 --nlist 4096 --m 32 --seed 1 --rows 64:16,8:64,1:16 --env PRAG_GPU_TAIL_ONDEMAND --per 0,148,296,592 --reps 9 > $OUT/B_tail.jsonl 2>>$OUT/err
timeout 600 python tools/item_sweep.py --n 10000000 --nlist 4096 --m 32 --seed 1 --rows 64:16,8:64 --env PRAG_GPU_L2_PREFETCH --per 0,2,4,8 --reps 9 > $OUT/B_pf.jsonl 2>>$OUT/err
timeout 900 python tools/item_sweep.py --rows 1:128,8:64,64:16 --env PRAG_GPU_TAIL_ONDEMAND --per 0,148,296 --reps 7 > $OUT/C_tail.jsonl 2>>$OUT/err
