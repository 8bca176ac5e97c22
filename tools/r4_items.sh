# K3 work-item size at small batches (config C trained fixture and config B): PRAG_GPU_ITEMS_PER_CTA sweep.
OUT=gpurun_out/${TAG:-r4c}; mkdir -p $OUT
timeout 1500 python tools/item_sweep.py --rows 1:16,1:64,1:128,4:64,8:64,64:16 --per 1,2,4,8,16 > $OUT/items_C.jsonl 2> $OUT/items_C.err
timeout 900 python tools/item_sweep.py --n 10000000 --nlist 4096 --m 32 --seed 1 --rows 1:16,1:64,1:128,8:64,64:16 --per 1,2,4,8,16 > $OUT/items_B.jsonl 2> $OUT/items_B.err
cat $OUT/items_C.jsonl $OUT/items_B.jsonl
for c in 0 1; do timeout 600 python tools/diag_latency.py --n 100000000 --nlist 16384 --m 64 --seed 3 --reps 10 --coarse $c > $OUT/diag_C_coarse$c.jsonl 2> $OUT/diag_C_coarse$c.err; done
cat $OUT/diag_C_coarse*.jsonl
