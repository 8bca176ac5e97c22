set -x
OUT=gpurun_out/r2j; mkdir -p $OUT
timeout 900 python tools/item_sweep.py --rows 1:64,1:128,8:64,64:16 --per 1,2,4,8 > $OUT/sweepC.jsonl 2> $OUT/sweepC.err
timeout 600 python tools/item_sweep.py --n 10000000 --nlist 4096 --m 32 --seed 1 --rows 64:16,16:16,1:16,64:64 --per 1,2,4 > $OUT/sweepB.jsonl 2> $OUT/sweepB.err
