set -x
OUT=gpurun_out/${TAG:-sw}; mkdir -p $OUT
timeout 600 python tools/item_sweep.py --n 10000000 --nlist 4096 --m 32 --seed 1 --rows 64:16,1:16,64:64 --env PRAG_GPU_L2_PREFETCH --per 0,2,4,8,16 > $OUT/pfB.jsonl 2> $OUT/pfB.err
timeout 900 python tools/item_sweep.py --rows 1:64,1:128,64:16 --env PRAG_GPU_L2_PREFETCH --per 0,2,4,8 > $OUT/pfC.jsonl 2> $OUT/pfC.err
for pf in 0 8; do
PRAG_GPU_L2_PREFETCH=$pf timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:scan_skew -s 2 -c 1 --csv python tools/prof_search.py --iters 3 > $OUT/ncu_pf$pf.csv 2>/dev/null
done
