# Item-size sensitivity of the scan (config B): PRAG_GPU_ITEMS_PER_CTA in {3, 8, 24, 64}
set -x
OUT=gpurun_out/${TAG:-items}; mkdir -p $OUT
for v in 3 8 24 64; do PRAG_GPU_ITEMS_PER_CTA=$v timeout 600 python tools/diag_latency.py > $OUT/diag_ipc$v.jsonl 2> $OUT/diag_ipc$v.err; done
ls -la $OUT
