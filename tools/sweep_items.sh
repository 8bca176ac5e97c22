# Item-size sensitivity of the scan (config B): PRAG_GPU_ITEMS_PER_CTA over $ITEMS (default 1 2 3 4 6)
set -x
OUT=gpurun_out/${TAG:-items}; mkdir -p $OUT
for v in ${ITEMS:-1 2 3 4 6}; do PRAG_GPU_ITEMS_PER_CTA=$v timeout 600 python tools/diag_latency.py > $OUT/diag_ipc$v.jsonl 2> $OUT/diag_ipc$v.err; done
ls -la $OUT
