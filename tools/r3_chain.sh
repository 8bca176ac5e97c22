set -x
mkdir -p gpurun_out/r3g
for s in "--nq 64 --nprobe 16 --k 10" "--nq 64 --nprobe 128 --k 10" "--nq 1 --nprobe 16 --k 2" "--nq 8 --nprobe 64 --k 10"; do
  timeout 600 python tools/chain_trace.py $s >> gpurun_out/r3g/chain.jsonl 2>>gpurun_out/r3g/chain.err
done
