# Copies one tools/r3_final.sh session (gpurun_out/$TAG) into profiles/${TAG}_* and refreshes the K3 traffic stamp.
set -e
T=${1:?tag}; S=gpurun_out/$T; P=profiles/$T
cp $S/pytest_gpu.log ${P}_pytest_gpu.log; cp $S/smoke.log ${P}_smoke.log; cp $S/bench.json ${P}_bench.json
cp $S/bench_reference_arm.json ${P}_bench_reference_arm.json; cp $S/bench_configC.json ${P}_bench_configC.json
cp $S/bench_configC_reference_arm.json ${P}_bench_configC_reference_arm.json
cp $S/bench_n2_shard-lists.json ${P}_bench_n2_shard-lists_gloo_functional.json
cp $S/bench_n2_replicas.json ${P}_bench_n2_replicas_gloo_functional.json
cp $S/k3_B.txt ${P}_k3_B_ncu.txt; cp $S/k1_B.txt ${P}_k1_coarse_tc_ncu.txt
cp $S/k3C_1_128.txt ${P}_k3_configC_nq1_np128_ncu.txt; cp $S/k3C_1_64.txt ${P}_k3_configC_nq1_np64_ncu.txt
cp $S/launches_nq64.csv ${P}_launches_nq64.csv; cp $S/launches_nq1.csv ${P}_launches_nq1.csv
cp $S/chain_trace.jsonl ${P}_chain_trace.jsonl; cp $S/hbm_roofline.json ${P}_hbm_roofline_100M_m64.json
cp $S/config_d.json ${P}_config_d_1B_m64.json; cp $S/piperag.json ${P}_piperag_loop.json
cp $S/b1lat.jsonl ${P}_batch1_latency.jsonl; cp $S/b1time.jsonl ${P}_batch1_kernel_vs_chain.jsonl
cp $S/nvidia-smi.txt ${P}_nvidia-smi.txt; cp $S/traffic.json profiles/ncu_scan_traffic.json
echo "copied $T"
