# Round-2 re-entry check (one B200): fresh build's GPU suite, smoke and the bench line.
OUT=gpurun_out/${TAG:-r4a}; mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
tail -3 $OUT/pytest_gpu.log; tail -1 $OUT/smoke.log; cut -c1-400 $OUT/bench.json
