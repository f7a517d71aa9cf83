# moving-path iteration: GPU parity suite, c4 trace (2048 pairs), c4 + c5 bench lines
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider --tb=short -rf -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED|Error" gpurun_out/pytest_gpu.log | tail -8
timeout 600 python tools/trace_search.py --config c4 --pairs 2048 > gpurun_out/trace_c4.log 2>&1; echo "trace rc=$?"
grep "ltsg trace\] rows\|traverse\|problems" gpurun_out/trace_c4.log | cut -c1-400
for c in c4 c5; do
timeout 900 python bench.py --only --config $c --steps 5 --warmup 3 --no-cpu --no-allpairs > gpurun_out/bench_$c.log 2>&1; echo "$c rc=$?"
python tools/bench_table.py gpurun_out/bench_$c.log | sed -n 2p
done
