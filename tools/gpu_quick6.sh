cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider --tb=short > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED|Error" gpurun_out/pytest_gpu.log | tail -20
for c in ${@:-c4 c5}; do
timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu --no-allpairs > gpurun_out/bench_$c.log 2>&1; echo "$c rc=$?"
tail -1 gpurun_out/bench_$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], '%.4g' % d['value'], 'ms %.3f' % d['ms_per_step'], 'e2e %.4g' % d['e2e']['value'], 'ach', d['roofline']['achieved'], d['roofline']['screen_rows_exact_per_step'], d['breakdown_ms_per_step'])"
done
