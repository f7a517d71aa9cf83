cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider --tb=short > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED|Error" gpurun_out/pytest_gpu.log | tail -20
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_c1.log 2>&1; echo "rc=$?"
tail -1 gpurun_out/bench_c1.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c1', '%.4g' % d['value'], 'e2e %.4g' % d['e2e']['value'], d['roofline']['achieved'], d['roofline_distance_kernel'], d['clocks'])"
timeout 900 python bench.py --exhaustive --pairs 256 --steps 3 --warmup 2 --no-cpu --no-allpairs > gpurun_out/bench_ex.log 2>&1; echo "rc=$?"
tail -1 gpurun_out/bench_ex.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c1 ex', '%.4g' % d['value'], 'ms', d['ms_per_step'], d['tests_per_step'], d['roofline']['screen_rows_exact_per_step'], d['breakdown_ms_per_step'])"
