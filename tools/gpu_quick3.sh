cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider --tb=short > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED|Error" gpurun_out/pytest_gpu.log | tail -20
for C in "c1" "c2" "c3 --pairs 4000"; do
timeout 900 python bench.py --config $C --steps 3 --warmup 2 --no-cpu > gpurun_out/bench_cfg.log 2>&1; echo "rc=$?"
tail -1 gpurun_out/bench_cfg.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$C', 'value', '%.3g' % d['value'], 'e2e', '%.3g' % d['e2e']['value'], 'ms', round(d['ms_per_step'],3), 'e2e ms', round(d['e2e']['ms_per_step'],2), d['e2e']['phases_ms_per_step'])" || tail -5 gpurun_out/bench_cfg.log
done
