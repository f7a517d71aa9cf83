cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider --tb=short > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED|Error" gpurun_out/pytest_gpu.log | tail -20
for ENV in "LTSG_NO_STATIC=0" "LTSG_NO_STATIC=1"; do
env $ENV timeout 900 python bench.py --steps 5 --warmup 2 --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$ENV', d['value'], 'e2e', d['e2e']['value'], 'ms', d['ms_per_step'], d['roofline']['achieved'], d['breakdown_ms_per_step'])"
done
