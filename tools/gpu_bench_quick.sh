cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py --steps ${STEPS:-10} --warmup 3 --no-cpu ${EXTRA:-} > gpurun_out/bq.log 2>&1; echo "rc=$?"
python - <<'PY'
import json
d=json.loads(open('gpurun_out/bq.log').read().strip().splitlines()[-1])
print('value %.3e ms %.3f' % (d['value'], d['ms_per_step']))
print('e2e', json.dumps(d['e2e']))
print('e2e_cold', json.dumps(d.get('e2e_cold')))
PY
tail -3 gpurun_out/bq.log | head -2
