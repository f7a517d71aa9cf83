cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for C in "c2" "c3 --pairs 4000" "c4 --pairs 256" "c5 --pairs 500"; do
timeout 900 python bench.py --config $C --steps 3 --warmup 2 --no-cpu > gpurun_out/bench_cfg.log 2>&1; echo "rc=$?"
tail -1 gpurun_out/bench_cfg.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$C', 'value', d['value'], 'e2e', d['e2e']['value'], 'ms', d['ms_per_step'], 'tests/step', d['tests_per_step'], 'contacts', d['raw_contacts_per_step'], d['breakdown_ms_per_step'], 'setup', d['setup_s'], d['config'].get('problems_per_gpu'))" || tail -5 gpurun_out/bench_cfg.log
done
