cd $GRAFT_REPO_ROOT
for v in build/variants/*.so; do
  for m in near far; do LTSG_LIB=$PWD/$v timeout 300 python tools/rowbench.py 4194304 $m 2>&1 | tail -1; done
  LTSG_LIB=$PWD/$v timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench c1', d['value'], d['roofline']['achieved'], d['breakdown_ms_per_step']['screen'], d['e2e'])"
done
