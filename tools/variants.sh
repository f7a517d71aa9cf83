cd $GRAFT_REPO_ROOT
for v in build/variants/*.so; do
  echo "== $v"
  LTSG_LIB=$PWD/$v timeout 600 python bench.py --config c4 --pairs 512 --steps 3 --warmup 2 --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c4', '%.4g' % d['value'], d['roofline']['achieved'], d['breakdown_ms_per_step']['screen'])"
done
