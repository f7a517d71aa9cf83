# bench each build/variants/*.so on config $1 (default c1)
cd $GRAFT_REPO_ROOT
CFG=${1:-c1}
EXTRA=${2:-}
for v in build/variants/*.so; do
  echo "== $v"
  LTSG_LIB=$PWD/$v timeout 600 python bench.py --config $CFG --steps 5 --warmup 3 --no-cpu --no-allpairs $EXTRA 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], '%.4g' % d['value'], 'ms %.3f' % d['ms_per_step'], d['roofline']['achieved'], d['breakdown_ms_per_step']['screen'])"
done
