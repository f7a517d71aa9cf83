cd $GRAFT_REPO_ROOT
for c in ${@:-c1}; do
  echo "== $c"
  timeout 600 python tools/trace_search.py --config $c 2>&1 | grep -v Warning | tail -14
done
