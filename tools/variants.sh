cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in build/variants/*.so; do
  echo "== $v"
  LTSG_LIB=$PWD/$v timeout 300 python tools/rowbench.py 4194304 2>&1 | tail -1
  LTSG_LIB=$PWD/$v timeout 600 python bench.py --pairs 256 --steps 3 --warmup 2 --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', d['value'], d['roofline']['achieved'], d['breakdown_ms_per_step'])"
done
