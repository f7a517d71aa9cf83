# Per-config A/B of library variants: for each CFG in $CFGS, bench the default
# library and every variants/lib_*.so (--only, no CPU leg), print a table line.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for CFG in ${CFGS:-c1 c4}; do
  for v in default variants/lib_*.so; do
    if [ "$v" = default ]; then unset LTSG_LIB; else export LTSG_LIB=$v; fi
    timeout 900 python bench.py --only --config $CFG --steps ${STEPS:-10} --warmup 3 --no-cpu --no-allpairs > gpurun_out/var_${CFG}_$(basename $v .so).log 2>&1 || echo "FAIL $CFG $v"
    echo -n "$CFG $(basename $v .so): "; python tools/bench_table.py gpurun_out/var_${CFG}_$(basename $v .so).log | sed -n 2p
    python - gpurun_out/var_${CFG}_$(basename $v .so).log <<'PY'
import json,sys
d=json.loads([l for l in open(sys.argv[1]) if l.startswith('{')][-1])
print('   breakdown', json.dumps(d['breakdown_ms_per_step']), 'bound', d['roofline'].get('bound_rows_per_step'), 'exact', d['roofline'].get('exact_rows_per_step'), 'kern_ms', d['roofline'].get('kernel_ms_per_step'))
PY
  done
done
